// icq_brute.cu — GPU ground truth: search_bruteforce.
//
// Reference: icq.search.search_bruteforce, /root/reference/pkg/src/icq/search.py:168-178
//     diff = x.astype(float64) - q ;  scores = (diff * diff).sum(axis=1)
//     order = lexsort((arange(n), scores))[:k]
// used for the truth="brute" recall of run_benchmark (evaluate.py:148) and
// `icq search --mode brute` (cli.py:140-144).  The reference cannot run it at
// c4/c5 (38 GB of raw float32 at c5 become 77 GB of float64 temporaries).
//
// Scores: the K1 LUT kernel (icq_lut.cu) with the raw rows in place of the
// codewords -- the same float64 direct difference in numpy's pairwise
// order, so every score is bitwise the reference's.  Queries run in groups
// whose (group x n) float64 score block fits a fixed budget.
// Selection, per query: every 64k-item chunk keeps its k best (score, id)
// (one CTA: radix select on the 64-bit score keys, then on the ids among
// the keys equal to the k-th, so ties go to the smaller id exactly as
// lexsort's (score, id) order), then one CTA selects the k best of the
// chunks' candidates and sorts them by (score, id).
#include <cstdint>

#include "icq_index.cuh"

namespace icq {

constexpr int kSelThreads = 512;
constexpr int kSelChunk = 65536;   // items per first-stage chunk
constexpr int kSelMaxK = 1024;     // bitonic sort capacity (smem)

__device__ __forceinline__ uint64_t score_key(double s) {
  // scores are sums of squares (>= +0); NaN sorts last, like lexsort
  if (!(s == s)) return ~0ull;
  return (uint64_t)__double_as_longlong(s + 0.0);  // (+0.0 folds a -0.0)
}

struct SelShared {
  unsigned int hist[256];
  unsigned long long prefix, pmask;
  int need, count;
  uint64_t skey[kSelMaxK];
  int64_t sid[kSelMaxK];
};

// k best (key, id) of N candidates into out (sorted by (key, id)); keys of
// padding entries are ~0 with id INT64_MAX.  All threads of the CTA call it.
template <typename KeyAt, typename IdAt>
__device__ void cta_select(SelShared& S, int N, int k, KeyAt key_at, IdAt id_at,
                           uint64_t* out_key, int64_t* out_id) {
  const int tid = threadIdx.x;
  const int take = min(k, N);
  // 1. radix select: the take-th smallest key t
  if (tid == 0) { S.prefix = 0; S.pmask = 0; S.need = take; }
  __syncthreads();
  for (int shift = 56; shift >= 0 && take > 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) S.hist[i] = 0;
    __syncthreads();
    const unsigned long long pre = S.prefix, pm = S.pmask;
    for (int i = tid; i < N; i += blockDim.x) {
      const uint64_t key = key_at(i);
      if ((key & pm) == pre) atomicAdd(&S.hist[(key >> shift) & 255], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int need = S.need, b = 0;
      while (b < 255 && (int)S.hist[b] < need) need -= (int)S.hist[b++];
      S.need = need;
      S.prefix = pre | ((unsigned long long)b << shift);
      S.pmask = pm | (255ull << shift);
    }
    __syncthreads();
  }
  const uint64_t t = S.prefix;
  // 2. among keys == t, the need-th smallest id u
  if (tid == 0) { S.prefix = 0; S.pmask = 0; }
  __syncthreads();
  for (int shift = 56; shift >= 0 && take > 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) S.hist[i] = 0;
    __syncthreads();
    const unsigned long long pre = S.prefix, pm = S.pmask;
    for (int i = tid; i < N; i += blockDim.x) {
      if (key_at(i) != t) continue;
      const uint64_t id = (uint64_t)id_at(i);
      if ((id & pm) == pre) atomicAdd(&S.hist[(id >> shift) & 255], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int need = S.need, b = 0;
      while (b < 255 && (int)S.hist[b] < need) need -= (int)S.hist[b++];
      S.need = need;
      S.prefix = pre | ((unsigned long long)b << shift);
      S.pmask = pm | (255ull << shift);
    }
    __syncthreads();
  }
  const uint64_t u = S.prefix;
  // 3. compact the take winners, pad to a power of two, bitonic sort
  if (tid == 0) S.count = 0;
  __syncthreads();
  for (int i = tid; i < N && take > 0; i += blockDim.x) {
    const uint64_t key = key_at(i);
    if (key < t || (key == t && (uint64_t)id_at(i) <= u)) {
      const int at = atomicAdd(&S.count, 1);
      if (at < kSelMaxK) { S.skey[at] = key; S.sid[at] = id_at(i); }
    }
  }
  __syncthreads();
  int P = 1;
  while (P < k) P <<= 1;
  for (int i = take + tid; i < P; i += blockDim.x) { S.skey[i] = ~0ull; S.sid[i] = INT64_MAX; }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < P; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = S.skey[i] > S.skey[j] || (S.skey[i] == S.skey[j] && S.sid[i] > S.sid[j]);
          if (gt == up) {
            const uint64_t tk = S.skey[i]; S.skey[i] = S.skey[j]; S.skey[j] = tk;
            const int64_t ti = S.sid[i]; S.sid[i] = S.sid[j]; S.sid[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < k; i += blockDim.x) { out_key[i] = S.skey[i]; out_id[i] = S.sid[i]; }
  __syncthreads();
}

// stage 1: (query, chunk) -> k candidates
__global__ void __launch_bounds__(kSelThreads) brute_chunk_kernel(const double* __restrict__ scores,
                                                                  int64_t n, int k, int nchunks,
                                                                  uint64_t* ck, int64_t* ci) {
  __shared__ SelShared S;
  const int c = blockIdx.x, q = blockIdx.y;
  const int64_t i0 = (int64_t)c * kSelChunk;
  const int N = (int)min((int64_t)kSelChunk, n - i0);
  const double* sc = scores + (size_t)q * n + i0;
  cta_select(S, N, k, [&](int i) { return score_key(sc[i]); }, [&](int i) { return i0 + i; },
             ck + ((size_t)q * nchunks + c) * k, ci + ((size_t)q * nchunks + c) * k);
}

// stage 2: per query, k best of the chunk candidates
__global__ void __launch_bounds__(kSelThreads) brute_final_kernel(const uint64_t* __restrict__ ck,
                                                                  const int64_t* __restrict__ ci,
                                                                  int ncand, int k, int64_t* ids,
                                                                  double* out_scores, uint64_t* tk,
                                                                  int64_t* ti) {
  __shared__ SelShared S;
  const int q = blockIdx.x;
  const uint64_t* kk = ck + (size_t)q * ncand;
  const int64_t* ii = ci + (size_t)q * ncand;
  cta_select(S, ncand, k, [&](int i) { return kk[i]; }, [&](int i) { return ii[i]; },
             tk + (size_t)q * k, ti + (size_t)q * k);
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    ids[(size_t)q * k + i] = ti[(size_t)q * k + i];
    out_scores[(size_t)q * k + i] = __longlong_as_double((long long)tk[(size_t)q * k + i]);
  }
}

}  // namespace icq

extern "C" icq_status icq_bruteforce(const float* x_dev, int64_t n, int32_t d, const double* q_dev,
                                     int32_t Q, int32_t k, int64_t* ids_dev, double* scores_dev,
                                     void* stream) {
  using namespace icq;
  if (n < 1 || d < 1) return icq_fail(ICQ_ERR_VALIDATION, "dataset must be (n >= 1, d >= 1)");
  if (!(k >= 1 && (int64_t)k <= n))
    return icq_fail(ICQ_ERR_VALIDATION, "k=%d out of range [1, %lld]", k, (long long)n);
  if (Q < 0) return icq_fail(ICQ_ERR_VALIDATION, "Q=%d < 0", Q);
  if (k > kSelMaxK) return icq_fail(ICQ_ERR_UNSUPPORTED, "k=%d > %d for the brute-force scan", k, kSelMaxK);
  if (n > 0x7fffffffLL) return icq_fail(ICQ_ERR_UNSUPPORTED, "n=%lld exceeds int32 rows", (long long)n);
  if (Q == 0) return ICQ_OK;
  LutProg prog;
  if (!make_lut_prog(d, &prog)) return icq_fail(ICQ_ERR_UNSUPPORTED, "d=%d out of range [1, 8192]", d);
  cudaStream_t s = (cudaStream_t)stream;
  const int nchunks = (int)((n + kSelChunk - 1) / kSelChunk);
  const int ncand = nchunks * k;
  // queries per group: the (group x n) float64 score block within 8 GiB
  int64_t qg = ((int64_t)8 << 30) / (n * 8);
  qg = qg < 1 ? 1 : (qg > Q ? Q : qg);
  const size_t b_sc = (size_t)qg * n * 8, b_ck = (size_t)qg * ncand * 8;
  const size_t b_tk = (size_t)qg * k * 8;
  char* buf = nullptr;
  const size_t total = b_sc + 2 * b_ck + 2 * b_tk + sizeof(LutProg) + sizeof(int32_t) + 1024;
  CUDA_TRY(cudaMallocAsync((void**)&buf, total, s));
  double* sc = reinterpret_cast<double*>(buf);
  uint64_t* ck = reinterpret_cast<uint64_t*>(buf + b_sc);
  int64_t* ci = reinterpret_cast<int64_t*>(buf + b_sc + b_ck);
  uint64_t* tk = reinterpret_cast<uint64_t*>(buf + b_sc + 2 * b_ck);
  int64_t* ti = reinterpret_cast<int64_t*>(buf + b_sc + 2 * b_ck + b_tk);
  LutProg* pd = reinterpret_cast<LutProg*>(buf + b_sc + 2 * b_ck + 2 * b_tk);
  int32_t* err = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(pd) + sizeof(LutProg));
  cudaError_t e = cudaMemcpyAsync(pd, &prog, sizeof(LutProg), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(err, 0, sizeof(int32_t), s);
  for (int q0 = 0; q0 < Q && e == cudaSuccess; q0 += (int)qg) {
    const int nq = (int)(Q - q0 < qg ? Q - q0 : qg);
    // scores[q][i] = sum_t (x[i][t] - q[t])^2: the LUT kernel with (K*m) = n rows
    e = launch_lut(x_dev, q_dev + (size_t)q0 * d, sc, 1, (int)n, d, nq, pd, err, s);
    if (e != cudaSuccess) break;
    brute_chunk_kernel<<<dim3(nchunks, nq), kSelThreads, 0, s>>>(sc, n, k, nchunks, ck, ci);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    brute_final_kernel<<<nq, kSelThreads, 0, s>>>(ck, ci, ncand, k, ids_dev + (size_t)q0 * k,
                                                   scores_dev + (size_t)q0 * k, tk, ti);
    e = cudaGetLastError();
  }
  int32_t herr = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&herr, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(buf, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return icq_fail(ICQ_ERR_CUDA, "bruteforce: %s", cudaGetErrorString(e));
  if (herr & 8) return icq_fail(ICQ_ERR_VALIDATION, "query contains non-finite values");
  return ICQ_OK;
}

// icq_encode.cu — GPU ICM encoder: encode_dataset / assign_codes.
//
// Reference: icq.train.assign_codes, /root/reference/pkg/src/icq/train.py:196-243
// (and encode_dataset :256-274), all float64:
//   greedy build-up (no starting codes):
//     res = x;  for k: dist = c_sq[k] - 2 (res @ b[k].T); code_k = argmin dist;
//                       res -= b[k][code_k]
//     recon = x - res
//   (starting codes: recon = sum_k b[k][code_k], book order, train.py:143-150)
//   up to max_sweeps sweeps, each over k = 0..K-1:
//     target = x - (recon - b[k][cur]);  dist = c_sq[k] - 2 (target @ b[k].T)
//     best = argmin dist;  improve iff dist[best] < dist[cur] (strict)
//     recon[hit] += b[k][best] - b[k][cur];  code = best
//   stop after a sweep that changes nothing.
// Rows are independent, so the database is encoded in row chunks: a row at
// a fixed point stays there, hence per-chunk stopping gives every row the
// same state as the reference's global loop.
//
// Kernel: one CTA per 64 rows computes the 64 x 256 dot-product tile
// (target . codeword) in float64 -- register-blocked 8 rows x 8 codewords per
// thread, d streamed in 16-element slabs through shared memory -- then the
// dist / first-minimum argmin epilogue and the row update, all fused.  The
// dot products are exact float64 FMA chains in d order; the reference's
// BLAS dgemm sums in its own blocked order, so codes can differ only where
// two codewords tie to ~1e-15 relative (documented near-ties, checked by the
// parity tests).  float64 is required for that parity: a tf32/bf16 tensor-
// core product would flip argmins at ordinary (1e-4 relative) gaps.
#include <cstdint>

#include "icq_index.cuh"

namespace icq {

constexpr int kEncRows = 64;     // rows per CTA
constexpr int kEncCols = 256;    // codewords per tile (m <= 256, padded)
constexpr int kEncThreads = 256;
constexpr int kEncSlab = 16;     // d elements per shared-memory slab

struct EncParams {
  const float* x;        // (rows, d) float32 chunk
  const double* books;   // (K, m, d) float64
  const double* c_sq;    // (K, m) float64 (numpy pairwise order, host-computed)
  double* res;           // (rows, d): greedy residual / sweep reconstruction
  int32_t* codes;        // (rows, K)
  int32_t* changed;      // sweep change counter
  int64_t rows;
  int32_t d, m, K, k;    // book k of this step
  int32_t sweep;         // 0 = greedy step, 1 = ICM sweep step
};

__global__ void __launch_bounds__(kEncThreads, 1) encode_step_kernel(const EncParams p) {
  __shared__ double sA[kEncRows][kEncSlab + 1];
  __shared__ double sB[kEncCols][kEncSlab + 1];
  __shared__ double s_best_d[kEncRows], s_cur_d[kEncRows];
  __shared__ int s_best[kEncRows], s_cur[kEncRows];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t r0 = (int64_t)blockIdx.x * kEncRows;
  const int d = p.d, m = p.m, K = p.K, k = p.k;
  const double* bk = p.books + (size_t)k * m * d;
  if (tid < kEncRows) {
    const int64_t r = r0 + tid;
    s_cur[tid] = (p.sweep && r < p.rows) ? p.codes[r * K + k] : 0;
  }
  __syncthreads();
  // thread tile: rows warp*8 .. +7, codewords lane + 32 u (u = 0..7)
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[a][u] = 0.0;
  for (int i0 = 0; i0 < d; i0 += kEncSlab) {
    const int w = min(kEncSlab, d - i0);
    // A slab: the row targets (greedy: res; sweep: x - (recon - b[k][cur]))
    for (int e = tid; e < kEncRows * kEncSlab; e += kEncThreads) {
      const int rr = e / kEncSlab, ii = e % kEncSlab;
      const int64_t r = r0 + rr;
      double v = 0.0;
      if (ii < w && r < p.rows) {
        const double rv = p.res[(size_t)r * d + i0 + ii];
        if (p.sweep) {
          const double xv = (double)p.x[(size_t)r * d + i0 + ii];
          v = __dsub_rn(xv, __dsub_rn(rv, bk[(size_t)s_cur[rr] * d + i0 + ii]));
        } else {
          v = rv;
        }
      }
      sA[rr][ii] = v;
    }
    for (int e = tid; e < kEncCols * kEncSlab; e += kEncThreads) {
      const int jj = e / kEncSlab, ii = e % kEncSlab;
      sB[jj][ii] = (ii < w && jj < m) ? bk[(size_t)jj * d + i0 + ii] : 0.0;
    }
    __syncthreads();
    for (int ii = 0; ii < w; ++ii) {
      double av[8], bv[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) av[a] = sA[warp * 8 + a][ii];
#pragma unroll
      for (int u = 0; u < 8; ++u) bv[u] = sB[lane + 32 * u][ii];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[a][u] = __fma_rn(av[a], bv[u], acc[a][u]);
    }
    __syncthreads();
  }
  // epilogue: dist = c_sq - 2 dot; first minimum over the codewords
  const double* cs = p.c_sq + (size_t)k * m;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int rr = warp * 8 + a;
    double bd = __longlong_as_double(0x7ff0000000000000LL);
    int bj = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = lane + 32 * u;
      if (j < m) {
        const double dist = __dsub_rn(cs[j], __dmul_rn(2.0, acc[a][u]));
        if (dist < bd || bj == 0x7fffffff) { bd = dist; bj = j; }
        if (p.sweep && j == s_cur[rr]) s_cur_d[rr] = dist;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (od < bd || (od == bd && oj < bj)) { bd = od; bj = oj; }
    }
    if (lane == 0) { s_best[rr] = bj; s_best_d[rr] = bd; }
  }
  __syncthreads();
  // row updates (one warp per row, lanes over d)
  for (int rr = warp; rr < kEncRows; rr += kEncThreads / 32) {
    const int64_t r = r0 + rr;
    if (r >= p.rows) break;
    const int best = s_best[rr];
    double* row = p.res + (size_t)r * d;
    if (!p.sweep) {  // res -= b[k][code]
      for (int i = lane; i < d; i += 32) row[i] = __dsub_rn(row[i], bk[(size_t)best * d + i]);
      if (lane == 0) p.codes[r * K + k] = best;
    } else if (s_best_d[rr] < s_cur_d[rr]) {  // strict improvement
      const int cur = s_cur[rr];
      for (int i = lane; i < d; i += 32)
        row[i] = __dadd_rn(row[i], __dsub_rn(bk[(size_t)best * d + i], bk[(size_t)cur * d + i]));
      if (lane == 0) {
        p.codes[r * K + k] = best;
        atomicAdd(p.changed, 1);
      }
    }
  }
}

// recon = x - res (greedy) elementwise
__global__ void encode_recon_kernel(const float* x, double* res, int64_t total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) res[i] = __dsub_rn((double)x[i], res[i]);
}
// recon = sum_k b[k][code_k] in book order (starting codes, train.py:143-150)
__global__ void encode_reconstruct_kernel(const double* books, const int32_t* codes, double* recon,
                                          int64_t rows, int d, int m, int K) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * d) return;
  const int64_t r = i / d;
  const int t = (int)(i - r * d);
  double s = 0.0;
  for (int k = 0; k < K; ++k) s = __dadd_rn(s, books[((size_t)k * m + codes[r * K + k]) * d + t]);
  recon[i] = s;
}
__global__ void encode_res_init_kernel(const float* x, double* res, int64_t total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) res[i] = (double)x[i];
}
__global__ void encode_codes_in_kernel(const uint8_t* in, int32_t* codes, int64_t total, int m,
                                       int32_t* err) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int c = in[i];
  if (c >= m) atomicOr(err, 2);
  codes[i] = c;
}
__global__ void encode_codes_out_kernel(const int32_t* codes, uint8_t* out, int64_t total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) out[i] = (uint8_t)codes[i];
}

}  // namespace icq

extern "C" icq_status icq_encode(const float* x_dev, int64_t n, int32_t d, const double* books_dev,
                                 const double* c_sq_dev, int32_t K, int32_t m,
                                 const uint8_t* codes_in_dev, int32_t max_sweeps,
                                 uint8_t* codes_out_dev, int32_t* sweeps_out, void* stream) {
  using namespace icq;
  if (n < 0 || d < 1 || K < 1 || m < 1) return icq_fail(ICQ_ERR_VALIDATION, "bad encoder shape");
  if (m > kEncCols) return icq_fail(ICQ_ERR_UNSUPPORTED, "m=%d > %d codewords", m, kEncCols);
  if (max_sweeps < 0) return icq_fail(ICQ_ERR_VALIDATION, "max_sweeps must be >= 0");
  if (n == 0) return ICQ_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // row chunks: the float64 residual / reconstruction block within ~4 GiB
  int64_t chunk = ((int64_t)4 << 30) / ((int64_t)d * 8);
  chunk = chunk / kEncRows * kEncRows;
  if (chunk < kEncRows) chunk = kEncRows;
  if (chunk > n) chunk = n;
  double* res = nullptr;
  int32_t* codes = nullptr;
  int32_t* counters = nullptr;  // [0] changed, [1] error
  CUDA_TRY(cudaMallocAsync((void**)&res, (size_t)chunk * d * 8, s));
  CUDA_TRY(cudaMallocAsync((void**)&codes, (size_t)chunk * K * 4, s));
  CUDA_TRY(cudaMallocAsync((void**)&counters, 8, s));
  int32_t* hbuf = nullptr;
  CUDA_TRY(cudaMallocHost((void**)&hbuf, 8));
  cudaError_t e = cudaMemsetAsync(counters, 0, 8, s);
  int32_t max_used = 0;
  for (int64_t c0 = 0; c0 < n && e == cudaSuccess; c0 += chunk) {
    const int64_t rows = n - c0 < chunk ? n - c0 : chunk;
    const float* xc = x_dev + (size_t)c0 * d;
    const int64_t tot = rows * d;
    const unsigned eb = (unsigned)((tot + 255) / 256);
    EncParams P;
    P.x = xc; P.books = books_dev; P.c_sq = c_sq_dev; P.res = res; P.codes = codes;
    P.changed = counters; P.rows = rows; P.d = d; P.m = m; P.K = K;
    const unsigned grid = (unsigned)((rows + kEncRows - 1) / kEncRows);
    if (!codes_in_dev) {
      encode_res_init_kernel<<<eb, 256, 0, s>>>(xc, res, tot);
      P.sweep = 0;
      for (int k = 0; k < K; ++k) {
        P.k = k;
        encode_step_kernel<<<grid, kEncThreads, 0, s>>>(P);
      }
      encode_recon_kernel<<<eb, 256, 0, s>>>(xc, res, tot);
    } else {
      const int64_t ct = rows * K;
      encode_codes_in_kernel<<<(unsigned)((ct + 255) / 256), 256, 0, s>>>(
          codes_in_dev + (size_t)c0 * K, codes, ct, m, counters + 1);
      encode_reconstruct_kernel<<<eb, 256, 0, s>>>(books_dev, codes, res, rows, d, m, K);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    P.sweep = 1;
    int used = 0;
    for (int sw = 0; sw < max_sweeps; ++sw) {
      if ((e = cudaMemsetAsync(counters, 0, 4, s)) != cudaSuccess) break;
      for (int k = 0; k < K; ++k) {
        P.k = k;
        encode_step_kernel<<<grid, kEncThreads, 0, s>>>(P);
      }
      if ((e = cudaMemcpyAsync(hbuf, counters, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
      ++used;
      if (hbuf[1] & 2) break;
      if (hbuf[0] == 0) break;  // a sweep that changed nothing (train.py:241-242)
    }
    if (e == cudaSuccess && (hbuf[1] & 2)) break;
    if (used > max_used) max_used = used;
    const int64_t ct = rows * K;
    encode_codes_out_kernel<<<(unsigned)((ct + 255) / 256), 256, 0, s>>>(
        codes, codes_out_dev + (size_t)c0 * K, ct);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(hbuf, counters, 8, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(res, s);
  cudaFreeAsync(codes, s);
  cudaFreeAsync(counters, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  const int32_t err = hbuf[1];
  cudaFreeHost(hbuf);
  if (e != cudaSuccess) return icq_fail(ICQ_ERR_CUDA, "encode: %s", cudaGetErrorString(e));
  if (err & 2) return icq_fail(ICQ_ERR_VALIDATION, "codes reference codewords beyond m");
  if (sweeps_out) *sweeps_out = max_used;
  return ICQ_OK;
}

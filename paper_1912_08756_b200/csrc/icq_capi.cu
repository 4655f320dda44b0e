// icq_capi.cu — extern "C" boundary (include/icq_b200.h) and index repack.
//
// Replaces the Python entry points of /root/reference/pkg/src/icq/search.py
// (build_lut :61, search_exact :97, search_two_step :112) and the argument
// layout of icq.data.SearchIndex (data.py:193-263).  Validation mirrors
// search.py:47-58, :123-131 and data.py:145-176.
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "icq_index.cuh"


using namespace icq;

static thread_local std::string g_err;

// Kernel timing instrumentation (icq_profile_enable / icq_profile_read):
// CUDA events recorded on the launch stream around each pipeline kernel.
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<cudaEvent_t> g_prof_events;  // groups of kProfEvents per batch

static inline icq_status fail_v(icq_status code, const char* fmt, va_list ap) {
  char buf[512];
  vsnprintf(buf, sizeof(buf), fmt, ap);
  g_err = buf;
  return code;
}
#define fail icq_fail

icq_status icq_fail(icq_status code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  const icq_status r = fail_v(code, fmt, ap);
  va_end(ap);
  return r;
}


static int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// --------------------------------------------------------------------------
// repack: (n, K) codes -> uint8 full rows (stride KP) + fast rows (stride FP)
// --------------------------------------------------------------------------
template <typename CodeT>
__global__ void repack_kernel(const CodeT* __restrict__ codes, int64_t row0, int64_t rows, int K,
                              int m, int KP, uint8_t* __restrict__ full, int FP, int F,
                              const FastBooks fb, uint8_t* __restrict__ fastp,
                              uint8_t* __restrict__ xfull, int32_t* err) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int64_t i = row0 + r;
  uint8_t row[kMaxK];
  bool bad = false;
  for (int b = 0; b < K; ++b) {
    const uint64_t c = (uint64_t)codes[r * K + b];
    bad |= c >= (uint64_t)m;
    row[b] = (uint8_t)c;
  }
  if (bad) atomicOr(err, 2);
  for (int b = 0; b < KP; ++b) full[i * KP + b] = b < K ? row[b] : 0;
  // streamed rows in the tile-transposed layout (icq_common.cuh perm_chunk):
  // the fast books, and all books for the exact engine
  if (fastp) {
    uint8_t* dst = fastp + perm_offset(FP, i);
    for (int s = 0; s < FP; ++s) dst[s] = s < F ? row[fb.b[s]] : 0;
  }
  uint8_t* xd = xfull + perm_offset(KP, i);
  for (int b = 0; b < KP; ++b) xd[b] = b < K ? row[b] : 0;
}

void icq_index_free(icq_index_t h) {
  if (!h) return;
  cudaFree(h->books);
  cudaFree(h->codes_full);
  cudaFree(h->codes_fast);
  cudaFree(h->codes_xfull);
  cudaFree(h->prog_dev);
  cudaFree(h->err_dev);
  cudaFree(h->host_buf);
  delete h;
}

icq_status icq_index_alloc(const float* books, bool books_on_device, int32_t K, int32_t m,
                           int32_t d, int64_t n, const uint32_t* fast, int32_t F,
                           cudaStream_t stream, icq_index_t* out) {
  if (!out) return fail(ICQ_ERR_VALIDATION, "out handle pointer is NULL");
  *out = nullptr;
  if (K < 1) return fail(ICQ_ERR_VALIDATION, "K must be >= 1, got %d", K);
  if (m < 2) return fail(ICQ_ERR_VALIDATION, "m must be >= 2, got %d", m);
  if (d < 1) return fail(ICQ_ERR_VALIDATION, "d must be >= 1, got %d", d);
  if (n < 1) return fail(ICQ_ERR_VALIDATION, "index must hold at least one element");
  if (K > kMaxK) return fail(ICQ_ERR_UNSUPPORTED, "K=%d > %d books is not supported", K, kMaxK);
  if (m > 256) return fail(ICQ_ERR_UNSUPPORTED, "m=%d > 256 codewords (uint8 codes)", m);
  if (n > 0x7fffffffLL) return fail(ICQ_ERR_UNSUPPORTED, "n=%lld exceeds int32 ids", (long long)n);
  if (F < 0 || F > K) return fail(ICQ_ERR_VALIDATION, "fast set must hold codebook indices in [0, K)");
  for (int s = 0; s < F; ++s) {
    if (fast[s] >= (uint32_t)K)
      return fail(ICQ_ERR_VALIDATION, "fast set must hold codebook indices in [0, K)");
    if (s && fast[s] <= fast[s - 1])
      return fail(ICQ_ERR_VALIDATION, "fast set must be sorted and unique");
  }
  LutProg prog;
  if (!make_lut_prog(d, &prog)) return fail(ICQ_ERR_UNSUPPORTED, "d=%d out of range [1, 8192]", d);

  auto* h = new icq_index_s();
  h->K = K; h->m = m; h->d = d; h->F = F; h->n = n;
  h->KP = pow2_ceil(K);
  h->FP = F ? pow2_ceil(F) : 0;
  h->n_pad = (n + kRangeAlign - 1) / kRangeAlign * kRangeAlign;
  memset(h->fast_books, 0, sizeof(h->fast_books));
  memset(&h->fb, 0, sizeof(h->fb));
  for (int s = 0; s < F; ++s) {
    h->fast_books[s] = (uint8_t)fast[s];
    h->fb.b[s] = (uint8_t)fast[s];
  }
  const size_t bbytes = (size_t)K * m * d * sizeof(float);
  const size_t fullb = (size_t)h->n_pad * h->KP;
  const size_t fastb = F ? (size_t)h->n_pad * h->FP : 0;
  cudaError_t e;
  if ((e = cudaMalloc(&h->books, bbytes)) != cudaSuccess ||
      (e = cudaMalloc(&h->codes_full, fullb)) != cudaSuccess ||
      (fastb && (e = cudaMalloc(&h->codes_fast, fastb)) != cudaSuccess) ||
      (e = cudaMalloc(&h->codes_xfull, fullb)) != cudaSuccess ||
      (e = cudaMalloc(&h->prog_dev, sizeof(LutProg))) != cudaSuccess ||
      (e = cudaMalloc(&h->err_dev, sizeof(int32_t))) != cudaSuccess) {
    icq_index_free(h);
    return fail(ICQ_ERR_NOMEM, "device allocation failed: %s", cudaGetErrorString(e));
  }
  h->bytes = (int64_t)(bbytes + 2 * fullb + fastb);
  const cudaMemcpyKind kind = books_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if ((e = cudaMemcpyAsync(h->books, books, bbytes, kind, stream)) != cudaSuccess ||
      (e = cudaMemcpyAsync(h->prog_dev, &prog, sizeof(LutProg), cudaMemcpyHostToDevice, stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(h->err_dev, 0, sizeof(int32_t), stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(h->codes_full, 0, fullb, stream)) != cudaSuccess ||
      (fastb && (e = cudaMemsetAsync(h->codes_fast, 0, fastb, stream)) != cudaSuccess) ||
      (e = cudaMemsetAsync(h->codes_xfull, 0, fullb, stream)) != cudaSuccess ||
      (e = cudaStreamSynchronize(stream)) != cudaSuccess) {  // (books may be a transient host buffer)
    icq_index_free(h);
    return fail(ICQ_ERR_CUDA, "index upload failed: %s", cudaGetErrorString(e));
  }
  *out = h;
  return ICQ_OK;
}

cudaError_t icq_index_repack_rows(icq_index_t h, const void* codes_dev, int code_bytes,
                                  int64_t row0, int64_t rows, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const int threads = 256;
  const unsigned blocks = (unsigned)((rows + threads - 1) / threads);
  if (code_bytes == 4)
    repack_kernel<uint32_t><<<blocks, threads, 0, s>>>(
        static_cast<const uint32_t*>(codes_dev), row0, rows, h->K, h->m, h->KP, h->codes_full,
        h->FP, h->F, h->fb, h->F ? h->codes_fast : nullptr, h->codes_xfull, h->err_dev);
  else
    repack_kernel<uint8_t><<<blocks, threads, 0, s>>>(
        static_cast<const uint8_t*>(codes_dev), row0, rows, h->K, h->m, h->KP, h->codes_full,
        h->FP, h->F, h->fb, h->F ? h->codes_fast : nullptr, h->codes_xfull, h->err_dev);
  return cudaGetLastError();
}

// 0 = ok, else the error word (bit 1: a code >= m)
int32_t icq_index_repack_errors(icq_index_t h) {
  int32_t err = 0;
  if (cudaMemcpy(&err, h->err_dev, sizeof(err), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return err;
}

template <typename CodeT>
static icq_status create_impl(const float* books, int32_t K, int32_t m, int32_t d,
                              const CodeT* codes, int64_t n, const uint32_t* fast, int32_t F,
                              bool on_device, cudaStream_t stream, icq_index_t* out) {
  icq_index_t h = nullptr;
  icq_status st = icq_index_alloc(books, on_device, K, m, d, n, fast, F, stream, &h);
  if (st != ICQ_OK) return st;
  const CodeT* codes_dev = codes;
  CodeT* staged = nullptr;
  cudaError_t e = cudaSuccess;
  if (!on_device) {
    const size_t cb = (size_t)n * K * sizeof(CodeT);
    if ((e = cudaMalloc(&staged, cb)) == cudaSuccess)
      e = cudaMemcpyAsync(staged, codes, cb, cudaMemcpyHostToDevice, stream);
    codes_dev = staged;
  }
  if (e == cudaSuccess) e = icq_index_repack_rows(h, codes_dev, (int)sizeof(CodeT), 0, n, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (staged) cudaFree(staged);
  if (e != cudaSuccess) {
    icq_index_free(h);
    return fail(ICQ_ERR_CUDA, "index upload/repack failed: %s", cudaGetErrorString(e));
  }
  if (icq_index_repack_errors(h) & 2) {
    icq_index_free(h);
    return fail(ICQ_ERR_VALIDATION, "codes reference codewords beyond m");
  }
  *out = h;
  g_err.clear();
  return ICQ_OK;
}

extern "C" {

const char* icq_last_error(void) { return g_err.c_str(); }

icq_status icq_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
  return ICQ_OK;
}

icq_status icq_profile_read(double* ms_out, int32_t* launches) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  double acc[5] = {0, 0, 0, 0, 0};  // prologue, filter, replay, count, refine
  const int groups = (int)(g_prof_events.size() / kProfEvents);
  for (int i = 0; i < groups; ++i) {
    cudaEvent_t* e = &g_prof_events[kProfEvents * i];
    if (cudaEventSynchronize(e[kProfEvents - 1]) != cudaSuccess)
      return fail(ICQ_ERR_CUDA, "profile: event synchronize failed");
    for (int j = 0; j + 1 < kProfEvents; ++j) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e[j], e[j + 1]);
      // interval j: 0 prologue; 1 + 3r filter, 2 + 3r refine, 3 + 3r replay; last count
      static const int kind3[3] = {1, 4, 2};
      acc[j == 0 ? 0 : (j == kProfEvents - 2 ? 3 : kind3[(j - 1) % 3])] += ms;
    }
  }
  for (cudaEvent_t e : g_prof_events) cudaEventDestroy(e);
  g_prof_events.clear();
  if (ms_out) for (int j = 0; j < 5; ++j) ms_out[j] = acc[j];
  if (launches) *launches = groups;
  return ICQ_OK;
}

int32_t icq_abi_version(void) { return 3; }

int64_t icq_kernel_launches(void) { return (int64_t)icq::kernel_launches(); }

icq_status icq_index_create(const float* books, int32_t K, int32_t m, int32_t d,
                            const uint32_t* codes, int64_t n, const uint32_t* fast, int32_t F,
                            icq_index_t* out) {
  return create_impl<uint32_t>(books, K, m, d, codes, n, fast, F, false, 0, out);
}

icq_status icq_index_create_u8(const float* books, int32_t K, int32_t m, int32_t d,
                               const uint8_t* codes, int64_t n, const uint32_t* fast, int32_t F,
                               icq_index_t* out) {
  return create_impl<uint8_t>(books, K, m, d, codes, n, fast, F, false, 0, out);
}

icq_status icq_index_create_device(const float* books, int32_t K, int32_t m, int32_t d,
                                   const uint8_t* codes, int64_t n, const uint32_t* fast,
                                   int32_t F, void* stream, icq_index_t* out) {
  return create_impl<uint8_t>(books, K, m, d, codes, n, fast, F, true, (cudaStream_t)stream, out);
}

icq_status icq_index_destroy(icq_index_t h) {
  icq_index_free(h);
  return ICQ_OK;
}

icq_status icq_index_read_codes(icq_index_t h, int64_t row0, int64_t rows, uint8_t* codes_host) {
  if (!h) return fail(ICQ_ERR_VALIDATION, "null index handle");
  if (row0 < 0 || rows < 0 || row0 + rows > h->n)
    return fail(ICQ_ERR_VALIDATION, "rows [%lld, %lld) outside [0, %lld)", (long long)row0,
                (long long)(row0 + rows), (long long)h->n);
  if (rows == 0) return ICQ_OK;
  // codes_full rows are KP wide: copy the K leading bytes of each row
  CUDA_TRY(cudaMemcpy2D(codes_host, (size_t)h->K, h->codes_full + row0 * h->KP, (size_t)h->KP,
                        (size_t)h->K, (size_t)rows, cudaMemcpyDeviceToHost));
  return ICQ_OK;
}

icq_status icq_index_info(icq_index_t h, int64_t* n, int32_t* K, int32_t* m, int32_t* d,
                          int32_t* F, int64_t* device_bytes) {
  if (!h) return fail(ICQ_ERR_VALIDATION, "null index handle");
  if (n) *n = h->n;
  if (K) *K = h->K;
  if (m) *m = h->m;
  if (d) *d = h->d;
  if (F) *F = h->F;
  if (device_bytes) *device_bytes = h->bytes;
  return ICQ_OK;
}

// Device error word of one call: bit 0 filter shared-memory layout, bit 2
// replay chunk descriptors dropped, bit 3 a query holds non-finite values.
static icq_status check_call_errors(int32_t err) {
  if (err & 8) return fail(ICQ_ERR_VALIDATION, "query contains non-finite values");
  if (err & 1) return fail(ICQ_ERR_CUDA, "filter kernel shared-memory layout check failed");
  if (err & 4) return fail(ICQ_ERR_CUDA, "replay dropped candidate chunks");
  if (err & 16) return fail(ICQ_ERR_CUDA, "count mode: more than %d insertions after the prologue", kMaxTraj);
  if (err) return fail(ICQ_ERR_CUDA, "device error word 0x%x", err);
  return ICQ_OK;
}

// one int32 of pinned host memory per thread: the error word's landing slot
static int32_t* host_err_slot() {
  static thread_local int32_t* slot = nullptr;
  if (!slot && cudaMallocHost((void**)&slot, sizeof(int32_t)) != cudaSuccess) slot = nullptr;
  return slot;
}

icq_status icq_build_lut(icq_index_t h, const double* q, int32_t Q, double* lut, void* stream) {
  if (!h) return fail(ICQ_ERR_VALIDATION, "null index handle");
  if (Q < 0) return fail(ICQ_ERR_VALIDATION, "Q=%d < 0", Q);
  if (Q == 0) return ICQ_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* err = nullptr;
  int32_t* herr = host_err_slot();
  if (!herr) return fail(ICQ_ERR_NOMEM, "pinned error slot allocation failed");
  CUDA_TRY(cudaMallocAsync((void**)&err, sizeof(int32_t), s));
  cudaError_t e = cudaMemsetAsync(err, 0, sizeof(int32_t), s);
  if (e == cudaSuccess) e = launch_lut(h->books, q, lut, h->K, h->m, h->d, Q, h->prog_dev, err, s);
  count_kernel_launches(1);
  if (e == cudaSuccess) e = cudaMemcpyAsync(herr, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(err, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(ICQ_ERR_CUDA, "build_lut: %s", cudaGetErrorString(e));
  return check_call_errors(*herr);
}

icq_status icq_workspace_size(icq_index_t h, int32_t Q, int32_t k, size_t* bytes) {
  if (!h || !bytes) return fail(ICQ_ERR_VALIDATION, "null argument");
  (void)k;
  *bytes = (size_t)(Q > 0 ? Q : 0) * h->K * h->m * sizeof(double) + 256;
  return ICQ_OK;
}

static icq_status search_impl(icq_index_t h, const double* q, const double* lut_in, int32_t Q,
                              int32_t k, double sigma, int32_t flags, int64_t* ids, double* scores,
                              int64_t* refine, uint32_t* survivors, int64_t* stats,
                              int32_t* fallback_out, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (!h) return fail(ICQ_ERR_VALIDATION, "null index handle");
  bool exact = (flags & ICQ_FLAG_EXACT) != 0;
  if (!(k >= 1 && (int64_t)k <= h->n))
    return fail(ICQ_ERR_VALIDATION, "k=%d out of range [1, %lld]", k, (long long)h->n);
  if (!exact && !(sigma >= 0)) return fail(ICQ_ERR_VALIDATION, "sigma must be >= 0, got %g", sigma);
  if (!exact && (flags & ICQ_FLAG_SIGMA_F32) && (double)(float)sigma != sigma)
    return fail(ICQ_ERR_VALIDATION, "ICQ_FLAG_SIGMA_F32 with a sigma that is not a float32 value");
  if (Q < 0) return fail(ICQ_ERR_VALIDATION, "Q=%d < 0", Q);
  const bool fallback = !exact && h->F == 0;  // search.py:127-131
  if (fallback_out) *fallback_out = fallback ? 1 : 0;
  if (fallback) exact = true;
  if (Q == 0) return ICQ_OK;
  int32_t* herr = host_err_slot();
  if (!herr) return fail(ICQ_ERR_NOMEM, "pinned error slot allocation failed");
  const double* lut = lut_in;
  if (!lut) {
    size_t need = 0;
    icq_workspace_size(h, Q, k, &need);
    if (!ws || ws_bytes < need)
      return fail(ICQ_ERR_NOMEM, "workspace too small: %zu < %zu bytes", ws_bytes, need);
  }
  if (survivors) {
    const int64_t words = (h->n + 31) / 32;
    CUDA_TRY(cudaMemsetAsync(survivors, 0, (size_t)Q * words * sizeof(uint32_t), s));
  }
  PipeParams p;
  memset(&p, 0, sizeof(p));
  p.codes_full = h->codes_full;
  p.n = h->n;
  p.words = (h->n + 31) / 32;
  p.K = h->K;
  p.m = h->m;
  p.KP = h->KP;
  p.k = k;
  p.exact_mode = exact ? 1 : 0;
  int FP;
  if (exact) {
    p.codes_fast = h->codes_xfull;
    p.F = h->K;
    FP = h->KP;
    for (int b = 0; b < h->K; ++b) p.fast_books[b] = (uint8_t)b;
    p.sigma = 0.0;
  } else {
    p.codes_fast = h->codes_fast;
    p.F = h->F;
    FP = h->FP;
    memcpy(p.fast_books, h->fast_books, sizeof(p.fast_books));
    p.sigma = sigma;
    p.sigma_f32 = (flags & ICQ_FLAG_SIGMA_F32) ? 1 : 0;
  }
  // ---- plan: sub-batches, ranges, unit order, candidate pool -------------
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  auto env_i = [](const char* name, int64_t dflt) {
    const char* v = getenv(name);
    return v ? (int64_t)atoll(v) : dflt;
  };
  // queries per sub-batch: as many as the per-batch scratch allows (fewer,
  // longer prologue / replay launches: c2, 10k queries: 211k -> 256k q/s in one
  // sub-batch instead of five); bounded below by the slice-table budget
  const int Qmax = (int)env_i("ICQ_QBATCH", 16384);
  int Qb = Q < Qmax ? Q : Qmax;
  const bool big = (int64_t)h->n * FP > (int64_t)48 << 20;  // fast stream larger than ~L2/2
  p.range_major = (int32_t)env_i("ICQ_RANGE_MAJOR", big ? 1 : 0);
  {
    const int64_t units = 8LL * sms;
    int64_t nr = (units + Qb - 1) / Qb;
    if (nr < 1) nr = 1;
    int64_t rs = (h->n + nr - 1) / nr;
    // slices (RS / 16 items) small enough that a loose threshold rarely
    // overflows a slice's kMaxPages * kPG candidates
    int64_t cap = h->n / 16;
    if (cap < ((int64_t)1 << 18)) cap = (int64_t)1 << 18;
    // (streams larger than L2: 1M-item ranges keep a range's fast codes and
    // candidate rows L2-resident while every query of the batch sweeps it, and
    // a 64k-item slice holds up to 25 % of its items as candidates)
    if (big) cap = (int64_t)1 << 20;
    if (rs > cap) rs = cap;
    rs = env_i("ICQ_RANGE_ITEMS", rs);
    rs = (rs + kRangeAlign - 1) / kRangeAlign * kRangeAlign;
    p.RS = rs;
    p.NR = (int32_t)((h->n + rs - 1) / rs);
    if (!getenv("ICQ_QBATCH")) {  // slice rows: <= 4 GiB per sub-batch
      const int64_t per_q = (int64_t)p.NR * kFW * kSliceInts * (int64_t)sizeof(int32_t);
      int64_t qb = ((int64_t)4 << 30) / per_q;
      qb = qb < 256 ? 256 : qb;
      if (Qb > qb) Qb = (int)qb;
    }
    // the count kernel sweeps 2 filter ranges at a time when the stream is
    // larger than L2 (measured on c5: 1 -> 22.5, 2 -> 21.5, 4 -> 22.3, 8 -> 24.1 ms)
    // refine / gather CTAs (one warp per slice of a range) can take a group of
    // ranges each, staging their tables once per CTA; measured no gain on c4
    // and a loss on c5 (fewer warps with row reads in flight): one range each
    {
      p.RG = (int32_t)env_i("ICQ_RANGE_GROUP", 1);
      if (p.RG < 1) p.RG = 1;
      p.NRG = (p.NR + p.RG - 1) / p.RG;
    }
    const int64_t mult = env_i("ICQ_COUNT_RANGES", big ? 2 : 1);
    p.RSC = rs * (mult < 1 ? 1 : mult);
    p.NRC = (int32_t)((h->n + p.RSC - 1) / p.RSC);
  }
  p.pro_div = (int32_t)env_i("ICQ_PRO_DIV", 512);
  p.debug = (int32_t)env_i("ICQ_DEBUG", 0);  // experiments only; results stay exact
  // list threshold theta = A_J + sigma (J = 0: the live threshold at the
  // prologue end; deeper J: looser lists, fewer in-order walks); by default
  // the prologue picks the loosest J whose list share stays <= 1/list_div
  p.list_j = (int32_t)env_i("ICQ_LIST_J", -1);
  // (list length ~ n / list_div: small databases take looser lists -- fewer
  // walks; c1 +14 %, c2 +4 % at 1/32 -- large ones tighter: c5 at sigma = 0
  // loses 36 % at 1/32)
  {
    int64_t ld = h->n / 500000;
    ld = ld < 32 ? 32 : (ld > 128 ? 128 : ld);
    p.list_div = (int32_t)env_i("ICQ_LIST_DIV", ld);
  }
  p.pro_live = (int32_t)env_i("ICQ_PRO_LIVE", 0);
  // count mode (refinement-heavy queries: the live threshold passes > 1/count_div
  // of the sampled items): lists of possible insertions + a parallel count
  p.count_div = exact ? 0 : (int32_t)env_i("ICQ_COUNT_DIV", 256);
  p.force_count = exact ? 0 : (int32_t)env_i("ICQ_COUNT_MODE", 0);
  // ... and only when those lists would be long: a replay CTA decides short
  // lists faster than the count pass streams the database once more
  p.count_min = env_i("ICQ_COUNT_MIN", (int64_t)1 << 18);
  p.count_used = (FP <= 8 && (p.count_div > 0 || p.force_count)) ? 1 : 0;
  {
    const int64_t r = env_i("ICQ_ROUNDS", kMaxRounds);
    p.rounds = (int32_t)(r < 1 ? 1 : (r > kMaxRounds ? kMaxRounds : r));
    // one replay CTA walks ~1 item per clock; a filter round lists a query's
    // rest on every SM in microseconds: hand over after max(128k, n/512) items
    int64_t wc = h->n / 512;
    if (wc < ((int64_t)1 << 17)) wc = (int64_t)1 << 17;
    p.walk_cap = env_i("ICQ_WALK_CAP", wc);
  }
  p.pro_min = env_i("ICQ_PRO_MIN", 8192);
  {
    // prologue length cap: queries whose stale threshold stays loose are
    // better handed to the filter early (the stop rule ends most queries
    // well before)
    // (small databases: at most n / 8, the filter and the lists take the rest
    // -- c1, 100k items: 16k instead of 64k prologue items, 645k -> 790k q/s)
    int64_t pm = h->n / 384;
    int64_t floor_ = h->n / 8;
    floor_ = floor_ < ((int64_t)1 << 14) ? (int64_t)1 << 14 : (floor_ > ((int64_t)1 << 16) ? (int64_t)1 << 16 : floor_);
    if (pm < floor_) pm = floor_;
    p.pro_max = env_i("ICQ_PRO_MAX", pm);
    // refinement-heavy queries continue in count style (float32 exact
    // pre-filter, ~1 cycle per item): longer, for a tighter T at the hand-over
    // (off by default: the same prefix is listed by a first filter round on
    // every SM instead, cm_prefix below)
    p.pro_max_cm = p.count_used ? env_i("ICQ_PRO_MAX_CM", 0) : 0;
    p.cm_prefix = p.count_used ? env_i("ICQ_CM_PREFIX", h->n / 128) : 0;
    {
      const int64_t pe = p.cm_prefix < h->n ? p.cm_prefix : h->n;
      p.NRD = (p.cm_prefix > 0 && p.rounds >= 2) ? (int32_t)((pe + p.RS - 1) / p.RS) : 0;
    }
  }
  {
    // candidate pool: a shared bump allocator of 128-entry pages; when it runs
    // dry every slice still growing overflows into a walk of its items, so it
    // is sized generously -- HBM is plentiful, the pool is never cleared
    // (only its top counter)
    int64_t entries = (int64_t)Qb * h->n / 8;
    const int64_t lo = (int64_t)1 << 20;
    int64_t hi_ = (int64_t)1 << 31;  // <= 32 GiB, and <= 1/5 of the device's memory
    {
      static int64_t total_mem[64];  // (per device, queried once)
      int dev = 0;
      if (cudaGetDevice(&dev) == cudaSuccess && dev >= 0 && dev < 64) {
        if (total_mem[dev] == 0) {
          size_t fr = 0, tot = 0;
          total_mem[dev] = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? (int64_t)tot : -1;
        }
        if (total_mem[dev] > 0) {
          const int64_t by_mem = total_mem[dev] / 5 / (int64_t)sizeof(uint4);
          if (by_mem < hi_) hi_ = by_mem;
        }
      }
    }
    entries = entries < lo ? lo : (entries > hi_ ? hi_ : entries);
    p.pool_pages = env_i("ICQ_POOL_PAGES", (entries + kPG - 1) / kPG);
  }
  {
    const int64_t mp = env_i("ICQ_MAX_PAGES", kListPages);
    p.max_pages = (int32_t)(mp < 1 ? 1 : (mp > kListPages ? kListPages : mp));
    const int64_t mc = env_i("ICQ_MAX_PAGES_CM", kMaxPages);
    p.max_pages_cm = (int32_t)(mc < 1 ? 1 : (mc > kMaxPages ? kMaxPages : mc));
  }
  const int filter_ctas = (int)env_i("ICQ_FILTER_CTAS", sms);
  // ---- stream-ordered scratch (pool cached across calls) -----------------
  static std::once_flag pool_once;
  std::call_once(pool_once, [] {
    int dev = 0;
    cudaMemPool_t mp;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t b_lut = lut ? 0 : al((size_t)Q * h->K * h->m * sizeof(double));
  const size_t b_qs = al(sizeof(QState) * Qb);
  const size_t b_he = al((size_t)Qb * k * 8), b_hi = al((size_t)Qb * k * 4);
  const size_t b_pool = al((size_t)p.pool_pages * kPG * sizeof(uint4));
  const size_t b_top = 256;  // pool_top, error word
  const size_t b_sl = al((size_t)Qb * p.NR * kFW * kSliceInts * sizeof(int32_t));
  const size_t b_tr = p.count_used ? al((size_t)Qb * kMaxTraj * sizeof(TrajEntry)) : 0;
  const size_t b_cm = al(sizeof(int32_t) * (1 + (size_t)Qb));
  // count-mode lists after the refine kernel, contiguous per query (a query
  // that does not fit is decided from its slices instead)
  {
    int64_t c = (int64_t)Qb << 19;
    const int64_t lo = (int64_t)1 << 20, hi_ = (int64_t)1 << 28;
    c = c < lo ? lo : (c > hi_ ? hi_ : c);
    p.cl_cap = env_i("ICQ_CL_CAP", c);
    p.cl_enable = (int32_t)env_i("ICQ_CL", 1);
  }
  const size_t b_cle = al((size_t)p.cl_cap * sizeof(uint4)), b_clx = al((size_t)p.cl_cap * sizeof(double));
  const size_t scratch =
      b_qs + 2 * b_he + b_hi + b_pool + b_top + b_sl + b_tr + b_cm + b_cle + b_clx;
  char* sc = nullptr;
  const bool trace = (p.debug & 32) != 0;  // host-side timing of this call (stderr)
  const auto tr0 = std::chrono::steady_clock::now();
  auto tr_ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr0).count();
  };
  CUDA_TRY(cudaMallocAsync((void**)&sc, scratch, s));
  const double tr_alloc = tr_ms();
  {
    char* o = sc;
    p.qs = reinterpret_cast<QState*>(o); o += b_qs;
    p.heap_e = reinterpret_cast<double*>(o); o += b_he;
    p.heap_f = reinterpret_cast<double*>(o); o += b_he;
    p.heap_i = reinterpret_cast<int32_t*>(o); o += b_hi;
    p.pool = reinterpret_cast<uint4*>(o); o += b_pool;
    p.pool_top = reinterpret_cast<int32_t*>(o);
    p.error = p.pool_top + 1;
    o += b_top;
    p.slices = reinterpret_cast<int32_t*>(o); o += b_sl;
    p.traj = b_tr ? reinterpret_cast<TrajEntry*>(o) : nullptr;
    o += b_tr;
    p.cm_list = reinterpret_cast<int32_t*>(o);
    o += b_cm;
    p.cl_ent = reinterpret_cast<uint4*>(o); o += b_cle;
    p.cl_ex = reinterpret_cast<double*>(o);
    p.cl_top = reinterpret_cast<unsigned long long*>(p.pool_top + 2);  // (b_top: 256 bytes)
    p.round_cnt = p.pool_top + 4;
  }
  (void)b_lut;
  icq_status st = ICQ_OK;
  cudaError_t e = cudaMemsetAsync(p.error, 0, sizeof(int32_t), s);
  if (e == cudaSuccess && !lut) {  // K1: the float64 LUTs of every query into the workspace
    double* w = reinterpret_cast<double*>(ws);
    e = launch_lut(h->books, q, w, h->K, h->m, h->d, Q, h->prog_dev, p.error, s);
    count_kernel_launches(1);
    lut = w;
  }
  if (e != cudaSuccess) st = fail(ICQ_ERR_CUDA, "search setup: %s", cudaGetErrorString(e));
  for (int q0 = 0; q0 < Q && st == ICQ_OK; q0 += Qb) {
    const int nq = Q - q0 < Qb ? Q - q0 : Qb;
    PipeParams b = p;
    b.Q = nq;
    b.lut64 = lut + (size_t)q0 * h->K * h->m;
    b.ids = ids + (size_t)q0 * k;
    b.scores = scores + (size_t)q0 * k;
    b.refinements = refine ? refine + q0 : nullptr;
    b.survivors = (!exact && survivors) ? survivors + (size_t)q0 * p.words : nullptr;
    b.stats = stats ? stats + (size_t)q0 * kStats : nullptr;
    e = cudaMemsetAsync(p.pool_top, 0, sizeof(int32_t), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p.cm_list, 0, sizeof(int32_t), s);
    if (e == cudaSuccess)  // cl_top and the per-round hand-over counters
      e = cudaMemsetAsync(p.cl_top, 0, sizeof(unsigned long long) + sizeof(int32_t) * (kMaxRounds + 1), s);
    int unsupported = 0;
    cudaEvent_t* ev = nullptr;
    cudaEvent_t evs[kProfEvents];
    {
      std::lock_guard<std::mutex> g(g_prof_mu);
      if (g_prof_on) {
        for (int j = 0; j < kProfEvents; ++j) {
          cudaEventCreate(&evs[j]);
          g_prof_events.push_back(evs[j]);
        }
        ev = evs;
      }
    }
    if (e == cudaSuccess) e = launch_pipeline(b, FP, filter_ctas, s, &unsupported, ev);
    if (e != cudaSuccess) st = fail(ICQ_ERR_CUDA, "search launch: %s", cudaGetErrorString(e));
    else if (unsupported)
      st = fail(ICQ_ERR_UNSUPPORTED, "k=%d does not fit the on-chip heap for K=%d, m=%d", k,
                h->K, h->m);
  }
  // every entry point reports the device error word of its own call
  if (st == ICQ_OK) {
    e = cudaMemcpyAsync(herr, p.error, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) st = fail(ICQ_ERR_CUDA, "search: %s", cudaGetErrorString(e));
  }
  const double tr_launch = tr_ms();
  cudaFreeAsync(sc, s);
  const double tr_free = tr_ms();
  if (st != ICQ_OK) return st;
  CUDA_TRY(cudaStreamSynchronize(s));
  if (trace)
    fprintf(stderr, "[icq trace] scratch %.1f MiB: alloc %.3f ms, launches done %.3f, free %.3f, sync %.3f\n",
            scratch / 1048576.0, tr_alloc, tr_launch, tr_free, tr_ms());
  return check_call_errors(*herr);
}

icq_status icq_search_two_step(icq_index_t h, const double* q, int32_t Q, int32_t k, double sigma,
                               int64_t* ids, double* scores, int64_t* refine, uint32_t* survivors,
                               int64_t* stats, int32_t* fallback_out, void* ws, size_t ws_bytes,
                               void* stream) {
  return search_impl(h, q, nullptr, Q, k, sigma, 0, ids, scores, refine, survivors, stats,
                     fallback_out, ws, ws_bytes, (cudaStream_t)stream);
}

icq_status icq_search_exact(icq_index_t h, const double* q, int32_t Q, int32_t k, int64_t* ids,
                            double* scores, void* ws, size_t ws_bytes, void* stream) {
  return search_impl(h, q, nullptr, Q, k, 0.0, ICQ_FLAG_EXACT, ids, scores, nullptr, nullptr,
                     nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

icq_status icq_search_with_lut(icq_index_t h, const double* lut_dev, int32_t Q, int32_t k,
                               double sigma, int32_t flags, int64_t* ids_dev, double* scores_dev,
                               int64_t* refine_dev, uint32_t* survivors_dev, int64_t* stats_dev,
                               int32_t* fallback_out, void* stream) {
  if (!lut_dev) return fail(ICQ_ERR_VALIDATION, "lut_dev is NULL");
  return search_impl(h, nullptr, lut_dev, Q, k, sigma, flags, ids_dev, scores_dev, refine_dev,
                     survivors_dev, stats_dev, fallback_out, nullptr, 0, (cudaStream_t)stream);
}

icq_status icq_search_host(icq_index_t h, const double* q_host, int32_t Q, int32_t k,
                           double sigma, int32_t flags, int64_t* ids_host, double* scores_host,
                           int64_t* refine_host, int32_t* fallback_out) {
  if (!h) return fail(ICQ_ERR_VALIDATION, "null index handle");
  if (Q < 0) return fail(ICQ_ERR_VALIDATION, "Q=%d < 0", Q);
  const bool exact = (flags & ICQ_FLAG_EXACT) != 0;
  if (!(k >= 1 && (int64_t)k <= h->n))
    return fail(ICQ_ERR_VALIDATION, "k=%d out of range [1, %lld]", k, (long long)h->n);
  if (!exact && !(sigma >= 0)) return fail(ICQ_ERR_VALIDATION, "sigma must be >= 0, got %g", sigma);
  if (fallback_out) *fallback_out = (!exact && h->F == 0) ? 1 : 0;
  if (Q == 0) return ICQ_OK;
  for (int64_t i = 0; i < (int64_t)Q * h->d; ++i)  // search.py:51-52, before any device work
    if (!std::isfinite(q_host[i])) return fail(ICQ_ERR_VALIDATION, "query contains non-finite values");
  cudaStream_t s = cudaStreamPerThread;
  size_t ws_bytes = 0;
  icq_workspace_size(h, Q, k, &ws_bytes);
  const size_t qb = (size_t)Q * h->d * sizeof(double);
  const size_t ib = (size_t)Q * k * sizeof(int64_t);
  const size_t sb = (size_t)Q * k * sizeof(double);
  const size_t rb = (size_t)Q * sizeof(int64_t);
  const size_t total = ws_bytes + qb + ib + sb + rb + 4 * 256;
  std::lock_guard<std::mutex> guard(h->host_mu);
  if (h->host_buf_bytes < total) {
    cudaFree(h->host_buf);
    h->host_buf = nullptr;
    h->host_buf_bytes = 0;
    CUDA_TRY(cudaMalloc((void**)&h->host_buf, total));
    h->host_buf_bytes = total;
  }
  char* buf = h->host_buf;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  char* ws = buf;
  double* qd = reinterpret_cast<double*>(buf + al(ws_bytes));
  int64_t* idd = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(qd) + al(qb));
  double* scd = reinterpret_cast<double*>(reinterpret_cast<char*>(idd) + al(ib));
  int64_t* rfd = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(scd) + al(sb));
  CUDA_TRY(cudaMemcpyAsync(qd, q_host, qb, cudaMemcpyHostToDevice, s));
  const icq_status st =
      search_impl(h, qd, nullptr, Q, k, sigma, flags, idd, scd, rfd, nullptr, nullptr, nullptr, ws,
                  ws_bytes, s);  // (synchronises and checks the call's error word)
  if (st != ICQ_OK) return st;
  cudaError_t e = cudaMemcpyAsync(ids_host, idd, ib, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(scores_host, scd, sb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && refine_host)
    e = cudaMemcpyAsync(refine_host, rfd, rb, cudaMemcpyDeviceToHost, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(ICQ_ERR_CUDA, "search: %s", cudaGetErrorString(e));
  if (e2 != cudaSuccess) return fail(ICQ_ERR_CUDA, "search: %s", cudaGetErrorString(e2));
  return ICQ_OK;
}

}  // extern "C"

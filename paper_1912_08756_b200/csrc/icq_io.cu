// icq_io.cu — ICQI index files straight into device memory.
//
// Reference: icq.data.load_index, /root/reference/pkg/src/icq/data.py:348-394
// (format written by save_index, data.py:306-322).  The reference reads the
// whole file into memory and copies the (n, K) uint32 code block out of it
// (3.2 GB at n = 100M, K = 8).  Here the header and tail are parsed and
// validated first (the reference's FormatError / UnsupportedVersionError
// conditions, data.py:355-394, plus Config.__post_init__ :102-122 and
// SearchIndex.__post_init__ :213-263), then the code block is streamed in
// chunks through two pinned host buffers: while the CPU reads chunk i from
// the file, the GPU copies chunk i-1 and repacks it to the uint8 fast/full
// row blocks (icq_index_repack_rows) -- the uint32 block never exists in
// host or device memory as a whole.
//
// Layout (little-endian): "ICQI", u32 version (1), Config "<IIddddddIIdQ"
// (80 bytes), u32 n, u32 d, f32 codewords[K*m*d], u32 codes[n*K], u32 d +
// u8 xi[d], u32 K + u8 fast_mask[K], u32 d + f32 lambdas[d], f32 sigma.
#include <sys/stat.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "icq_index.cuh"

namespace {

constexpr uint32_t kIndexFormatVersion = 1;  // data.py:22
constexpr size_t kConfigBytes = 80;          // struct "<IIddddddIIdQ" (data.py:28)

struct File {
  FILE* f = nullptr;
  int64_t size = 0, off = 0;
  ~File() {
    if (f) fclose(f);
  }
};

template <typename T>
T rd(const unsigned char* p) {
  T v;
  memcpy(&v, p, sizeof(T));
  return v;
}

// r.take(count) of the reference: a short read is a FormatError naming the offset
icq_status take(File& F, void* dst, int64_t count, const char* path) {
  if (count < 0 || F.off + count > F.size)
    return icq_fail(ICQ_ERR_FORMAT, "index file %s truncated at offset %lld", path, (long long)F.off);
  if (count && fread(dst, 1, (size_t)count, F.f) != (size_t)count)
    return icq_fail(ICQ_ERR_FORMAT, "index file %s: read error at offset %lld", path, (long long)F.off);
  F.off += count;
  return ICQ_OK;
}

// Config.__post_init__ (data.py:102-122); a failure is FormatError (data.py:364-366)
icq_status check_config(const icq_index_file_info& c) {
  const char* why = nullptr;
  if (c.K < 1) why = "K must be >= 1";
  else if (c.m < 2) why = "m must be >= 2";
  else if (c.gamma1 < 0 || c.gamma2 < 0) why = "gamma1 and gamma2 must be non-negative";
  else if (!(c.pi1 > c.pi2 && c.pi2 > 0)) why = "need pi1 > pi2 > 0";
  else if (std::fabs(c.pi1 + c.pi2 - 1.0) > 1e-12) why = "pi1 + pi2 must equal 1";
  else if (c.alpha2 >= 0) why = "alpha2 must be negative";
  else if (c.sigma_scale < 0) why = "sigma_scale must be >= 0";
  else if (c.epochs < 1 || c.batch_size < 1) why = "epochs and batch_size must be >= 1";
  else if (c.learning_rate <= 0) why = "learning_rate must be > 0";
  if (why) return icq_fail(ICQ_ERR_FORMAT, "index config invalid: %s", why);
  return ICQ_OK;
}

// header (magic, version, config, n, d): leaves the file positioned after d
icq_status read_header(File& F, const char* path, icq_index_file_info* info) {
  F.f = fopen(path, "rb");
  if (!F.f) return icq_fail(ICQ_ERR_VALIDATION, "cannot open %s", path);
  struct stat sb;
  if (fstat(fileno(F.f), &sb) != 0) return icq_fail(ICQ_ERR_VALIDATION, "cannot stat %s", path);
  F.size = (int64_t)sb.st_size;
  unsigned char b[kConfigBytes];
  icq_status st;
  if ((st = take(F, b, 4, path)) != ICQ_OK) return st;
  if (memcmp(b, "ICQI", 4) != 0) return icq_fail(ICQ_ERR_FORMAT, "bad index magic in %s", path);
  if ((st = take(F, b, 4, path)) != ICQ_OK) return st;
  const uint32_t version = rd<uint32_t>(b);
  if (version != kIndexFormatVersion)
    return icq_fail(ICQ_ERR_VERSION, "index format version %u, this build reads %u", version,
                    kIndexFormatVersion);
  if ((st = take(F, b, kConfigBytes, path)) != ICQ_OK) return st;
  memset(info, 0, sizeof(*info));
  const uint32_t K = rd<uint32_t>(b), m = rd<uint32_t>(b + 4);
  info->K = (int64_t)K;
  info->m = (int64_t)m;
  info->gamma1 = rd<double>(b + 8);
  info->gamma2 = rd<double>(b + 16);
  info->pi1 = rd<double>(b + 24);
  info->pi2 = rd<double>(b + 32);
  info->alpha2 = rd<double>(b + 40);
  info->sigma_scale = rd<double>(b + 48);
  info->epochs = rd<uint32_t>(b + 56);
  info->batch_size = rd<uint32_t>(b + 60);
  info->learning_rate = rd<double>(b + 64);
  info->seed = rd<uint64_t>(b + 72);
  if ((st = check_config(*info)) != ICQ_OK) return st;
  if ((st = take(F, b, 8, path)) != ICQ_OK) return st;
  info->n = rd<uint32_t>(b);
  info->d = rd<uint32_t>(b + 4);
  info->file_bytes = F.size;
  return ICQ_OK;
}

// the sections after the code block, validated like data.py:369-385 and
// SearchIndex.__post_init__ (xi in {0,1}, lambdas finite >= 0, sigma finite >= 0)
icq_status read_tail(File& F, const char* path, icq_index_file_info* info, uint8_t* xi,
                     float* lam) {
  const int64_t K = info->K, d = info->d;
  unsigned char b[4];
  icq_status st;
  if ((st = take(F, b, 4, path)) != ICQ_OK) return st;
  if ((int64_t)rd<uint32_t>(b) != d)
    return icq_fail(ICQ_ERR_FORMAT, "mask length %u does not match d=%lld", rd<uint32_t>(b), (long long)d);
  if ((st = take(F, xi, d, path)) != ICQ_OK) return st;
  if ((st = take(F, b, 4, path)) != ICQ_OK) return st;
  if ((int64_t)rd<uint32_t>(b) != K)
    return icq_fail(ICQ_ERR_FORMAT, "fast mask length %u does not match K=%lld", rd<uint32_t>(b), (long long)K);
  std::vector<uint8_t> fm((size_t)K);
  if ((st = take(F, fm.data(), K, path)) != ICQ_OK) return st;
  if ((st = take(F, b, 4, path)) != ICQ_OK) return st;
  if ((int64_t)rd<uint32_t>(b) != d)
    return icq_fail(ICQ_ERR_FORMAT, "variance length %u does not match d=%lld", rd<uint32_t>(b), (long long)d);
  if ((st = take(F, lam, 4 * d, path)) != ICQ_OK) return st;
  if ((st = take(F, b, 4, path)) != ICQ_OK) return st;
  info->sigma = rd<float>(b);
  if (F.off != F.size)
    return icq_fail(ICQ_ERR_FORMAT, "index file %s has %lld trailing bytes", path,
                    (long long)(F.size - F.off));
  // SearchIndex validation (a failure is FormatError, data.py:386-394)
  for (int64_t i = 0; i < d; ++i)
    if (xi[i] > 1) return icq_fail(ICQ_ERR_FORMAT, "index fields invalid: xi entries must be 0 or 1");
  for (int64_t i = 0; i < d; ++i)
    if (!std::isfinite(lam[i]) || lam[i] < 0)
      return icq_fail(ICQ_ERR_FORMAT, "index fields invalid: lambdas must be finite and non-negative");
  if (!std::isfinite(info->sigma) || info->sigma < 0)
    return icq_fail(ICQ_ERR_FORMAT, "index fields invalid: sigma must be finite and >= 0");
  info->F = 0;  // fast = flatnonzero(fast_mask) (data.py:390)
  for (int64_t b2 = 0; b2 < K && b2 < 64; ++b2)
    if (fm[(size_t)b2]) info->fast[info->F++] = (uint32_t)b2;
  return ICQ_OK;
}

}  // namespace

extern "C" {

icq_status icq_index_file_info_read(const char* path, icq_index_file_info* info) {
  if (!path || !info) return icq_fail(ICQ_ERR_VALIDATION, "null argument");
  File F;
  return read_header(F, path, info);
}

icq_status icq_index_load(const char* path, float* books_host, uint8_t* xi_host,
                          float* lambdas_host, icq_index_file_info* info, void* stream,
                          icq_index_t* out) {
  if (!path || !info || !out) return icq_fail(ICQ_ERR_VALIDATION, "null argument");
  *out = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  File F;
  icq_status st = read_header(F, path, info);
  if (st != ICQ_OK) return st;
  const int64_t K = info->K, m = info->m, d = info->d, n = info->n;
  const int64_t book_bytes = K * m * d * 4, code_bytes = n * K * 4;
  const int64_t books_off = F.off, codes_off = books_off + book_bytes;
  // sections the reference parses after the codes first: a malformed tail
  // fails before any device work (every case is a FormatError there too)
  std::vector<uint8_t> xi((size_t)(d > 0 ? d : 1));
  std::vector<float> lam((size_t)(d > 0 ? d : 1));
  if (codes_off + code_bytes > F.size) {  // r.take of the codeword / code block
    const int64_t at = books_off + book_bytes > F.size ? books_off : codes_off;
    return icq_fail(ICQ_ERR_FORMAT, "index file %s truncated at offset %lld", path, (long long)at);
  }
  if (fseeko(F.f, (off_t)(codes_off + code_bytes), SEEK_SET) != 0)
    return icq_fail(ICQ_ERR_FORMAT, "index file %s: seek failed", path);
  F.off = codes_off + code_bytes;
  if ((st = read_tail(F, path, info, xi.data(), lam.data())) != ICQ_OK) return st;
  // valid for the reference; outside this build?
  if (K > icq::kMaxK) return icq_fail(ICQ_ERR_UNSUPPORTED, "K=%lld > %d books", (long long)K, icq::kMaxK);
  if (m > 256) return icq_fail(ICQ_ERR_UNSUPPORTED, "m=%lld > 256 codewords (uint8 codes)", (long long)m);
  if (n < 1) return icq_fail(ICQ_ERR_UNSUPPORTED, "empty index (n = 0)");
  if (d < 1 || d > 8192) return icq_fail(ICQ_ERR_UNSUPPORTED, "d=%lld out of range [1, 8192]", (long long)d);
  // books (small) through the host
  std::vector<float> books((size_t)(K * m * d));
  if (fseeko(F.f, (off_t)books_off, SEEK_SET) != 0)
    return icq_fail(ICQ_ERR_FORMAT, "index file %s: seek failed", path);
  F.off = books_off;
  if ((st = take(F, books.data(), book_bytes, path)) != ICQ_OK) return st;
  icq_index_t h = nullptr;
  if ((st = icq_index_alloc(books.data(), false, (int32_t)K, (int32_t)m, (int32_t)d, n, info->fast,
                            info->F, s, &h)) != ICQ_OK)
    return st;
  // stream the code block: file -> pinned[b] -> device staging[b] -> repack
  const int64_t chunk_rows = std::max<int64_t>(1, ((int64_t)64 << 20) / (K * 4));
  const size_t cbytes = (size_t)(chunk_rows * K * 4);
  uint32_t* pin[2] = {nullptr, nullptr};
  uint32_t* dst[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  cudaError_t e = cudaSuccess;
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = cudaMallocHost((void**)&pin[b], cbytes);
    if (e == cudaSuccess) e = cudaMalloc((void**)&dst[b], cbytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
  }
  int64_t row = 0;
  for (int c = 0; e == cudaSuccess && st == ICQ_OK && row < n; ++c) {
    const int b = c & 1;
    const int64_t rows = std::min(chunk_rows, n - row);
    if (c >= 2) e = cudaEventSynchronize(done[b]);  // pin[b]'s previous copy has landed
    if (e != cudaSuccess) break;
    st = take(F, pin[b], rows * K * 4, path);       // CPU: read chunk c while the GPU repacks c-1
    if (st != ICQ_OK) break;
    e = cudaMemcpyAsync(dst[b], pin[b], (size_t)(rows * K * 4), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(done[b], s);
    if (e == cudaSuccess) e = icq_index_repack_rows(h, dst[b], 4, row, rows, s);
    row += rows;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  for (int b = 0; b < 2; ++b) {
    cudaFreeHost(pin[b]);
    cudaFree(dst[b]);
    if (done[b]) cudaEventDestroy(done[b]);
  }
  if (st == ICQ_OK && e != cudaSuccess)
    st = icq_fail(ICQ_ERR_CUDA, "index code stream failed: %s", cudaGetErrorString(e));
  if (st == ICQ_OK && (icq_index_repack_errors(h) & 2))
    st = icq_fail(ICQ_ERR_FORMAT, "index fields invalid: codes reference codewords beyond m");
  if (st != ICQ_OK) {
    icq_index_free(h);
    return st;
  }
  if (books_host) memcpy(books_host, books.data(), (size_t)book_bytes);
  if (xi_host) memcpy(xi_host, xi.data(), (size_t)d);
  if (lambdas_host) memcpy(lambdas_host, lam.data(), (size_t)(4 * d));
  *out = h;
  return ICQ_OK;
}

}  // extern "C"

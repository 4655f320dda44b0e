// icq_index.cuh — the device-resident index behind icq_index_t and the
// internal helpers shared by the C-ABI translation units (icq_capi.cu:
// create/search, icq_io.cu: ICQI streaming loader, icq_brute.cu).
#pragma once
#include <cstdarg>
#include <mutex>

#include "../../include/icq_b200.h"
#include "icq_common.cuh"

struct icq_index_s {
  int32_t K, m, d, F, KP, FP;
  int64_t n, n_pad;
  float* books;
  uint8_t* codes_full;   // (n_pad, KP) row-major: random row reads (refinements)
  uint8_t* codes_fast;   // fast books, tile-transposed (streamed by the filter)
  uint8_t* codes_xfull;  // all books, tile-transposed (the exact engine's stream)
  uint8_t fast_books[icq::kMaxK];
  icq::FastBooks fb;
  icq::LutProg* prog_dev;
  int32_t* err_dev;      // repack error word (bit 1: a code >= m)
  int64_t bytes;
  // device scratch of the synchronous host-buffer path, reused across calls
  std::mutex host_mu;
  char* host_buf = nullptr;
  size_t host_buf_bytes = 0;
};

// thread-local error message of the C ABI (icq_last_error)
icq_status icq_fail(icq_status code, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return icq_fail(ICQ_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                      __LINE__);                                                             \
  } while (0)

// shape validation, device allocation, books upload (synchronous); codes zeroed
icq_status icq_index_alloc(const float* books, bool books_on_device, int32_t K, int32_t m,
                           int32_t d, int64_t n, const uint32_t* fast, int32_t F,
                           cudaStream_t stream, icq_index_t* out);
// repack rows [row0, row0 + rows) from a device (rows, K) block of uint32
// (code_bytes 4) or uint8 (1) codes; asynchronous on s
cudaError_t icq_index_repack_rows(icq_index_t h, const void* codes_dev, int code_bytes,
                                  int64_t row0, int64_t rows, cudaStream_t s);
int32_t icq_index_repack_errors(icq_index_t h);
void icq_index_free(icq_index_t h);

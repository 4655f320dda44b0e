// icq_types.cuh — parameter blocks shared by the host launcher and kernels.
#pragma once
#include <cstdint>

#include "icq_device.cuh"

namespace icq {

// Postfix program of numpy's pairwise float64 summation over d elements
// (leaves of <= 128 elements; op >= 0 is a leaf start, -1 adds the top two).
struct LutProg {
  int32_t nops;
  int32_t op[256];
  int32_t len[256];
};

struct FastBooks {
  uint8_t b[kMaxK];
};

struct ScanParams {
  const uint8_t* codes_fast;  // [n_pad * FP]   fast books only (row-major), zero padded
  const uint8_t* codes_full;  // [n_pad * KP]   all books (row-major), zero padded
  const double* lut64;        // [Q][K][m]
  int64_t* ids;               // [Q*k]
  double* scores;             // [Q*k]
  int64_t* refinements;       // [Q] or null
  uint32_t* survivors;        // [Q*words] or null
  int64_t* stats;             // [Q*kStats] or null
  int32_t* error;             // device error word
  int64_t n;
  int64_t nseg;
  int64_t words;              // survivors bitmap words per query
  double sigma;
  int32_t K, m, KP, F;
  int32_t k;
  int32_t exact_mode;         // search_exact: report refinements = n (search.py:108)
  int32_t debug;              // experiments only (ICQ_DEBUG env): bit 0 = replay skips phase 2
  int32_t nb;                 // slots in the ring
  uint32_t off_lut64, off_heap_e, off_heap_f, off_heap_i, off_ctrl;
  uint32_t off_slots;         // contiguous ring of nb slots (aliased by the prologue buffer)
  uint32_t slot_bytes;
  // sub-layout of one slot (byte offsets from the slot start): per-warp meta
  // (candidate count, filter threshold used, warp minimum), then per-warp
  // candidate lists (id, fast32, code row)
  uint32_t so_lmin, so_eid, so_ef32, so_erow;  // so_lmin: per-lane minima (fallback gating)
  int32_t cw;                 // candidate list capacity per scan warp per segment
  int32_t dense_chunk;        // items per prologue chunk
  uint32_t smem_end;          // absolute end of the planned layout
  uint32_t dyn_bytes;
  uint8_t fast_books[kMaxK];
};

bool make_lut_prog(int d, LutProg* out);
cudaError_t launch_lut(const float* books, const double* q, double* lut, int K, int m, int d,
                       int Q, const LutProg* prog_dev, cudaStream_t s);
cudaError_t launch_scan(ScanParams& p, int FP, int Q, cudaStream_t s, int* unsupported);

}  // namespace icq

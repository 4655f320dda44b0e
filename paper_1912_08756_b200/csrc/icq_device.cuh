// icq_device.cuh — device helpers shared by the ICQ query kernels (sm_100a).
//
// Float64 helpers reproduce numpy's float64 add.reduce order exactly
// (identity 0, then pairwise blocks of 8 up to 128 elements, recursive
// halving above) — the order the reference uses at search.py:66 and :94.
// All float64 arithmetic that must match the reference goes through the
// __d*_rn intrinsics so nvcc never contracts it into an FMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace icq {

constexpr int kMaxK = 16;          // books per index supported by this build
constexpr uint32_t kPage = 65536;  // lane-private LUT pages live at 64 KiB-aligned smem addresses
constexpr uint32_t kSmemWindow = 233472;  // B200: 1 KiB reserved + 227 KiB dynamic
constexpr uint32_t kDynBase = 1024;       // dynamic smem base when the kernel has no static smem
constexpr int kStats = 16;                // int64 diagnostics per query (icq_b200.h stats_dev)

// --------------------------------------------------------------------------
// shared-memory access by absolute (window) address
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32x4(uint32_t a, float v) {  // v in 4 consecutive floats
  asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}

// bulk prefetch of `bytes` (multiple of 16, 16-B aligned) into L2
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// --------------------------------------------------------------------------
// streaming 16-byte code loads (read once per query; do not pollute L1)
// --------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// --------------------------------------------------------------------------
// numpy float64 reduction order of the reference's gathered scores
// (search.py:94: lut[books[None, :], codes[:, books]].sum(axis=1)).
// numpy lays the fancy-indexed (n, t) result out F-contiguous whenever
// n >= 2, so the row sum accumulates sequentially in book order
// (((0 + x0) + x1) + x2) ...; for n == 1 the array is also C-contiguous and
// numpy's pairwise kernel runs (8 strided accumulators for t >= 8).  Pinned
// against the reference in tests/test_oracle_golden.py.
// --------------------------------------------------------------------------
template <typename TermFn>
__device__ __forceinline__ double ref_row_sum(int nterms, bool pairwise, TermFn t) {
  if (!pairwise || nterms < 8) {
    // issue every table load first (nterms <= kMaxK), then the dependent adds
    double v[kMaxK];
#pragma unroll
    for (int i = 0; i < kMaxK; ++i) v[i] = i < nterms ? t(i) : 0.0;
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
      if (i < nterms) r = __dadd_rn(r, v[i]);
    return r;
  }
  double r0 = t(0), r1 = t(1), r2 = t(2), r3 = t(3), r4 = t(4), r5 = t(5), r6 = t(6), r7 = t(7);
  int i = 8;
  const int top = nterms - (nterms % 8);
  for (; i < top; i += 8) {
    r0 = __dadd_rn(r0, t(i + 0));
    r1 = __dadd_rn(r1, t(i + 1));
    r2 = __dadd_rn(r2, t(i + 2));
    r3 = __dadd_rn(r3, t(i + 3));
    r4 = __dadd_rn(r4, t(i + 4));
    r5 = __dadd_rn(r5, t(i + 5));
    r6 = __dadd_rn(r6, t(i + 6));
    r7 = __dadd_rn(r7, t(i + 7));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                         __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
  for (; i < nterms; ++i) res = __dadd_rn(res, t(i));
  return __dadd_rn(0.0, res);
}

// Certified float32 decision thresholds for "x64 < thr64" given a float32
// value x32 that approximates x64 = (numpy-order float64 sum of `nterms`
// non-negative table entries) with |x32 - x64| <= nterms*2^-24*x64 (+tiny):
//   x32 <  lo  =>  x64 <  thr64   (sure)
//   x32 >= hi  =>  x64 >= thr64   (sure)
//   otherwise the caller recomputes x64 exactly.
// A NaN threshold yields NaN bounds: every comparison is false, which is
// the reference's own NaN behaviour for search.py:149.
__device__ __forceinline__ void certified_bounds(double thr64, int nterms, float& lo, float& hi) {
  const double e = 2.0 * nterms * 5.9604644775390625e-08;       // 2 * nterms * 2^-24
  const double a = nterms * 7.174648137343064e-43;               // nterms * 2^-140
  const double H = __dadd_rn(__dmul_rn(thr64, 1.0 + e), a);
  const double L = __dsub_rn(__dmul_rn(thr64, 1.0 - e), a);
  hi = __double2float_ru(H);
  lo = __double2float_rd(L);
}

}  // namespace icq

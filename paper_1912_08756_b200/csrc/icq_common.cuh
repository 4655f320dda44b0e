// icq_common.cuh — device pieces shared by the prologue, filter and replay
// kernels: float64 row scores in the reference's order, the (exact, id) key,
// the replay warp's heap, and the live threshold state.
//
// Reference semantics: search_two_step, /root/reference/pkg/src/icq/search.py:112-165
//   heap seeded with ids 0..k-1 scored exactly                      (:141-143)
//   element i >= k refined iff fast[i] < bound + sigma, where bound is the
//   FAST score of the current heap maximum by (exact, id)            (:149, :154)
//   inserted iff exact[i] < exact(heap max) (strict)                 (:152-153)
//   result: the heap sorted ascending by (score, id)                 (:156)
#pragma once

#include "icq_types.cuh"

namespace icq {

#define kInf (__int_as_float(0x7f800000))
#define kInf64 (__longlong_as_double(0x7ff0000000000000LL))

// --------------------------------------------------------------------------
// code rows and float64 scores in the reference's order (search.py:94)
// --------------------------------------------------------------------------
struct Row {
  uint32_t w[4];
  __device__ __forceinline__ uint32_t byte(int b) const {
    const uint32_t x = (b < 4) ? w[0] : (b < 8) ? w[1] : (b < 12) ? w[2] : w[3];
    return (x >> ((b & 3) * 8)) & 0xffu;
  }
};

__device__ __forceinline__ Row load_row(const uint8_t* codes_full, int KP, int64_t id) {
  Row r;
  r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0;
  const uint8_t* p = codes_full + id * KP;
  if (KP == 16) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    r.w[0] = v.x; r.w[1] = v.y; r.w[2] = v.z; r.w[3] = v.w;
  } else if (KP == 8) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    r.w[0] = v.x; r.w[1] = v.y;
  } else if (KP == 4) {
    r.w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
  } else if (KP == 2) {
    r.w[0] = __ldg(reinterpret_cast<const uint16_t*>(p));
  } else {
    r.w[0] = __ldg(p);
  }
  return r;
}

// Same, with an L2 evict_last policy: count-mode candidate rows are re-read
// by every query of a batch scanning the same range; keep them resident
// against the fast-code stream.
__device__ __forceinline__ Row load_row_keep(const uint8_t* codes_full, int KP, int64_t id,
                                             uint64_t pol) {
  Row r;
  r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0;
  const uint8_t* p = codes_full + id * KP;
  if (KP == 16) {
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]) : "l"(p), "l"(pol));
  } else if (KP == 8) {
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.w[0]), "=r"(r.w[1]) : "l"(p), "l"(pol));
  } else {
    return load_row(codes_full, KP, id);
  }
  return r;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Tile-transposed layout of the streamed fast rows (codes_fast): within each
// tile of 128 16-byte chunks, logical chunk lc = 4*lane + v is stored at
// physical chunk 32*v + lane.  A coalesced warp load of chunks 32*v + lane
// (v = 0..3) then hands every lane 4 CONSECUTIVE logical chunks, so a lane's
// items form one contiguous id run (ordered compaction = one lane scan).
__host__ __device__ inline int64_t perm_chunk(int64_t lc) {
  return (lc & ~(int64_t)127) | ((lc & 3) << 5) | ((lc & 127) >> 2);
}
__host__ __device__ inline int64_t perm_offset(int FP, int64_t i) {  // byte offset of item i
  const int ipc = 16 / FP;
  return perm_chunk(i / ipc) * 16 + (i % ipc) * FP;
}
__device__ __forceinline__ Row load_fast_row(const uint8_t* codes_fast, int FP, int64_t i) {
  Row r;
  r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0;
  const uint8_t* q = codes_fast + perm_offset(FP, i);
  if (FP == 16) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(q));
    r.w[0] = v.x; r.w[1] = v.y; r.w[2] = v.z; r.w[3] = v.w;
  } else if (FP == 8) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(q));
    r.w[0] = v.x; r.w[1] = v.y;
  } else if (FP == 4) {
    r.w[0] = __ldg(reinterpret_cast<const uint32_t*>(q));
  } else if (FP == 2) {
    r.w[0] = __ldg(reinterpret_cast<const uint16_t*>(q));
  } else {
    r.w[0] = __ldg(q);
  }
  return r;
}

__device__ __forceinline__ double exact64(const double* lut, int m, int K, bool pw, const Row& r) {
  return ref_row_sum(K, pw, [&](int b) { return lut[b * m + (int)r.byte(b)]; });
}

__device__ __forceinline__ double fast64(const double* lut, int m, int F, bool pw,
                                         const uint8_t* fb, const Row& r) {
  return ref_row_sum(F, pw, [&](int s) {
    const int b = fb[s];
    return lut[b * m + (int)r.byte(b)];
  });
}

// float32 sum of a code row over a [KP][m] float32 table whose rows b >= K are
// zero (code rows are zero-padded to KP bytes): the certified pre-test of
// "exact64 < T" (certified_bounds with K terms; adding the zero rows is exact).
template <int KPc>
__device__ __forceinline__ float exact32_row(const float* lut32k, int m, const Row& r) {
  float e = 0.f;
#pragma unroll
  for (int b = 0; b < KPc; ++b) e += lut32k[b * m + (int)((r.w[b >> 2] >> ((b & 3) * 8)) & 0xffu)];
  return e;
}
__device__ __forceinline__ float exact32_any(const float* lut32k, int m, int KP, const Row& r) {
  switch (KP) {  // (warp-uniform)
    case 16: return exact32_row<16>(lut32k, m, r);
    case 8: return exact32_row<8>(lut32k, m, r);
    case 4: return exact32_row<4>(lut32k, m, r);
    case 2: return exact32_row<2>(lut32k, m, r);
    default: return exact32_row<1>(lut32k, m, r);
  }
}
// stage that table from the float64 LUT of a query (all threads of the CTA)
__device__ __forceinline__ void stage_lut32k(float* lut32k, const double* glut, int K, int KP, int m,
                                             int tid, int nthreads) {
  for (int i = tid; i < KP * m; i += nthreads) lut32k[i] = i < K * m ? __double2float_rn(glut[i]) : 0.f;
}

// (exact, id) ordering of the reference heap (search.py:140: keys (-exact, -id))
__device__ __forceinline__ bool key_gt(double e1, int32_t i1, double e2, int32_t i2) {
  // branch-free (no short-circuit): the replay warp's hot compares must not
  // open divergence regions
  const bool gt = e1 > e2, eq = e1 == e2, ig = i1 > i2;
  return gt | (eq & ig);
}

// Replace the maximum (entry 0) of a descending-sorted heap in shared memory.
static __device__ void heap_replace_max(double* he, double* hf, int32_t* hi, int k, double e,
                                        int32_t id, double f, int lane) {
  int g = 0;
  for (int base = 1; base < k; base += 32) {
    const int i = base + lane;
    const bool gt = (i < k) && key_gt(he[i < k ? i : 0], hi[i < k ? i : 0], e, id);
    g += __popc(__ballot_sync(0xffffffffu, gt));
  }
  for (int base = 0; base < g; base += 32) {
    const int i = base + lane;
    double te = 0, tf = 0;
    int32_t ti = 0;
    if (i < g) { te = he[i + 1]; tf = hf[i + 1]; ti = hi[i + 1]; }
    __syncwarp();
    if (i < g) { he[i] = te; hf[i] = tf; hi[i] = ti; }
    __syncwarp();
  }
  if (lane == 0) { he[g] = e; hf[g] = f; hi[g] = id; }
  __syncwarp();
}

// The replay warp's view of the heap: the k best (exact, id) entries sorted
// descending (entry 0 = heap maximum, search.py:140).  For k <= 128 the
// entries live in warp registers in a BLOCKED layout (lane l holds entries
// 4l..4l+3): an insertion shifts registers locally, moves only the lane
// boundary entry with one shuffle per field, and finds its position with one
// __reduce_add_sync.  Larger k keeps the sorted array in shared memory.  A
// warp-uniform copy of the top entry (refreshed by shuffles from lane 0 after
// each insertion) gives T and the bound; a deeper uniform cache (2 or 4
// entries, kept sorted with per-lane ALU work) measured slower.
constexpr int kRegHeapRegs = 4;
constexpr int kTopC = 1;
struct WarpHeap {
  int k;
  bool reg;
  double e[kRegHeapRegs], f[kRegHeapRegs];
  int32_t id[kRegHeapRegs];
  double* he;
  double* hf;
  int32_t* hi;
  double ue[kTopC], uf[kTopC];
  int32_t ui[kTopC];
  int uc;

  __device__ __forceinline__ void load(int lane) {
    if (reg) {
#pragma unroll
      for (int r = 0; r < kRegHeapRegs; ++r) {
        const int i = kRegHeapRegs * lane + r;
        e[r] = i < k ? he[i] : 0.0;
        f[r] = i < k ? hf[i] : 0.0;
        id[r] = i < k ? hi[i] : 0;
      }
    }
    refill();
  }
  __device__ __forceinline__ void store(int lane) {
    if (!reg) return;
#pragma unroll
    for (int r = 0; r < kRegHeapRegs; ++r) {
      const int i = kRegHeapRegs * lane + r;
      if (i < k) { he[i] = e[r]; hf[i] = f[r]; hi[i] = id[r]; }
    }
    __syncwarp();
  }
  __device__ __forceinline__ void refill() {
#pragma unroll
    for (int j = 0; j < kTopC; ++j) {
      if (reg) {  // entries 0..kTopC-1 sit in lane 0 (kTopC <= kRegHeapRegs)
        ue[j] = __shfl_sync(0xffffffffu, e[j], 0);
        uf[j] = __shfl_sync(0xffffffffu, f[j], 0);
        ui[j] = __shfl_sync(0xffffffffu, id[j], 0);
      } else {
        ue[j] = j < k ? he[j] : 0.0;
        uf[j] = j < k ? hf[j] : 0.0;
        ui[j] = j < k ? hi[j] : 0;
      }
    }
    uc = k < kTopC ? k : kTopC;
  }
  __device__ __forceinline__ double top_e() const { return ue[0]; }
  __device__ __forceinline__ double top_f() const { return uf[0]; }
  __device__ __forceinline__ int32_t top_i() const { return ui[0]; }
  __device__ __forceinline__ void replace_max(double xe, int32_t xid, double xf, int lane) {
    // 1. uniform top cache: drop entry 0, insert x if it ranks inside the prefix
    double le = ue[0];
    int32_t li = ui[0];
#pragma unroll
    for (int j = 1; j < kTopC; ++j)
      if (j == uc - 1) { le = ue[j]; li = ui[j]; }
    const bool in = uc >= 2 && key_gt(xe, xid, le, li);
#pragma unroll
    for (int j = 0; j < kTopC; ++j) {
      const int jn = j + 1 < kTopC ? j + 1 : j;
      const bool above_gt = (j + 1 < uc) && key_gt(ue[jn], ui[jn], xe, xid);
      const bool here_gt = j == 0 ? true : ((j < uc) && key_gt(ue[j], ui[j], xe, xid));
      if (above_gt) { ue[j] = ue[jn]; uf[j] = uf[jn]; ui[j] = ui[jn]; }
      else if (here_gt && in) { ue[j] = xe; uf[j] = xf; ui[j] = xid; }
    }
    if (!in) --uc;
    // 2. the full sorted array (lanes or shared memory)
    replace_max_array(xe, xid, xf, lane);
    if (uc < 2 && k >= 2) refill();
    if (k == 1) { ue[0] = xe; uf[0] = xf; ui[0] = xid; uc = 1; }
  }
  __device__ __forceinline__ void replace_max_array(double xe, int32_t xid, double xf, int lane) {
    if (!reg) {
      heap_replace_max(he, hf, hi, k, xe, xid, xf, lane);
      return;
    }
    int cnt = 0;  // this lane's entries among 1..k-1 that stay above x
#pragma unroll
    for (int r = 0; r < kRegHeapRegs; ++r) {
      const int i = kRegHeapRegs * lane + r;
      cnt += ((i >= 1) & (i < k) & key_gt(e[r], id[r], xe, xid)) ? 1 : 0;
    }
    const int g = __reduce_add_sync(0xffffffffu, cnt);  // sorted: they are entries 1..g
    const double ne = __shfl_down_sync(0xffffffffu, e[0], 1);
    const double nf = __shfl_down_sync(0xffffffffu, f[0], 1);
    const int32_t ni = __shfl_down_sync(0xffffffffu, id[0], 1);
#pragma unroll
    for (int r = 0; r < kRegHeapRegs; ++r) {
      const int i = kRegHeapRegs * lane + r;
      const int rn = r + 1 < kRegHeapRegs ? r + 1 : r;
      const double se = r + 1 < kRegHeapRegs ? e[rn] : ne;
      const double sf = r + 1 < kRegHeapRegs ? f[rn] : nf;
      const int32_t si = r + 1 < kRegHeapRegs ? id[rn] : ni;
      if (i < g) { e[r] = se; f[r] = sf; id[r] = si; }
      else if (i == g) { e[r] = xe; f[r] = xf; id[r] = xid; }
    }
  }
};

// --------------------------------------------------------------------------
// The refinement threshold of search.py:149, `fast[i] < bound + sigma`, as a
// float64 value t with the reference's test == `fast64 < t`.
//
// float64 sigma (a Python float / np.float64 argument, and index.sigma, which
// data.py:252 stores as a Python float): t = bound + sigma, one float64 add.
//
// np.float32 sigma (sigma_f32, numpy >= 2 promotion rules, NEP 50): while the
// heap maximum is a seed (id < k) its cached fast score is an np.float64
// (search.py:141, indexing fast_all) and the sum stays float64.  Once it is an
// inserted entry the cached score is a Python float (:153, from fast_list), so
// `bound + sigma` is a float32 add of float32(bound), and the comparison
// `fast_list[i] < np.float32` rounds fast_list[i] to float32 as well.
// float32(x) < t32 <=> x < lb(t32), lb = the smallest double that rounds to a
// float32 >= t32 (round-to-nearest-even is monotone).
// --------------------------------------------------------------------------
__device__ __forceinline__ double f32_lower_boundary(float t) {
  if (!(t == t)) return (double)t;                 // NaN: every comparison false
  if (t <= 0.f) return 0.0;                        // (fast >= 0) nothing rounds below 0
  if (t == kInf) return 3.4028235677973366e38;     // 2^128 - 2^103 rounds to inf (tie, even)
  const uint32_t b = __float_as_uint(t);
  const double mid = ((double)__uint_as_float(b - 1u) + (double)t) * 0.5;  // exact
  // a tie rounds to the even neighbour: mid itself rounds up to t iff t is even
  return (b & 1u) ? __longlong_as_double(__double_as_longlong(mid) + 1) : mid;
}
__device__ __forceinline__ double live_thr(double bound, int32_t max_id, double sigma, int k,
                                           bool f32) {
  if (!f32 || max_id < k) return __dadd_rn(bound, sigma);
  return f32_lower_boundary(__fadd_rn(__double2float_rn(bound), (float)sigma));
}
// an upper bound of live_thr over every bound <= b (both forms are monotone in b)
__device__ __forceinline__ double thr_cover(double b, double sigma, bool f32, bool round_up) {
  double t = round_up ? __dadd_ru(b, sigma) : __dadd_rn(b, sigma);
  if (f32) t = fmax(t, f32_lower_boundary(__fadd_rn(__double2float_rn(b), (float)sigma)));
  return t;
}

// Replay state (one warp; warp-uniform registers)
struct Live {
  double T64, bound64, thr64;
  float lo, hi;
  int64_t refinements, insertions, candidates, certified;
  int32_t ntraj;  // count mode: trajectory entries recorded
  WarpHeap H;
};

__device__ __forceinline__ void live_update64(Live& L, double sigma, int k, bool f32) {
  L.T64 = L.H.top_e();
  L.bound64 = L.H.top_f();
  L.thr64 = live_thr(L.bound64, L.H.top_i(), sigma, k, f32);  // search.py:149 `bound + sigma`
}

// + certified float32 thresholds of "fast64 < thr64"
__device__ __forceinline__ void live_update(Live& L, int F, double sigma, int k, bool f32,
                                            bool wide) {
  live_update64(L, sigma, k, f32);
  if (wide) {
    L.lo = -kInf;
    L.hi = kInf;
  } else {
    certified_bounds(L.thr64, F, L.lo, L.hi);
  }
}

// Stale filter threshold valid for EVERY later item:
//  sigma == 0: M = max fast over the heap never increases (an inserted item
//              has fast < bound <= M), and bound <= M;
//  sigma  > 0: U = max(M, T - Smin) never increases (inserted x: fast(x) <=
//              exact(x) - Smin < T - Smin) and bound <= U; filter at U + sigma.
// An item is a candidate iff fast64 < thr.  The float32 pre-test: x32 < lo
// => candidate, x32 >= hi => not; in between (near-ties, and the exact ties
// that few-codeword books produce in bulk) the caller sums fast64 exactly.
struct StaleThr {
  double thr;
  float lo, hi;
};
__device__ __forceinline__ StaleThr stale_core(double M, bool nan, double T, int F, double sigma,
                                               double smin, bool wide, bool f32) {
  StaleThr r{__longlong_as_double(0x7ff0000000000000LL), kInf, kInf};
  if (wide || nan) return r;
  double thr;
  if (sigma == 0.0 && !f32) {
    thr = M;
  } else if (sigma == 0.0) {
    thr = thr_cover(M, 0.0, true, false);
  } else {
    // (T - Smin) with float64 slack for the different summation orders of
    // fast and exact scores (relative 1e-12 >> K * 2^-53)
    const double ts = __dsub_ru(T, smin);
    const double u = fmax(M, __dadd_ru(ts, fabs(T) * 1e-12));
    thr = thr_cover(u, sigma, f32, true);
  }
  if (!(thr == thr)) return r;
  r.thr = thr;
  certified_bounds(thr, F, r.lo, r.hi);
  return r;
}
// stale threshold from a heap array in shared memory (any order; entry 0 = maximum), one warp
__device__ __forceinline__ StaleThr stale_from_heap(const double* he, const double* hf, int k,
                                                    int F, double sigma, double smin, bool wide,
                                                    bool f32, int lane) {
  double M = -__longlong_as_double(0x7ff0000000000000LL);
  bool nan = false;
  for (int i = lane; i < k; i += 32) {
    M = fmax(M, hf[i]);
    nan |= !(hf[i] == hf[i]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
  nan = __any_sync(0xffffffffu, nan);
  return stale_core(M, nan, he[0], F, sigma, smin, wide, f32);
}

__device__ __forceinline__ void record_survivor(uint32_t* surv, int64_t id) {
  if (surv) atomicOr(surv + (id >> 5), 1u << (id & 31));
}

}  // namespace icq

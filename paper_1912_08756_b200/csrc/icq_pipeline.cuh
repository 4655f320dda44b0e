// icq_pipeline.cuh — the ICQ two-step query path as kernels per batch.
// (templates; instantiated per fast-row width in icq_pipe_fp*.cu, dispatched
// by icq_pipeline.cu)
//
// Reference: search_two_step, /root/reference/pkg/src/icq/search.py:112-165
// (search_exact :97-109 is the same pipeline with the fast set = all books and
// sigma = 0: then fast == exact and the prune predicate is the top-k test).
//
// The reference walks the database in order with a heap whose FAST score of
// the maximum is the pruning bound (:149).  The chain is sequential, but
// thresholds that dominate the live one let the streaming run on all SMs
// (tests/test_threshold_theory.py):
//
//   K2 icq_prologue_kernel  one CTA per query: the insertion-heavy start of
//        the database, in order (stale-threshold fp32 prefilter, float64
//        scores, warp-0 ballot-window decisions).  Ends with the list
//        threshold theta = A_J + sigma (J from a sampled ladder) or, for
//        refinement-heavy queries, count mode.
//   K3 icq_filter_kernel    the hot path: every SM streams fast-code bytes
//        (16-byte loads, register double buffer), gathers |F| fp32 entries
//        per item from lane-private replicated LUT pages (one byte_perm per
//        lookup, bank-conflict free) and compacts items under theta, in item
//        order, into per-(query, range, warp) slices of a paged pool
//        (count mode: only items that can still be inserted).
//   K4 icq_replay_kernel    one CTA per query: resumes the reference loop at
//        the prologue end over the slices in database order against the LIVE
//        bound; walks the database in order while the live threshold is
//        above theta; long walks hand the query to the next round.  Count
//        mode: insertions only, recording the threshold trajectory.
//   K5 icq_count_kernel     count mode: refinement counts and survivor bits
//        of every item against the trajectory, streamed like K3.
//
// Every decision compares the reference's float64 values, so ids, scores,
// refinement counts and survivor sets are bitwise the reference's.
#pragma once
#include <mutex>
#include <type_traits>

#ifndef ICQ_PREFETCH_TILES
#define ICQ_PREFETCH_TILES 0
#endif
// candidate mask of the filter: 1 = one funnel shift per item (ALU pipe),
// 0 = Horner multiply-adds (two FMA-pipe instructions per item)
// replay CTAs per SM the register budget is cut for (2: 255 registers, no spills)
#ifndef ICQ_REPLAY_CTAS
#define ICQ_REPLAY_CTAS 2
#endif
#ifndef ICQ_MASK_SHF
#define ICQ_MASK_SHF 1
#endif

#include "icq_common.cuh"

namespace icq {

constexpr uint32_t kFull = 0xffffffffu;

// --------------------------------------------------------------------------
// decision context shared by the prologue and replay warps
// --------------------------------------------------------------------------
struct RCtx {
  const double* lut;  // float64 LUT [K][m] in shared memory
  const uint8_t* codes_full;
  const uint8_t* fb;  // fast books
  int KP, m, K, F, k;
  double sigma;
  bool f32;  // numpy float32-sigma promotion (live_thr)
  bool pw, wide;
  bool count_mode;  // decide insertions only; record the threshold trajectory
  uint32_t* surv;
  TrajEntry* traj;
  int32_t* error;
};

struct Decided {
  int first;      // inserting lane or -1
  uint32_t done;  // lanes decided in this round
};

__device__ __forceinline__ uint32_t sel_u32(int c, uint32_t a, uint32_t b) {  // c ? a : b
  uint32_t r;
  asm("{ .reg .pred p; setp.ne.s32 p, %1, 0; selp.b32 %0, %2, %3, p; }" : "=r"(r) : "r"(c), "r"(a), "r"(b));
  return r;
}

// Fast-code tuple of item j of a 16-byte chunk (FP <= 8 bytes, little-endian
// in .x/.y); runtime j selects words, no dynamically indexed arrays.
template <int FP>
__device__ __forceinline__ uint2 chunk_tuple(const uint4& xv, int j) {
  if (FP <= 4) {
    const int bo = j * FP;
    const int wi = bo >> 2;
    // three selects on the bits of wi (no branches in the candidate loops)
    const uint32_t lo = sel_u32(wi & 1, xv.y, xv.x), hi = sel_u32(wi & 1, xv.w, xv.z);
    uint32_t w = sel_u32(wi & 2, hi, lo) >> ((bo & 3) * 8);
    if constexpr (FP < 4) w &= (1u << (8 * FP)) - 1u;
    return make_uint2(w, 0u);
  }
  return j == 0 ? make_uint2(xv.x, xv.y) : make_uint2(xv.z, xv.w);  // FP == 8
}

// float64 fast score of a tuple in the reference's order (search.py:94,
// sequential in book order for n >= 2); lut64f holds the fast books' rows.
template <int FP>
__device__ __forceinline__ double tuple_f64(uint2 t, const double* lut64f, int m, int F) {
  double d = 0.0;
#pragma unroll
  for (int s = 0; s < FP; ++s) {
    const uint32_t w = s < 4 ? t.x : t.y;
    if (s < F) d = __dadd_rn(d, lut64f[s * m + ((w >> (8 * (s & 3))) & 0xffu)]);
  }
  return d;
}

// --------------------------------------------------------------------------
// shared-memory layouts
// --------------------------------------------------------------------------
struct ProLayout {
  uint32_t lut64, lut32, lut32k, he, hf, hi, cf, ce, cid, ctrl, total;
};
__host__ __device__ inline uint32_t al16(uint32_t x) { return (x + 15u) & ~15u; }
__host__ __device__ inline ProLayout pro_layout(int K, int m, int F, int k) {
  ProLayout L;
  uint32_t o = 0;
  L.lut64 = o; o = al16(o + (uint32_t)K * m * 8);
  L.lut32 = o; o = al16(o + (uint32_t)(F > 0 ? F : 1) * m * 4);
  L.lut32k = o; o = al16(o + (uint32_t)(K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16) * m * 4);
  L.he = o;    o = al16(o + (uint32_t)k * 8);
  L.hf = o;    o = al16(o + (uint32_t)k * 8);
  L.hi = o;    o = al16(o + (uint32_t)k * 4);
  L.cf = o;    o = al16(o + kProBlock * 8);
  L.ce = o;    o = al16(o + kProBlock * 8);
  L.cid = o;   o = al16(o + kProBlock * 4);
  L.ctrl = o;  o = al16(o + 128);
  L.total = o;
  return L;
}

constexpr int kWU = 8;  // replay window: kWU x 32 entries
struct RepLayout {
  uint32_t lut64, lutf, he, hf, hi, wid, widx, wfv, wfe, meta, cum, chunks, ring, ringe, plist, ctl,
      total;
};
constexpr int kSG = 16;    // slices whose meta the replay stages in shared memory at once
constexpr int kCH = 512;   // candidate entries per staged chunk (replay ring slot)
constexpr int kRSlots = 4;  // replay ring: decide c | prepare c+1 | in flight c+2, c+3
__host__ __device__ inline RepLayout rep_layout(int K, int m, int F, int k) {
  RepLayout L;
  uint32_t o = 0;
  L.lut64 = o; o = al16(o + (uint32_t)K * m * 8);
  L.lutf = o;  o = al16(o + (uint32_t)(F > 0 ? F : 1) * m * 8);
  L.he = o;    o = al16(o + (uint32_t)k * 8);
  L.hf = o;    o = al16(o + (uint32_t)k * 8);
  L.hi = o;    o = al16(o + (uint32_t)k * 4);
  L.wid = o;   o = al16(o + kWU * 32 * 4);
  L.wfv = o;   o = al16(o + kWU * 32 * 8);
  L.wfe = o;   o = al16(o + kWU * 32 * 8);
  L.widx = o;  o = al16(o + kWU * 32 * 4);
  L.meta = o;  o = al16(o + kSG * kStageInts * 4);
  L.cum = o;   o = al16(o + (kSG + 1) * 4);
  L.chunks = o; o = al16(o + 512 * 3 * 4);
  L.ring = o;  o = al16(o + kRSlots * kCH * 16);
  L.ringe = o; o = al16(o + kRSlots * kCH * 8);
  L.plist = o; o = al16(o + kCH * 4);
  L.ctl = o;   o = al16(o + 128);
  L.total = o;
  return L;
}

// float64 min over the non-fast books' LUT rows, rounded down (U threshold)
static __device__ double smin_rd(const double* lut, int K, int m, const uint8_t* fb, int F, int lane) {
  double s = 0.0;
  for (int b = 0; b < K; ++b) {
    bool fast = false;
    for (int t = 0; t < F; ++t) fast |= fb[t] == b;
    if (fast) continue;
    double mn = __longlong_as_double(0x7ff0000000000000LL);
    for (int j = lane; j < m; j += 32) mn = fmin(mn, lut[b * m + j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
    s = __dadd_rd(s, mn);
  }
  return s;
}

// ==========================================================================
// K2: prologue
// ==========================================================================
// max fast score over the J+1 largest-exact heap entries (he/hf sorted
// descending by (exact, id): entries 0..J), warp-wide; *arg = its entry
__device__ __forceinline__ double heap_AJ(const double* hf, int k, int J, int lane, int* arg) {
  const int top = min(k, J + 1);
  double A = -kInf64;
  int ai = 0;
  for (int i = lane; i < top; i += 32)
    if (hf[i] > A) { A = hf[i]; ai = i; }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double oA = __shfl_xor_sync(kFull, A, o);
    const int oi = __shfl_xor_sync(kFull, ai, o);
    if (oA > A || (oA == A && oi < ai)) { A = oA; ai = oi; }
  }
  if (arg) *arg = ai;
  return A;
}

template <int FP>
__global__ void __launch_bounds__(kProThreads, 2) icq_prologue_kernel(const __grid_constant__ PipeParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = blockIdx.x;
  const int K = p.K, m = p.m, F = p.F, k = p.k;
  const int64_t n = p.n;
  const bool f32s = p.sigma_f32 != 0;
  const ProLayout Ly = pro_layout(K, m, F, k);
  double* lut = reinterpret_cast<double*>(dsm + Ly.lut64);
  float* lut32 = reinterpret_cast<float*>(dsm + Ly.lut32);
  double* he = reinterpret_cast<double*>(dsm + Ly.he);
  double* hf = reinterpret_cast<double*>(dsm + Ly.hf);
  int32_t* hi = reinterpret_cast<int32_t*>(dsm + Ly.hi);
  double* cf = reinterpret_cast<double*>(dsm + Ly.cf);
  double* ce = reinterpret_cast<double*>(dsm + Ly.ce);
  int32_t* cid = reinterpret_cast<int32_t*>(dsm + Ly.cid);
  int32_t* wsum = reinterpret_cast<int32_t*>(dsm + Ly.ctrl);          // [8]
  volatile float* pub_lo = reinterpret_cast<volatile float*>(dsm + Ly.ctrl + 64);
  volatile float* pub_hi = reinterpret_cast<volatile float*>(dsm + Ly.ctrl + 68);
  volatile int32_t* flag = reinterpret_cast<volatile int32_t*>(dsm + Ly.ctrl + 72);
  volatile double* pub_thr = reinterpret_cast<volatile double*>(dsm + Ly.ctrl + 80);
  int* nL_total = reinterpret_cast<int*>(dsm + Ly.ctrl + 92);  // block items under the list bound
  int* band_total = reinterpret_cast<int*>(dsm + Ly.ctrl + 96);  // near-ties seen by the prefilter
  volatile float* pub_hiL = reinterpret_cast<volatile float*>(dsm + Ly.ctrl + 120);  // list bound hi
  const long long t0 = clock64();

  // 1. float64 LUT -> smem, float32 copy of the fast books (prefilter)
  const double* glut = p.lut64 + (size_t)q * K * m;
  for (int i = tid; i < K * m; i += kProThreads) lut[i] = glut[i];
  bool bad = false;
  for (int i = tid; i < F * m; i += kProThreads) {
    const int s = i / m, j = i - s * m;
    const double x = glut[p.fast_books[s] * m + j];
    // float32 certification needs finite entries with headroom; otherwise
    // the query runs in float64 only ("wide" mode)
    bad |= !(x <= 1.2676506002282294e30);  // 2^100 (also catches NaN)
    lut32[i] = __double2float_rn(x);
  }
  const bool wide = __syncthreads_or(bad) != 0;

  RCtx c;
  c.lut = lut;
  c.codes_full = p.codes_full;
  c.fb = p.fast_books;
  c.KP = p.KP; c.m = m; c.K = K; c.F = F; c.k = k;
  c.sigma = p.sigma;
  c.f32 = f32s;
  c.pw = n == 1;  // numpy row-sum order, see ref_row_sum
  c.wide = wide;
  c.surv = p.survivors ? p.survivors + (int64_t)q * p.words : nullptr;

  // 2. seeds: ids 0..k-1 scored exactly (search.py:141), sorted descending
  //    by (exact, id) -> the sorted array is a valid max-heap.
  constexpr int kSeedPer = 8;
  double se[kSeedPer], sf[kSeedPer];
  int32_t sr[kSeedPer];
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kProThreads;
    if (i < k) {
      const Row row = load_row(p.codes_full, p.KP, i);
      se[r] = exact64(lut, m, K, c.pw, row);
      sf[r] = fast64(lut, m, F, c.pw, p.fast_books, row);
      he[i] = se[r];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kProThreads;
    if (i < k) {
      int rank = 0;
      for (int j = 0; j < k; ++j) rank += key_gt(he[j], j, se[r], i) ? 1 : 0;
      sr[r] = rank;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kProThreads;
    if (i < k) {
      he[sr[r]] = se[r];
      hf[sr[r]] = sf[r];
      hi[sr[r]] = i;
    }
  }
  __syncthreads();

  // the list threshold theta the filter would get if the prologue ended here
  // (A_J + sigma over the current heap, sorted descending by (exact, id))
  auto list_theta = [&](int lane_) -> double {
    const double A = heap_AJ(hf, k, p.list_j, lane_, nullptr);
    return thr_cover(A, p.sigma, f32s, false);
  };
  int64_t refinements = 0, insertions = 0;
  double smin = 0.0;
  if (warp == 0) {
    smin = p.sigma == 0.0 ? 0.0 : smin_rd(lut, K, m, p.fast_books, F, lane);
    const StaleThr t = stale_from_heap(he, hf, k, F, p.sigma, smin, wide, f32s, lane);
    float lL = kInf, hL = kInf;
    certified_bounds(list_theta(lane), F, lL, hL);
    if (lane == 0) {
      *pub_lo = t.lo; *pub_hi = t.hi; *pub_thr = t.thr; *flag = k < n ? 1 : 0;
      *band_total = 0;
      *pub_hiL = p.pro_live ? hL : t.hi;
      *nL_total = 0;
    }
  }
  __syncthreads();

  // the heap: the seeds' sorted array, held by warp 0 as a WarpHeap
  // (registers for k <= 128, else the shared-memory array itself)
  WarpHeap H;
  H.k = k;
  H.reg = k <= 32 * kRegHeapRegs;
  H.he = he;
  H.hf = hf;
  H.hi = hi;
  if (warp == 0) H.load(lane);

  // 3. blocks of kProBlock items in database order
  int64_t pos = k;
  int64_t pro_cand = 0;
  long long tp[3] = {0, 0, 0};
  int64_t nblocks = 0;
  while (*flag == 1) {
    const long long ta = clock64();
    ++nblocks;
    const int64_t base = (pos / kProBlock) * kProBlock;
    const int64_t bend = min(n, base + kProBlock);
    const float h = *pub_hi, hl = *pub_lo;
    const double hthr = *pub_thr;
    const float hL = *pub_hiL;
    // 3a. fp32 prefilter of 8 consecutive items per thread (codes_fast rows)
    const int64_t i0 = base + (int64_t)tid * 8;
    uint32_t w[2 * FP];
    {
      // 8 consecutive items = FP/2 logical chunks (half of one for FP == 1)
      // of the tile-transposed fast rows
      if (FP == 1) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p.codes_fast + perm_offset(1, i0)));
        w[0] = v.x; w[1] = v.y;
      } else {
        constexpr int kIpc = 16 / (FP > 1 ? FP : 1);
#pragma unroll
        for (int t = 0; t < FP / 2; ++t) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.codes_fast) +
                                perm_chunk(i0 / kIpc + t));
          w[4 * t] = v.x; w[4 * t + 1] = v.y; w[4 * t + 2] = v.z; w[4 * t + 3] = v.w;
        }
      }
    }
    uint32_t mask = 0;
    int nband = 0;  // items float32 could not decide (near / exact ties with the threshold)
    int nl = 0;     // items under the list bound (how long the filter's lists would be)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float x = 0.f;
#pragma unroll
      for (int s = 0; s < FP; ++s) {
        const int b = j * FP + s;
        const uint32_t code = (w[b >> 2] >> ((b & 3) * 8)) & 0xffu;
        if (s < F) x += lut32[s * m + code];
      }
      const int64_t i = i0 + j;
      bool cand = wide || x < hl;
      if (!cand && x < h) {  // float32 cannot decide: exact float64 fast score
        nband += (i0 + j >= pos) & (i0 + j < bend);
        double d = 0.0;
#pragma unroll
        for (int s = 0; s < FP; ++s) {
          const int b = j * FP + s;
          const uint32_t code = (w[b >> 2] >> ((b & 3) * 8)) & 0xffu;
          if (s < F) d = __dadd_rn(d, lut[p.fast_books[s] * m + code]);
        }
        cand = d < hthr;
      }
      mask |= ((i >= pos) & (i < bend) & cand) ? (1u << j) : 0u;
      nl += (i >= pos) & (i < bend) & (x < hL);
    }
    // 3b. ordered compaction (thread order = item order)
    if (nband) atomicAdd(band_total, nband);
    if (nl) atomicAdd(nL_total, nl);
    const int cnt = __popc(mask);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int off = incl - cnt, ncand = 0;
#pragma unroll
    for (int t = 0; t < kProThreads / 32; ++t) {
      const int v = wsum[t];
      off += t < warp ? v : 0;
      ncand += v;
    }
    while (mask) {
      const int j = __ffs(mask) - 1;
      mask &= mask - 1;
      cid[off++] = (int32_t)(i0 + j);
    }
    __syncthreads();
    const long long tb = clock64();
    // 3c. float64 fast/exact scores of the prefiltered items (rows from L2/HBM)
    {
      Row rows[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int ci = tid + r * kProThreads;
        if (ci < ncand) rows[r] = load_row(p.codes_full, p.KP, cid[ci]);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int ci = tid + r * kProThreads;
        if (ci < ncand) {
          cf[ci] = fast64(lut, m, F, c.pw, p.fast_books, rows[r]);
          ce[ci] = exact64(lut, m, K, c.pw, rows[r]);
        }
      }
    }
    pro_cand += ncand;
    __syncthreads();
    const long long tc = clock64();
    // 3d. warp 0 applies search.py:148-154 in order (float64 compares), 32
    //     candidates per window: refine iff fast < bound + sigma, insert iff
    //     exact < T.  The first inserting lane ends the window's decided
    //     prefix (the bound moves there); the lanes after it are re-tested
    //     against the new bound.  The heap is the sorted-array WarpHeap.
    const int64_t ref_before = refinements, ins_before = insertions;
    if (warp == 0) {
      double T = H.top_e();
      double thr = live_thr(H.top_f(), H.top_i(), p.sigma, k, f32s);
      for (int c0 = 0; c0 < ncand; c0 += 32) {
        const int ci = c0 + lane;
        const bool ok = ci < ncand;
        const double fv = ok ? cf[ci] : 0.0;
        const double ev = ok ? ce[ci] : 0.0;
        const int32_t id = ok ? cid[ci] : 0;
        uint32_t pending = __ballot_sync(kFull, ok);
        while (pending) {
          const bool mine = (pending >> lane) & 1u;
          const bool ref = mine && fv < thr;
          const bool ins = ref && ev < T;
          const uint32_t im = __ballot_sync(kFull, ins);
          const int first = im ? __ffs(im) - 1 : 31;
          const uint32_t decided = pending & (first == 31 ? kFull : ((2u << first) - 1u));
          const uint32_t rm = __ballot_sync(kFull, ref) & decided;
          refinements += __popc(rm);
          if ((rm >> lane) & 1u) record_survivor(c.surv, id);
          pending &= ~decided;
          if (!im) break;
          const double ne = __shfl_sync(kFull, ev, first);
          const double nf = __shfl_sync(kFull, fv, first);
          const int32_t nid = __shfl_sync(kFull, id, first);
          H.replace_max(ne, nid, nf, lane);
          T = H.top_e();
          thr = live_thr(H.top_f(), H.top_i(), p.sigma, k, f32s);
          ++insertions;
        }
      }
      H.store(lane);  // smem copy for the thresholds below and the hand-off
    }
    __syncwarp();
    if (warp == 0) {
      const StaleThr tn = stale_from_heap(he, hf, k, F, p.sigma, smin, wide, f32s, lane);
      // the heap array is sorted descending by (exact, id) (WarpHeap.store)
      float lL = kInf, hLn = kInf;
      if (p.pro_live) certified_bounds(list_theta(lane), F, lL, hLn);
      const int64_t nb = bend - max(pos, base);
      bool more = bend < n && bend < p.pro_max;
      // stop once the filter's lists would be short: the block's items under
      // the list bound theta (pro_live) or under the stale M are <= 1/pro_div
      if (bend >= p.pro_min) {
        const int64_t nX = p.pro_live ? (int64_t)(*nL_total) : (int64_t)ncand;
        if (nX * p.pro_div <= nb) more = false;
      }
      // refinement-heavy: the live threshold itself passes > 1/count_div of
      // the block, at that rate the rest of the database would list >
      // count_min items, and the refinements are not just the insertions of
      // a young heap (those decay as k / position; at small sigma a good part
      // of the refined items is inserted: > 16 refinements per insertion
      // means a near-exact heap, hence a tight T).  Such a query leaves the
      // prologue here, in
      // count mode (after optional count-style blocks, phase 2 below).
      bool heavy = false;
      if (FP <= 8 && p.count_used && !wide && bend < n && bend >= p.pro_min) {
        const int64_t rb = refinements - ref_before, ib = insertions - ins_before;
        heavy = p.force_count != 0 ||
                (p.count_div > 0 && rb * p.count_div > nb && rb > 16 * ib &&
                 (double)rb * (double)(n - bend) > (double)p.count_min * (double)nb);
      }
      if (lane == 0) {
        *pub_lo = tn.lo; *pub_hi = tn.hi; *pub_thr = tn.thr;
        *pub_hiL = p.pro_live ? hLn : tn.hi;
        *nL_total = 0;
        *flag = heavy ? 2 : (more ? 1 : 0);
      }
    }
    __syncthreads();
    pos = bend;
    tp[0] += tb - ta;
    tp[1] += tc - tb;
    tp[2] += clock64() - tc;
  }

  // 3'. phase 2 (refinement-heavy queries): blocks in count style.  Only items
  //     with exact < T can be inserted, so a block is pre-filtered by the
  //     float32 exact sum of ALL books (certified against hiT, K terms) -- a
  //     handful of items per block instead of the refined third of it -- and
  //     warp 0 decides those in order, recording the live threshold after
  //     every insertion.  Refinements and survivor bits of [P0, n) come from
  //     the count kernel.  Much cheaper per item than phase 1, so it runs
  //     longer (pro_max_cm) and hands the filter a tighter T.
  const bool phase2 = *flag == 2;  // (CTA-uniform: read after the loop's last barrier)
  int64_t P0 = pos;
  double thr0_cm = 0.0;
  int32_t ntraj = 0;
  __syncthreads();
  if (phase2) {
    float* lut32k = reinterpret_cast<float*>(dsm + Ly.lut32k);
    volatile float* pub_hiT = reinterpret_cast<volatile float*>(dsm + Ly.ctrl + 100);
    stage_lut32k(lut32k, lut, K, p.KP, m, tid, kProThreads);
    TrajEntry* traj = p.traj + (size_t)q * kMaxTraj;
    if (warp == 0) {
      thr0_cm = live_thr(H.top_f(), H.top_i(), p.sigma, k, f32s);
      float loT, hT;
      certified_bounds(H.top_e(), K, loT, hT);
      if (lane == 0) *pub_hiT = hT;
    }
    __syncthreads();
    while (pos < n && pos < p.pro_max_cm) {
      ++nblocks;
      const int64_t base = (pos / kProBlock) * kProBlock;
      const int64_t bend = min(n, base + kProBlock);
      const float hT = *pub_hiT;
      const int64_t i0 = base + (int64_t)tid * 8;
      Row rows[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) rows[j] = load_row(p.codes_full, p.KP, i0 + j);  // (padded rows)
      uint32_t mask = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float e = exact32_any(lut32k, m, p.KP, rows[j]);
        const int64_t i = i0 + j;
        mask |= ((i >= pos) & (i < bend) & (e < hT)) ? (1u << j) : 0u;
      }
      const int cnt = __popc(mask);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      int off = incl - cnt, ncand = 0;
#pragma unroll
      for (int t = 0; t < kProThreads / 32; ++t) {
        const int v = wsum[t];
        off += t < warp ? v : 0;
        ncand += v;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if ((mask >> j) & 1u) {
          cf[off] = fast64(lut, m, F, c.pw, p.fast_books, rows[j]);
          ce[off] = exact64(lut, m, K, c.pw, rows[j]);
          cid[off] = (int32_t)(i0 + j);
          ++off;
        }
      }
      pro_cand += ncand;
      __syncthreads();
      if (warp == 0 && ncand > 0) {
        double T = H.top_e();
        double thr = live_thr(H.top_f(), H.top_i(), p.sigma, k, f32s);
        for (int c0 = 0; c0 < ncand; c0 += 32) {
          const int ci = c0 + lane;
          const bool ok = ci < ncand;
          const double fv = ok ? cf[ci] : 0.0;
          const double ev = ok ? ce[ci] : 0.0;
          const int32_t id = ok ? cid[ci] : 0;
          uint32_t pending = __ballot_sync(kFull, ok);
          while (pending) {
            const bool mine = (pending >> lane) & 1u;
            const bool ins = mine && fv < thr && ev < T;
            const uint32_t im = __ballot_sync(kFull, ins);
            if (!im) break;
            const int first = __ffs(im) - 1;
            pending &= ~((2u << first) - 1u);
            const double ne = __shfl_sync(kFull, ev, first);
            const double nf = __shfl_sync(kFull, fv, first);
            const int32_t nid = __shfl_sync(kFull, id, first);
            H.replace_max(ne, nid, nf, lane);
            T = H.top_e();
            thr = live_thr(H.top_f(), H.top_i(), p.sigma, k, f32s);
            ++insertions;
            if (lane == 0) {  // items after nid are refined against the new threshold
              if (ntraj < kMaxTraj) traj[ntraj] = TrajEntry{(int64_t)nid, thr};
              else atomicOr(p.error, 16);
            }
            ++ntraj;
          }
        }
        float loT, hTn;
        certified_bounds(T, K, loT, hTn);
        if (lane == 0) *pub_hiT = hTn;
      }
      __syncthreads();
      pos = bend;
    }
    if (warp == 0) H.store(lane);
    __syncthreads();
  }

  // 4. hand the state to the filter / replay kernels: the heap sorted
  //    descending by (exact, id) (WarpHeap.store keeps the array sorted), and
  //    the list threshold theta = A_J + sigma (A_J: max fast over the J+1
  //    largest-exact entries; J = 0 makes theta the live threshold itself).
  //    The filter lists every later item with fast < theta; the replay walks
  //    the database in order wherever the live threshold rises above theta.
  __syncthreads();
  // 4a. the list threshold: theta_J = A_J + sigma for J on a ladder; the
  //     loosest one whose share of the last <= 16k prologue items stays
  //     <= 1/list_div (the items after P come from the same stream).  Loose
  //     lists cost list entries (cheap, filtered on every SM), tight ones
  //     cost walks whenever the live threshold rises above theta (in order,
  //     one CTA).  ICQ_LIST_J >= 0 fixes J.
  int listJ = p.list_j;
  bool count_mode = FP <= 8 && (p.force_count != 0 || phase2) && !wide && (pos < n || phase2);
  if (!phase2 && (listJ < 0 || p.count_div > 0)) {
    // (rungs 0..8: theta_J; rung 9: T - Smin, what count mode would list)
    constexpr int kLad = 10;
    const int ladder[kLad] = {0, 1, 2, 4, 8, 16, 32, 64, 1 << 30, 0};
    float* lad_hi = reinterpret_cast<float*>(cf);        // (cf/ce are free now)
    int* lad_cnt = reinterpret_cast<int*>(cf + 16);
    if (warp == 0) {
      for (int r = 0; r < kLad - 1; ++r) {
        const double A = heap_AJ(hf, k, min(ladder[r], k - 1), lane, nullptr);
        float lo_ = kInf, hi_ = kInf;
        certified_bounds(thr_cover(A, p.sigma, f32s, false), F, lo_, hi_);
        if (lane == 0) { lad_hi[r] = hi_; lad_cnt[r] = 0; }
      }
      float lo_ = kInf, hi_ = kInf;
      if (FP <= 8 && p.count_div > 0) {
        const double sm = smin_rd(lut, K, m, p.fast_books, F, lane);
        const double T = he[0];
        certified_bounds(__dadd_ru(__dsub_ru(T, sm), fabs(T) * 1e-12), F, lo_, hi_);
      }
      if (lane == 0) { lad_hi[kLad - 1] = hi_; lad_cnt[kLad - 1] = 0; }
    }
    __syncthreads();
    int64_t S = (pos - k) / kProBlock * kProBlock;
    if (S > 8 * kProBlock) S = 8 * kProBlock;
    if (wide || pos >= n) S = 0;
    int cnt[kLad];
#pragma unroll
    for (int r = 0; r < kLad; ++r) cnt[r] = 0;
    for (int64_t i0 = pos - S + (int64_t)tid * 8; i0 < pos; i0 += kProThreads * 8) {
      uint32_t w[2 * FP];
      if (FP == 1) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p.codes_fast + perm_offset(1, i0)));
        w[0] = v.x; w[1] = v.y;
      } else {
        constexpr int kIpc = 16 / (FP > 1 ? FP : 1);
#pragma unroll
        for (int t = 0; t < FP / 2; ++t) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(p.codes_fast) + perm_chunk(i0 / kIpc + t));
          w[4 * t] = v.x; w[4 * t + 1] = v.y; w[4 * t + 2] = v.z; w[4 * t + 3] = v.w;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float x = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < FP; ++s2) {
          const int b = j * FP + s2;
          const uint32_t code = (w[b >> 2] >> ((b & 3) * 8)) & 0xffu;
          if (s2 < F) x += lut32[s2 * m + code];
        }
#pragma unroll
        for (int r = 0; r < kLad; ++r) cnt[r] += x < lad_hi[r] ? 1 : 0;
      }
    }
#pragma unroll
    for (int r = 0; r < kLad; ++r) {
      const int c2 = __reduce_add_sync(kFull, cnt[r]);
      if (lane == 0 && c2) atomicAdd(&lad_cnt[r], c2);
    }
    __syncthreads();
    if (p.list_j < 0) {
      listJ = 0;
      for (int r = 0; r < kLad - 1; ++r)
        if (S > 0 && (int64_t)lad_cnt[r] * p.list_div <= S) listJ = ladder[r];
    }
    listJ = min(listJ, k - 1);
    // refinement-heavy: even the live threshold passes > 1/count_div of the
    // sample -> the lists would hold the refined items themselves.  Count
    // mode lists the items under T - Smin instead, which only pays while
    // that bound is selective (a poor heap -- small sigma, low recall --
    // leaves T loose: <= 1/8 of the sample, else the query stays in list mode)
    if (FP <= 8 && p.count_div > 0 && S > 0 && (int64_t)lad_cnt[0] * p.count_div > S &&
        (double)lad_cnt[0] * (double)(n - pos) > (double)p.count_min * (double)S &&
        (int64_t)lad_cnt[kLad - 1] * 8 <= S)
      count_mode = true;
    __syncthreads();
  }
  if (warp == 0) {
    int best = 0;
    const double A = heap_AJ(hf, k, listJ, lane, &best);
    double thr = wide ? kInf64 : thr_cover(A, p.sigma, f32s, false);
    float hiT = kInf;
    double smin_cm = 0.0;
    if (count_mode) {
      // the lists keep every possible insertion, whatever sigma: an item
      // inserted later has exact < T_P (T never increases), hence
      // fast < T_P - Smin (its slow part is >= Smin); float64 slack for the
      // different summation orders of fast and exact scores
      const double sm = smin_rd(lut, K, m, p.fast_books, F, lane);
      smin_cm = sm;
      const double T = he[0];
      thr = __dadd_ru(__dsub_ru(T, sm), fabs(T) * 1e-12);
      float loT;
      certified_bounds(T, K, loT, hiT);
    }
    float flo = kInf, fhi = kInf;
    if (!wide) certified_bounds(thr, F, flo, fhi);
    // tie rejection costs the filter a tuple compare per candidate: enabled
    // only where the prologue saw near-ties in bulk (few-codeword books);
    // items with the threshold item's fast-code tuple tie at thr exactly
    const bool ties = (int64_t)(*band_total) * 2048 > pos && !(p.debug & 1);
    const bool ok = ties && FP <= 8 && p.sigma == 0.0 && !f32s && !wide && !count_mode;
    uint2 tup = make_uint2(0u, 0u);
    if (ok && lane == 0) {
      const Row r = load_fast_row(p.codes_fast, FP, hi[best]);
      tup = make_uint2(r.w[0], r.w[1]);
    }
    if (lane == 0) {
      QState st;
      st.P = pos;
      st.refinements = refinements;
      st.insertions = insertions;
      st.pro_cand = pro_cand;
      st.pro_cycles = clock64() - t0;
      st.pro_t[0] = tp[0];
      st.pro_t[1] = tp[1];
      st.pro_t[2] = tp[2];
      st.pro_t[3] = nblocks;
      st.hi = fhi;
      st.lo = flo;
      st.thr = thr;
      st.mtup[0] = tup.x;
      st.mtup[1] = tup.y;
      st.mt_valid = ok ? 1 : 0;
      st.wide = wide ? 1 : 0;
      st.done = 0;
      st.rounds = 0;
      st.walked = 0;
      st.count_mode = count_mode ? 1 : 0;
      st.hiT = hiT;
      st.smin = smin_cm;
      st.ntraj = ntraj;
      st.thr0 = phase2 ? thr0_cm : live_thr(hf[0], hi[0], p.sigma, k, f32s);
      st.P0 = P0;
      st.ovf_pages = 0;
      st.ovf_pool = 0;
      st.skipped = 0;
      st.listed_raw = 0;
      // count mode: the first round lists a prefix only; the replay hands the
      // rest to the next round with the heap (and T) it has by then
      st.list_end = (count_mode && p.rounds >= 2 && pos < p.cm_prefix) ? min(p.cm_prefix, n) : n;
      st.dense = st.list_end < n ? 1 : 0;  // (FP <= 8: count mode)
      st.cm_end = n;
      p.qs[q] = st;
      if (count_mode) p.cm_list[1 + atomicAdd(p.cm_list, 1)] = q;
    }
  }
  for (int i = tid; i < k; i += kProThreads) {
    p.heap_e[(size_t)q * k + i] = he[i];
    p.heap_f[(size_t)q * k + i] = hf[i];
    p.heap_i[(size_t)q * k + i] = hi[i];
  }
}

// Drop, in place and in order, the entries of one slice that cannot be
// inserted: float32 exact sum e32 >= hiT (exact64 < T implies e32 < hiT).
// One warp; lut32k: the float32 table [KP][m] (zero rows for b >= K).  Returns
// the number of entries kept.
__device__ __forceinline__ int refine_slice(uint4* pool, const int32_t* slice, int cnt,
                                            const uint8_t* codes_full, int KP, int m, float hiT,
                                            int lane, const float* lut32k) {
  const uint32_t lt = (1u << lane) - 1u;
  int w = 0;  // entries kept so far (write position <= read position: in place)
  constexpr int U = kPG / 32;
  for (int pi = 0; pi * kPG < cnt; ++pi) {
    const uint4* src = pool + ((size_t)(uint32_t)slice[1 + pi] << 7);
    uint4 ent[U];
    Row rows[U];
    bool valid[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      valid[u] = pi * kPG + u * 32 + lane < cnt;
      ent[u] = valid[u] ? src[u * 32 + lane] : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) rows[u] = load_row(codes_full, KP, (int64_t)ent[u].x);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float e = exact32_any(lut32k, m, KP, rows[u]);
      const bool keep = valid[u] && e < hiT;
      const uint32_t km = __ballot_sync(kFull, keep);
      if (keep) ent[u].y = (uint32_t)(w + __popc(km & lt));  // (write position)
      valid[u] = keep;
      w += __popc(km);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (valid[u]) {
        const int wp = (int)ent[u].y;
        pool[((size_t)(uint32_t)slice[1 + (wp >> 7)] << 7) | (uint32_t)(wp & (kPG - 1))] =
            make_uint4(ent[u].x, 0u, ent[u].z, ent[u].w);
      }
    }
  }
  return w;
}
// ==========================================================================
// K3: filter (the streaming hot path)
// ==========================================================================
template <int FP>
struct FGeo {
  static constexpr int R = FP <= 4 ? 32 : (FP == 8 ? 16 : 8);  // replicas per entry
  static constexpr int BPR = 64 / R;                             // book slots per 256-B row
  static constexpr int P = (FP + BPR - 1) / BPR;                 // 64 KiB pages
  static constexpr int IPC = 16 / FP;                            // items per 16-B chunk
  static constexpr int V = 4;                                    // chunks per lane per tile
  static constexpr int TILE = 32 * V * IPC;                      // items per warp tile
  static constexpr uint32_t kSmemEnd = kPage * (1 + P);          // absolute end of the pages
};
constexpr int kPrefetchTiles = ICQ_PREFETCH_TILES;  // L2 bulk-prefetch distance (tiles; 0 = off)

template <int FP>
__global__ void __launch_bounds__(kFW * 32, 1) icq_filter_kernel(const __grid_constant__ PipeParams p) {
  using G = FGeo<FP>;
  constexpr int IPC = G::IPC, V = G::V, TILE = G::TILE;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // The lane-private pages sit at absolute 64 KiB boundaries; the planned
  // layout assumes the dynamic window starts at kDynBase.
  uint32_t dyn_size;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_size));
  const uint32_t dbase = smem_addr(dsm);
  if (dbase != kDynBase || dbase + dyn_size < G::kSmemEnd) {
    if (tid == 0) atomicExch(p.error, 1);
    return;
  }
  // page address template of fast book s for this lane: (page << 16) | lane offset;
  // byte 1 (the codeword) is filled in by one byte_perm per lookup
  uint32_t Lp[FP];
#pragma unroll
  for (int s = 0; s < FP; ++s)
    Lp[s] = ((uint32_t)(1 + s / G::BPR) << 16) |
            (uint32_t)((s % G::BPR) * 4 * G::R + (lane % G::R) * 4);

  if (p.round > 0 && p.round_cnt[p.round] == 0) return;  // no query was handed to this round
  const int K = p.K, m = p.m, F = p.F;
  const int64_t RS = p.RS, SW = p.RS / kFW;
  const int64_t U = (int64_t)p.Q * p.NR;
  int64_t u0, u1, ustep;
  const bool rmaj = p.range_major != 0 || p.round > 0;
  const bool rmaj_stream = p.range_major != 0;
  if (rmaj) {  // all CTAs sweep the ranges together: codes reused in L2 (and in later
               // rounds the few unfinished queries spread over all SMs)
    u0 = blockIdx.x; u1 = U; ustep = gridDim.x;
  } else {     // contiguous unit blocks: one query's LUT serves many units
    u0 = U * blockIdx.x / gridDim.x; u1 = U * (blockIdx.x + 1) / gridDim.x; ustep = 1;
  }
  const uint4* codes = reinterpret_cast<const uint4*>(p.codes_fast);
  double* lut64f = reinterpret_cast<double*>(dsm);  // [F][m] below the first page
#if !ICQ_MASK_SHF
  const uint32_t two = 2u + (uint32_t)(p.n < 0);    // 2, opaque to the compiler (keeps IMADs)
#endif
  const uint32_t lt_mask = (1u << lane) - 1u;
  int cur_q = -1;
  for (int64_t u = u0; u < u1; u += ustep) {
    const int q = rmaj ? (int)(u % p.Q) : (int)(u / p.NR);
    const int r = rmaj ? (int)(u / p.Q) : (int)(u % p.NR);
    const int64_t P = p.qs[q].P;
    const float hi = p.qs[q].hi;
    const double thr = p.qs[q].thr;  // (FP = 16 entries carry the float64 fast score)
    (void)thr;
    const uint2 mtup = make_uint2(p.qs[q].mtup[0], p.qs[q].mtup[1]);
    const bool mt_valid = p.qs[q].mt_valid != 0;
    const int wide = p.qs[q].wide;
    // (a count-mode query first lists a prefix [P, list_end) only: its replay
    // hands the rest to the next round with a much tighter T)
    const int64_t lend = p.qs[q].list_end;
    const int64_t r_lo = (int64_t)r * RS, r_hi = min(lend, r_lo + RS);
    int32_t* slice = p.slices + ((int64_t)(q * p.NR + r) * kFW + warp) * kSliceInts;
    if (P >= r_hi || p.qs[q].done || p.qs[q].dense) {  // decided by the prologue / an earlier
                                                          // round / later / the dense kernel
      if (lane == 0) slice[0] = 0;
      continue;
    }
    if (wide) {  // float64 only: the replay rescans these slices
      if (lane == 0) slice[0] = -1;
      continue;
    }
    if (q != cur_q) {
      __syncthreads();  // every warp is done with the previous query's pages
      const double* glut = p.lut64 + (size_t)q * K * m;
      // one table entry per thread and pass (a single L2 read), written to
      // its R lane replicas with 16-byte stores
      for (int i = tid; i < FP * m; i += kFW * 32) {
        const int s = i / m, j = i - s * m;
        const float v = s < F ? __double2float_rn(glut[p.fast_books[s] * m + j]) : 0.f;
        const uint32_t a0 = kPage * (1 + s / G::BPR) + j * 256 + (s % G::BPR) * 4 * G::R;
#pragma unroll
        for (int rr = 0; rr < G::R; rr += 4) sts_f32x4(a0 + rr * 4, v);
      }
      for (int i = tid; i < F * m; i += kFW * 32) {  // float64 fast tables (near-ties)
        const int s = i / m, j = i - s * m;
        lut64f[i] = glut[p.fast_books[s] * m + j];
      }
      __syncthreads();
      cur_q = q;
    }
    const int64_t w_lo = r_lo + warp * SW;
    const int64_t w_hi = min(w_lo + SW, lend);
    const int64_t start = max(w_lo, P);
    if (start >= w_hi) {
      if (lane == 0) slice[0] = 0;
      continue;
    }
    int cnt = 0, npages = 0, cur_page = 0;
    bool overflow = false;
    // exact float64 fast score of item j of a code chunk, reference order
    auto fast_f64 = [&](const uint4& xv, int j) -> double {
      if constexpr (FP <= 8) {
        return tuple_f64<FP>(chunk_tuple<FP>(xv, j), lut64f, m, F);
      } else {
        const uint32_t wd[4] = {xv.x, xv.y, xv.z, xv.w};
        double d = 0.0;
#pragma unroll
        for (int s = 0; s < FP; ++s)
          if (s < F) d = __dadd_rn(d, lut64f[s * m + ((wd[s >> 2] >> (8 * (s & 3))) & 0xffu)]);
        return d;
      }
    };
    int64_t t = w_lo + ((start - w_lo) / TILE) * TILE;
    // 32-bit tile counters and a running chunk pointer (no 64-bit index math per tile)
    // tile-transposed rows: the coalesced load of physical chunks 32 v + lane
    // gives lane l the logical chunks 4 l .. 4 l + 3 of the tile, one
    // contiguous id run, so an ordered append is a single lane scan
    static_assert(V == 4, "the tile-transposed layout assumes 4 chunks per lane");
    const uint4* cptr = codes + t / IPC + lane;
    const int ntile = (int)((w_hi - t + TILE - 1) / TILE);
    // tiles [it_full0, it_full1) lie wholly inside [start, w_hi)
    const int it_full0 = t < start ? 1 : 0;
    const int it_full1 = t + (int64_t)ntile * TILE > w_hi ? ntile - 1 : ntile;
    uint4 a[V];
#pragma unroll
    for (int v = 0; v < V; ++v) a[v] = ldg_stream(cptr + v * 32);
#pragma unroll 2
    for (int it = 0; it < ntile; ++it, t += TILE) {
      uint4 x[V];
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = a[v];
      cptr += TILE / IPC;
      if (it + 1 < ntile) {
#pragma unroll
        for (int v = 0; v < V; ++v) a[v] = ldg_stream(cptr + v * 32);
      }
      // L2 bulk prefetch kPrefetchTiles ahead, 4 tiles per request
      // (only for streams larger than L2: an L2-resident stream gains nothing
      // and the issue slots are the scarce resource there)
      if (kPrefetchTiles > 0 && rmaj_stream && lane == 0 && (it & 3) == 0 &&
          it + kPrefetchTiles + 4 <= ntile)
        prefetch_l2_bulk(cptr - lane + (kPrefetchTiles - 1) * (TILE / IPC), 4 * TILE * FP);
      // one warp tile: 32 lanes x V 16-byte chunks, items (v, lane, j).  The
      // fast sums of item pairs run packed (FADD2: two fp32 adds per issue,
      // each rounded as the scalar add, denormals kept), in the same tree order
      // the certified bounds assume; d = f - hi keeps the sign of f - hi
      // exactly (no flush), so d < 0 iff f < hi.
      constexpr int N = V * IPC;
      const float2 nhi2 = make_float2(-hi, -hi);
      float2 d2[N / 2];
#pragma unroll
      for (int pr = 0; pr < N / 2; ++pr) {
        float2 acc[FP];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int idx = 2 * pr + h, v = idx / IPC, j = idx % IPC;
          const uint32_t wd[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
#pragma unroll
          for (int s = 0; s < FP; ++s) {
            const int byte = j * FP + s;
            const uint32_t sel = 0x7604u | ((uint32_t)(byte & 3) << 4);
            const float val = lds_f32(__byte_perm(wd[byte >> 2], Lp[s], sel));
            if (h == 0) acc[s].x = val; else acc[s].y = val;
          }
        }
#pragma unroll
        for (int h = 1; h < FP; h *= 2)
#pragma unroll
          for (int s = 0; s + h < FP; s += 2 * h) acc[s] = __fadd2_rn(acc[s], acc[s + h]);
        d2[pr] = __fadd2_rn(acc[0], nhi2);
      }
      // candidate bits (bit v*IPC + j): d < 0.  Built on the FMA pipe (the
      // ALU pipe carries the byte_perm address of every lookup): the sign bit
      // of d is mul.hi(bits(d), 2), accumulated Horner-style (acc = acc * 2 +
      // s) with a runtime two.  Items whose fast-code tuple is the threshold
      // item's are dropped below (fast == thr exactly: never a candidate;
      // few-codeword books make such ties common).  The kept set is a
      // superset of the refined items; the replay decides exactly with the
      // float64 score of the tuple.
      using Mask = typename std::conditional<(N > 32), unsigned long long, uint32_t>::type;
      Mask cm = 0;
      if constexpr (N <= 32) {
        // four independent Horner chains (short dependency paths), then merged
        constexpr int NC = N >= 16 ? 4 : 1, L = N / NC;
        uint32_t acc[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          acc[c] = 0;
#pragma unroll
          for (int i = L - 1; i >= 0; --i) {
            const int idx = c * L + i;
            const float dd = (idx & 1) ? d2[idx >> 1].y : d2[idx >> 1].x;
#if ICQ_MASK_SHF
            acc[c] = __funnelshift_l(__float_as_uint(dd), acc[c], 1);  // (acc << 1) | sign(d)
#else
            acc[c] = acc[c] * two + __umulhi(__float_as_uint(dd), two);
#endif
          }
        }
        uint32_t mk = acc[0];
#pragma unroll
        for (int c = 1; c < NC; ++c) mk |= acc[c] << (c * L);
        cm = mk;
      } else {
#pragma unroll
        for (int idx = 0; idx < N; ++idx) {
          const float dd = (idx & 1) ? d2[idx >> 1].y : d2[idx >> 1].x;
          if (dd < 0.f) cm |= (Mask)1 << idx;
        }
      }
      if (!__any_sync(kFull, cm != 0)) continue;
      // ---- slow path (most tiles hold a candidate or two) ----
      if (it < it_full0 || it >= it_full1) {  // edge tile: keep items in [start, w_hi)
        const int lo_t = (int)(start - t), hi_t = (int)min((int64_t)TILE, w_hi - t);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int c0 = (lane * V + v) * IPC;  // first item of chunk v, relative to t
          const int a0 = min(max(lo_t - c0, 0), IPC), a1 = min(max(hi_t - c0, 0), IPC);
          const Mask keep = (a1 > a0) ? (((((Mask)1 << (a1 - a0)) - 1) << a0) << (v * IPC)) : (Mask)0;
          const Mask band = (((Mask)1 << IPC) - 1) << (v * IPC);
          cm &= ~band | keep;
        }
      }
      constexpr uint32_t kChunkBits = IPC >= 32 ? 0xffffffffu : ((1u << IPC) - 1u);
      if constexpr (FP <= 8) {
        if (mt_valid) {  // lane-parallel tie check over the few candidate bits
#pragma unroll
          for (int v = 0; v < V; ++v) {
            uint32_t b = (uint32_t)(cm >> (v * IPC)) & kChunkBits;
            while (b) {
              const int j = __ffs(b) - 1;
              b &= b - 1;
              const uint2 tj = chunk_tuple<FP>(x[v], j);
              if (tj.x == mtup.x && tj.y == mtup.y) cm &= ~((Mask)1 << (v * IPC + j));
            }
          }
        }
      }
      // positions: item order is (lane, v, j) -> an exclusive scan of the
      // per-lane counts; one ballot when no lane holds two
      const int mine = __popcll((unsigned long long)cm);
      const uint32_t has = __ballot_sync(kFull, mine != 0);
      int excl, T;
      if (!__any_sync(kFull, mine > 1)) {
        excl = __popc(has & lt_mask);
        T = __popc(has);
      } else {
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, incl, o);
          if (lane >= o) incl += y;
        }
        excl = incl - mine;
        T = __shfl_sync(kFull, incl, 31);
      }
      if (T == 0) continue;
      const int need = (cnt + T + kPG - 1) / kPG - npages;
      int base_pg = 0;
      if (!overflow && need > 0) {
        // (count-mode slices may list every item: the replay reads them through
        // the contiguous list, not through the staged page table)
        if (npages + need > (p.qs[q].count_mode ? p.max_pages_cm : p.max_pages)) {
          overflow = true;
          if (lane == 0) atomicAdd(&p.qs[q].ovf_pages, 1);
        } else {
          if (lane == 0) base_pg = atomicAdd(p.pool_top, need);
          base_pg = __shfl_sync(kFull, base_pg, 0);
          if ((int64_t)base_pg + need > p.pool_pages) {
            overflow = true;
            if (lane == 0) atomicAdd(&p.qs[q].ovf_pool, 1);
          } else if (lane < need) {
            slice[1 + npages + lane] = base_pg + lane;
          }
        }
      }
      if (overflow) {  // the replay rescans this slice: stop streaming it
        if (lane == 0) atomicAdd((unsigned long long*)&p.qs[q].skipped,
                                 (unsigned long long)max((int64_t)0, w_hi - (t + TILE)));
        break;
      } else {
        int gg = cnt + excl;
        // ids fit 32 bits (n < 2^31); chunk v of this lane starts at idb + v*IPC
        const uint32_t idb = (uint32_t)t + (uint32_t)(lane * N);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          uint32_t b = (uint32_t)(cm >> (v * IPC)) & kChunkBits;
          while (b) {
            const int j = __ffs(b) - 1;
            b &= b - 1;
            uint2 tail;
            if constexpr (FP <= 8) {
              tail = chunk_tuple<FP>(x[v], j);
            } else {
              const unsigned long long db = (unsigned long long)__double_as_longlong(fast_f64(x[v], j));
              tail = make_uint2((uint32_t)db, (uint32_t)(db >> 32));
            }
            const int pi = gg >> 7;
            const int pid = pi < npages ? cur_page : base_pg + (pi - npages);
            p.pool[((size_t)(uint32_t)pid << 7) | (uint32_t)(gg & (kPG - 1))] =
                make_uint4(idb + (uint32_t)(v * IPC + j), 0u, tail.x, tail.y);
            ++gg;
          }
        }
        if (need > 0) {
          npages += need;
          cur_page = base_pg + need - 1;
        }
      }
      cnt += T;
    }
    if (lane == 0) slice[0] = overflow ? -1 : cnt;
  }
}

// ==========================================================================
// K3a: dense prefix (count-mode queries, first round)
// ==========================================================================
// A count-mode query leaves the prologue early, with a loose heap: T - Smin
// would pass nearly every item.  Its first round therefore covers a prefix
// [P, list_end) only, and lists it here without the fast test: every SM reads
// the prefix rows (coalesced) and keeps the items whose float32 exact sum is
// under hiT (the only ones that can be inserted), in order, into the same
// paged slices the filter fills.  The replay decides them and hands the rest
// of the database to the next round with a tight T.
template <int FP>
__global__ void __launch_bounds__(kFW * 32) icq_dense_kernel(const __grid_constant__ PipeParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  float* lut32k = reinterpret_cast<float*>(dsm);  // [K][m]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = (int)(blockIdx.x % (unsigned)p.Q), r = (int)(blockIdx.x / (unsigned)p.Q);
  if (!p.qs[q].dense || p.qs[q].done) return;  // (CTA-uniform)
  const int64_t lend = p.qs[q].list_end, P = p.qs[q].P;
  const int64_t r_lo = (int64_t)r * p.RS, r_hi = min(lend, r_lo + p.RS);
  if (P >= r_hi) return;  // (the filter wrote empty slices)
  const int K = p.K, m = p.m, KP = p.KP, F = p.F;
  stage_lut32k(lut32k, p.lut64 + (size_t)q * K * m, K, KP, m, tid, kFW * 32);
  __syncthreads();
  const int64_t SW = p.RS / kFW;
  const int64_t w_lo = r_lo + warp * SW, w_hi = min(w_lo + SW, lend);
  const int64_t start = max(w_lo, P);
  if (start >= w_hi) return;
  int32_t* slice = p.slices + ((int64_t)(q * p.NR + r) * kFW + warp) * kSliceInts;
  const float hiT = p.qs[q].hiT;
  const uint32_t lt = (1u << lane) - 1u;
  int cnt = 0, npages = 0, pg_last = 0, pg_prev = 0;
  bool overflow = false;
  for (int64_t i0 = start; i0 < w_hi && !overflow; i0 += 128) {
    Row rows[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      rows[u] = load_row(p.codes_full, KP, i < w_hi ? i : start);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      const float e = exact32_any(lut32k, m, KP, rows[u]);
      const bool keep = i < w_hi && e < hiT;
      const uint32_t km = __ballot_sync(kFull, keep);
      if (!km || overflow) continue;  // (warp-uniform)
      const int T = __popc(km);
      if (cnt + T > npages * kPG) {  // one more page (T <= 32)
        int pgn = 0;
        if (npages + 1 > p.max_pages_cm) {
          overflow = true;
          if (lane == 0) atomicAdd(&p.qs[q].ovf_pages, 1);
        } else {
          if (lane == 0) pgn = atomicAdd(p.pool_top, 1);
          pgn = __shfl_sync(kFull, pgn, 0);
          if ((int64_t)pgn + 1 > p.pool_pages) {
            overflow = true;
            if (lane == 0) atomicAdd(&p.qs[q].ovf_pool, 1);
          } else {
            if (lane == 0) slice[1 + npages] = pgn;
            pg_prev = pg_last;
            pg_last = pgn;
            ++npages;
          }
        }
        if (overflow) continue;
      }
      if (keep) {
        const int pos = cnt + __popc(km & lt);
        const int pid = (pos >> 7) == npages - 1 ? pg_last : pg_prev;
        uint32_t tx = 0, ty = 0;  // the fast-code tuple, as the filter stores it
#pragma unroll
        for (int s2 = 0; s2 < (FP <= 8 ? FP : 8); ++s2) {
          if (s2 < F) {
            const uint32_t c2 = rows[u].byte(p.fast_books[s2]);
            if (s2 < 4) tx |= c2 << (8 * s2); else ty |= c2 << (8 * (s2 - 4));
          }
        }
        p.pool[((size_t)(uint32_t)pid << 7) | (uint32_t)(pos & (kPG - 1))] =
            make_uint4((uint32_t)i, 0u, tx, ty);
      }
      cnt += T;
    }
  }
  if (lane == 0) slice[0] = overflow ? -1 : cnt;
}

// ==========================================================================
// K3b: refine (count-mode queries)
// ==========================================================================
// The filter lists, for a count-mode query, every item with
// fast < T_P - Smin.  Only items with exact < T_P can ever be inserted (T
// never increases), so this kernel rescores the listed items with the full
// K-book table -- float32, certified against hiT with K terms: exact64 < T_P
// implies e32 < hiT -- and compacts each slice in place, in order.  One CTA
// per (query, range) with one warp per slice; units are range-major so the
// CTAs in flight read candidate rows of the same range from L2.  Thousands of
// warps each keep a page of row reads in flight: the random 8/16-byte row
// reads that stalled the streaming kernel run at memory-system throughput.
template <int FP>
__global__ void __launch_bounds__(kFW * 32) icq_refine_kernel(const __grid_constant__ PipeParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  float* lut32k = reinterpret_cast<float*>(dsm);  // [K][m]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (p.round > 0 && p.round_cnt[p.round] == 0) return;
  // units (query, group of RG ranges), query fastest; the table is staged once per unit
  const int K = p.K, m = p.m, KP = p.KP;
  const int64_t U = (int64_t)p.Q * p.NRG;
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    const int q = (int)(u % p.Q), rg = (int)(u / p.Q);
    // (the dense prefix kernel already applied this test to what it listed)
    if (!p.qs[q].count_mode || p.qs[q].done || p.qs[q].dense) continue;  // (CTA-uniform)
    const int r0 = rg * p.RG, r1 = min(p.NR, r0 + p.RG);
    if (p.qs[q].P >= min(p.qs[q].list_end, (int64_t)r1 * p.RS)) continue;
    __syncthreads();  // every warp is done with the previous unit's table
    stage_lut32k(lut32k, p.lut64 + (size_t)q * K * m, K, KP, m, tid, kFW * 32);
    __syncthreads();
    const float hiT = p.qs[q].hiT;
    unsigned long long raw = 0;
    for (int r = r0; r < r1; ++r) {
      int32_t* slice = p.slices + ((int64_t)(q * p.NR + r) * kFW + warp) * kSliceInts;
      const int cnt = slice[0];
      if (cnt <= 0) continue;  // empty, or overflowed (the replay walks it)
      const int w = refine_slice(p.pool, slice, cnt, p.codes_full, KP, m, hiT, lane, lut32k);
      if (lane == 0) slice[0] = w;
      raw += (unsigned long long)cnt;
    }
    if (lane == 0 && raw)
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.qs[q].listed_raw), raw);
  }
}

// K3c: per count-mode query, the offsets of its refined slices in one
// contiguous list (database order), and the list's place in cl_ent / cl_ex.
// A query with an overflowed slice, or whose list does not fit the buffer,
// keeps cl_base = -1: the replay decides it from the slices.
constexpr int kSliceOff = kSliceInts - 1;  // (the slice row's last int: offset in the list)
template <int FP>
__global__ void __launch_bounds__(256) icq_cl_scan_kernel(const __grid_constant__ PipeParams p) {
  __shared__ int wsum[8];
  __shared__ int carry_s, bad_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = blockIdx.x;
  if (p.round > 0 && p.round_cnt[p.round] == 0) return;
  if (p.qs[q].done) return;
  if (!p.cl_enable) {  // (ICQ_CL=0: every query is decided from its slices)
    if (tid == 0) p.qs[q].cl_base = -1;
    return;
  }
  const int NS = p.NR * kFW;
  int32_t* qsl = p.slices + (int64_t)q * NS * kSliceInts;
  if (tid == 0) { carry_s = 0; bad_s = 0; }
  __syncthreads();
  for (int s0 = 0; s0 < NS; s0 += 256) {
    const int s = s0 + tid;
    const int c = s < NS ? qsl[(int64_t)s * kSliceInts] : 0;
    if (c < 0) bad_s = 1;
    const int v = c > 0 ? c : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int off = carry_s + incl - v;
    for (int w = 0; w < warp; ++w) off += wsum[w];
    if (s < NS) qsl[(int64_t)s * kSliceInts + kSliceOff] = off;
    __syncthreads();
    if (tid == 255) carry_s = off + v;
    __syncthreads();
  }
  if (tid == 0) {
    const long long total = carry_s;
    long long base = -1;
    if (!bad_s) {
      base = (long long)atomicAdd(p.cl_top, (unsigned long long)total);
      if (base + total > p.cl_cap) base = -1;
    }
    p.qs[q].cl_base = base;
    p.qs[q].cl_count = total;
  }
}

// K3d: gather the refined slices into the query's contiguous list with the
// float64 exact score of every entry (reference order, exact64) -- the serial
// replay then streams 24 bytes per entry and reads no code rows.
template <int FP>
__global__ void __launch_bounds__(kFW * 32) icq_cl_gather_kernel(const __grid_constant__ PipeParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  double* lut = reinterpret_cast<double*>(dsm);  // [K][m]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (p.round > 0 && p.round_cnt[p.round] == 0) return;
  const int K = p.K, m = p.m, KP = p.KP;
  const int64_t U = (int64_t)p.Q * p.NRG;
  for (int64_t un = blockIdx.x; un < U; un += gridDim.x) {
  const int q = (int)(un % p.Q), rg = (int)(un / p.Q);
  if (p.qs[q].done || p.qs[q].cl_base < 0) continue;  // (CTA-uniform)
  const int r0 = rg * p.RG, r1 = min(p.NR, r0 + p.RG);
  if (p.qs[q].P >= min(p.qs[q].list_end, (int64_t)r1 * p.RS)) continue;
  __syncthreads();  // every warp is done with the previous unit's table
  const double* glut = p.lut64 + (size_t)q * K * m;
  for (int i = tid; i < K * m; i += kFW * 32) lut[i] = glut[i];
  __syncthreads();
  for (int r = r0; r < r1; ++r) {
  const int32_t* slice = p.slices + ((int64_t)(q * p.NR + r) * kFW + warp) * kSliceInts;
  const int cnt = slice[0];
  if (cnt <= 0) continue;
  const int64_t dst = p.qs[q].cl_base + slice[kSliceOff];
  for (int e0 = 0; e0 < cnt; e0 += 64) {
    uint4 ent[2];
    Row rows[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = e0 + u * 32 + lane;
      if (e < cnt) {
        ent[u] = p.pool[((size_t)(uint32_t)slice[1 + (e >> 7)] << 7) | (uint32_t)(e & (kPG - 1))];
        rows[u] = load_row(p.codes_full, KP, (int64_t)ent[u].x);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = e0 + u * 32 + lane;
      if (e < cnt) {
        p.cl_ent[dst + e] = ent[u];
        p.cl_ex[dst + e] = exact64(lut, m, K, false, rows[u]);
      }
    }
  }
  }
  }
}

// ==========================================================================
// K4: replay
// ==========================================================================
// float64 fast score of a candidate entry: from its fast-code tuple
// (FP <= 8) or stored directly (FP = 16)
template <int FP>
__device__ __forceinline__ double entry_f64(uint2 tail, const double* lutf, int m, int F) {
  if constexpr (FP <= 8) return tuple_f64<FP>(tail, lutf, m, F);
  else return __longlong_as_double((long long)(((unsigned long long)tail.y << 32) | tail.x));
}

// Decide one window of up to kWU*32 items in database order (u-major, then
// lane), each with its float64-decidable fast-code tuple (or float64 fast
// score, FP = 16) and, when known, its exact score.  Refined items (fast <
// bound + sigma, search.py:149) are compacted in order, their exact scores
// computed 32 at a time, and the first one under the heap maximum is
// inserted (search.py:152-154).  An insertion moves the bound (up or down):
// when it rises, the items after the insertion are compacted again.
// Returns -1 when the whole window is decided, else the window position
// (u * 32 + lane) of the insertion after which the live threshold left
// (floor_, cap]: above cap (the caller's list / pre-filter no longer covers
// the items after it) or at most floor_ (a walk may hand back to the lists).
template <int FP>
__device__ __forceinline__ int replay_window(Live& L, const RCtx& c, int lane,
                                             const int32_t (&ids)[kWU], const uint2 (&tail)[kWU],
                                             const double (&ex)[kWU], const bool (&valid)[kWU],
                                             int32_t* sid, int32_t* sidx, double* sfv,
                                             double* sfe, const double* lutf, double cap,
                                             double floor_) {
  int pos0 = 0;  // first undecided window position (u * 32 + lane)
  const uint32_t lt = (1u << lane) - 1u;
  for (;;) {
    const double thr = L.thr64;
    uint32_t lm[kWU];
    double d[kWU];
    int base[kWU];
    int tot = 0;
#pragma unroll
    for (int u = 0; u < kWU; ++u) {
      bool cand = valid[u] && (u * 32 + lane >= pos0);
      d[u] = 0.0;
      if (cand) {
        d[u] = entry_f64<FP>(tail[u], lutf, c.m, c.F);
        cand = d[u] < thr;
      }
      lm[u] = __ballot_sync(kFull, cand);
      base[u] = tot;
      tot += __popc(lm[u]);
    }
    if (tot == 0) return -1;
#pragma unroll
    for (int u = 0; u < kWU; ++u) {
      if ((lm[u] >> lane) & 1u) {
        const int pos = base[u] + __popc(lm[u] & lt);
        sid[pos] = ids[u];
        sidx[pos] = u * 32 + lane;
        sfv[pos] = d[u];
        sfe[pos] = ex[u];
      }
    }
    __syncwarp();
    bool restart = false;
    for (int b0 = 0; b0 < tot && !restart; b0 += 32) {
      const int j = b0 + lane;
      const bool v = j < tot;
      const int32_t id = v ? sid[j] : 0;
      const int32_t wpos = v ? sidx[j] : 0;
      const double f64 = v ? sfv[j] : 0.0;
      double e64 = v ? sfe[j] : 0.0;  // precomputed at chunk preparation, NaN = not yet
      if (v && !(e64 == e64)) e64 = exact64(c.lut, c.m, c.K, c.pw, load_row(c.codes_full, c.KP, id));
      uint32_t done = 0;
      for (;;) {
        const bool refined = v && !((done >> lane) & 1u) && (f64 < L.thr64);
        const bool ins = refined && (e64 < L.T64);
        const uint32_t rmask = __ballot_sync(kFull, refined);
        const uint32_t imask = __ballot_sync(kFull, ins);
        const int first = imask ? __ffs(imask) - 1 : 31;
        const uint32_t decided = imask ? (kFull >> (31 - first)) : kFull;
        if (!c.count_mode) {  // (count mode: the count kernel tallies refinements)
          L.refinements += __popc(rmask & decided);
          if (refined && ((decided >> lane) & 1u)) record_survivor(c.surv, id);
        }
        L.candidates += __popc(rmask & decided);
        done |= decided;
        if (!imask) break;
        const double ne = __shfl_sync(kFull, e64, first);
        const double nf = __shfl_sync(kFull, f64, first);
        const int32_t nid = __shfl_sync(kFull, id, first);
        L.H.replace_max(ne, nid, nf, lane);
        live_update64(L, c.sigma, c.k, c.f32);  // (the replay never uses the float32 bounds)
        ++L.insertions;
        if (c.count_mode) {  // items after nid are refined against the new threshold
          if (lane == 0) {
            if (L.ntraj < kMaxTraj) c.traj[L.ntraj] = TrajEntry{(int64_t)nid, L.thr64};
            else atomicOr(c.error, 16);
          }
          ++L.ntraj;
        }
        if (L.thr64 > cap || L.thr64 <= floor_) {
          const int r = __shfl_sync(kFull, wpos, first);
          __syncwarp();
          return r;
        }
        if (L.thr64 > thr) {  // bound rose: re-compact everything after the insertion
          pos0 = __shfl_sync(kFull, wpos, first) + 1;
          restart = true;
          break;
        }
      }
    }
    __syncwarp();
    if (!restart) return -1;
  }
}

// One CTA per query: warp 0 decides (the in-order reference loop), warps
// 1..3 prepare.  The candidate slices of a group (kSG slices) are cut into
// chunks of <= kCH entries (a rescan slice is a chunk of its own); chunk c+2
// is staged by cp.async, chunk c+1 prepared (float64 fast score from the
// tuple; exact score of every entry refined under the bound warp 0 last
// published) and chunk c decided, all at once, one CTA barrier per chunk.
//
// The lists hold every item with fast < theta (the list threshold the
// prologue chose).  They decide the reference loop exactly while the live
// threshold bound + sigma stays <= theta.  When an insertion lifts it above
// theta, the CTA WALKS the database in order from the next item: all four
// warps flag 64k-item sub-ranges against the live threshold (float64 fast
// scores from the codes), warp 0 decides the flagged items, and the walk
// hands back to the lists at the first insertion that brings the threshold
// back to <= theta.  Slices whose candidates overflowed their pages are
// walked the same way (without the early hand-back).
constexpr int kRW = 4;            // warps per replay CTA
constexpr int kRP = (kRW - 1) * 32;  // preparing threads
constexpr int kMaxChunks = 512;   // chunk descriptors per slice group (kSG * kListPages * kPG / kCH)
static_assert(kSG * ((kListPages * kPG + kCH - 1) / kCH) <= kMaxChunks,
              "a slice group always fits the chunk descriptors");

template <int FP>
__global__ void __launch_bounds__(kRW * 32, ICQ_REPLAY_CTAS) icq_replay_kernel(const __grid_constant__ PipeParams p) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = blockIdx.x;
  const int K = p.K, m = p.m, F = p.F, k = p.k;
  const int64_t n = p.n;
  const RepLayout Ly = rep_layout(K, m, F, k);
  double* lut = reinterpret_cast<double*>(dsm + Ly.lut64);
  double* he = reinterpret_cast<double*>(dsm + Ly.he);
  double* hf = reinterpret_cast<double*>(dsm + Ly.hf);
  int32_t* hi = reinterpret_cast<int32_t*>(dsm + Ly.hi);
  int32_t* sid = reinterpret_cast<int32_t*>(dsm + Ly.wid);
  int32_t* sidx = reinterpret_cast<int32_t*>(dsm + Ly.widx);
  double* sfv = reinterpret_cast<double*>(dsm + Ly.wfv);
  double* sfe = reinterpret_cast<double*>(dsm + Ly.wfe);
  double* lutf = reinterpret_cast<double*>(dsm + Ly.lutf);
  int32_t* smeta = reinterpret_cast<int32_t*>(dsm + Ly.meta);
  int32_t* scum = reinterpret_cast<int32_t*>(dsm + Ly.cum);
  int32_t* chunk = reinterpret_cast<int32_t*>(dsm + Ly.chunks);  // [kMaxChunks][3]
  uint4* ring = reinterpret_cast<uint4*>(dsm + Ly.ring);
  double* ring_e = reinterpret_cast<double*>(dsm + Ly.ringe);
  int32_t* plist = reinterpret_cast<int32_t*>(dsm + Ly.plist);   // prep: live-ish entries
  // control words: [0] chunks, [1] dropped entries, [2] prep list count,
  // [3] walk request, [16] stopped for the next round, [17] re-run the
  // chunk, [18] walk handed back (int32 words; bytes 16..63 hold the
  // 8-byte values below)
  volatile int32_t* ctl = reinterpret_cast<volatile int32_t*>(dsm + Ly.ctl);
  volatile double* pub_thr = reinterpret_cast<volatile double*>(dsm + Ly.ctl + 16);
  volatile long long* walk_from = reinterpret_cast<volatile long long*>(dsm + Ly.ctl + 24);
  volatile double* tsub = reinterpret_cast<volatile double*>(dsm + Ly.ctl + 32);
  volatile long long* snext = reinterpret_cast<volatile long long*>(dsm + Ly.ctl + 40);
  volatile long long* sskip = reinterpret_cast<volatile long long*>(dsm + Ly.ctl + 48);
  const long long t0 = clock64();
  const QState st = p.qs[q];
  for (int i = tid; i < k; i += kRW * 32) {
    he[i] = p.heap_e[(size_t)q * k + i];
    hf[i] = p.heap_f[(size_t)q * k + i];
    hi[i] = p.heap_i[(size_t)q * k + i];
  }
  const double* glut = p.lut64 + (size_t)q * K * m;
  if (st.P < n) {
    for (int i = tid; i < K * m; i += kRW * 32) lut[i] = glut[i];
    for (int i = tid; i < F * m; i += kRW * 32) {
      const int s2 = i / m, j = i - s2 * m;
      lutf[i] = glut[p.fast_books[s2] * m + j];
    }
  }
  if (st.done) return;  // finished in an earlier round
  if (tid == 0) {
    ctl[1] = 0; ctl[2] = 0; ctl[3] = 0; ctl[16] = 0; ctl[17] = 0; ctl[18] = 0;
    *sskip = st.P - 1;
  }
  __syncthreads();
  Live L;
  L.refinements = st.refinements;
  L.insertions = st.insertions;
  L.candidates = L.certified = 0;
  L.H.k = k;
  L.H.reg = k <= 32 * kRegHeapRegs;
  L.H.he = he;
  L.H.hf = hf;
  L.H.hi = hi;
  int64_t fallback_slices = 0, listed = 0, walked = 0;
  long long t_work = 0, t_wait = 0;  // warp 0: deciding vs waiting at the chunk barrier
  RCtx c;
  c.lut = lut;
  c.codes_full = p.codes_full;
  c.fb = p.fast_books;
  c.KP = p.KP; c.m = m; c.K = K; c.F = F; c.k = k;
  c.sigma = p.sigma;
  c.f32 = p.sigma_f32 != 0;
  c.pw = false;  // n >= 2 whenever the replay runs (P >= k >= 1 and P < n)
  c.wide = false;
  c.surv = p.survivors ? p.survivors + (int64_t)q * p.words : nullptr;
  c.count_mode = st.count_mode != 0;
  c.traj = p.traj + (size_t)q * kMaxTraj;
  c.error = p.error;
  L.ntraj = st.ntraj;
  const double theta = st.thr;  // the lists' threshold
  const int64_t SW = p.RS / kFW;

  // ---- the in-order walk (all threads; CTA-uniform control) ----------------
  auto fast_at = [&](int64_t i, uint2& tup) -> double {
    const Row r2 = load_fast_row(p.codes_fast, FP, i);
    double x;
    if constexpr (FP <= 8) {
      tup = make_uint2(r2.w[0], r2.w[1]);
      x = tuple_f64<FP>(tup, lutf, m, F);
    } else {
      x = 0.0;  // float64 fast score in the reference's order
#pragma unroll
      for (int s2 = 0; s2 < FP; ++s2)
        if (s2 < F) x = __dadd_rn(x, lutf[s2 * m + (int)r2.byte(s2)]);
      const unsigned long long db = (unsigned long long)__double_as_longlong(x);
      tup = make_uint2((uint32_t)db, (uint32_t)(db >> 32));
    }
    return x;
  };
  // warp 0: decide the items at positions [0, npos) given by position -> id
  auto decide_items = [&](auto id_at, int npos, double cap, double floor_) -> int {
    for (int w0 = 0; w0 < npos; w0 += kWU * 32) {
      int32_t ids2[kWU];
      uint2 t2[kWU];
      double e2[kWU];
      bool valid2[kWU];
#pragma unroll
      for (int u = 0; u < kWU; ++u) {
        const int x = w0 + u * 32 + lane;
        valid2[u] = x < npos;
        const int64_t i = valid2[u] ? id_at(x) : 0;
        ids2[u] = (int32_t)i;
        t2[u] = make_uint2(0u, 0u);
        e2[u] = __longlong_as_double(0x7ff8000000000000LL);
        if (valid2[u]) (void)fast_at(i, t2[u]);
      }
      const int b = replay_window<FP>(L, c, lane, ids2, t2, e2, valid2, sid, sidx, sfv, sfe,
                                      lutf, cap, floor_);
      if (b >= 0) return w0 + b;
    }
    return -1;
  };
  // Walk items [from, to) in order with the live threshold.  hand_back: stop
  // at the first insertion that brings the threshold back to <= theta (the
  // lists cover the rest).  Afterwards *sskip = the last decided item.
  // Sub-ranges are flagged by all four warps against the threshold T at
  // their start, with coalesced 16-byte reads of the tile-transposed fast
  // rows (a warp tile = 128 chunks; lane l holds the consecutive logical
  // chunks 4l..4l+3); warp 0 decides the flagged items in order.  An
  // insertion lifting the threshold above T restarts flagging right after
  // it, with a short sub-range that doubles while no restart happens.
  // Scratch: rmask holds max_sub/32 flag words, rlst 1024 positions.
  auto walk = [&](int64_t from, int64_t to, bool hand_back, uint32_t* rmask, int32_t* rlst,
                  int max_sub) {
    using G = FGeo<FP>;
    constexpr int IPC = G::IPC, TILE = G::TILE;
    constexpr int LB = 4 * IPC;                   // flag bits per lane and tile
    constexpr int LPW = LB >= 32 ? 1 : 32 / LB;   // lanes per flag word
    const int sub_cap = max_sub - TILE;           // (the first tile may start before s0)
    int sub = hand_back ? min(8192, sub_cap) : sub_cap;
    int64_t s0 = from;
    bool back = false;
    while (s0 < to && !back) {
      const int64_t s1 = min(to, s0 + (int64_t)sub);
      const int64_t base = s0 & ~(int64_t)(TILE - 1);
      if (tid == 0) *tsub = (p.debug & 16) ? kInf64 : L.thr64;  // debug: flag every item
      __syncthreads();
      const double T = *tsub;
      const int ntile = (int)((s1 - base + TILE - 1) / TILE);
      for (int t = warp; t < ntile; t += kRW) {
        const int64_t tb = base + (int64_t)t * TILE;
        const uint4* cp = reinterpret_cast<const uint4*>(p.codes_fast) + tb / IPC + lane;
        uint4 x[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) x[v] = __ldg(cp + v * 32);
        unsigned long long bits = 0;
        const int64_t i0 = tb + (int64_t)lane * LB;  // this lane's first item
#pragma unroll
        for (int v = 0; v < 4; ++v) {
#pragma unroll
          for (int j = 0; j < IPC; ++j) {
            const int64_t i = i0 + v * IPC + j;
            double f;
            if constexpr (FP <= 8) {
              f = tuple_f64<FP>(chunk_tuple<FP>(x[v], j), lutf, m, F);
            } else {
              const uint32_t wd[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
              f = 0.0;  // float64 fast score in the reference's order
#pragma unroll
              for (int s2 = 0; s2 < FP; ++s2)
                if (s2 < F) f = __dadd_rn(f, lutf[s2 * m + ((wd[s2 >> 2] >> (8 * (s2 & 3))) & 0xffu)]);
            }
            // (T = inf flags every item, NaN scores included)
            if (i >= s0 && i < s1 && !(f >= T)) bits |= 1ull << (v * IPC + j);
          }
        }
        const int w0 = (int)((tb - base) >> 5);  // first flag word of the tile
        if constexpr (LB >= 32) {
#pragma unroll
          for (int h = 0; h < LB / 32; ++h) rmask[w0 + lane * (LB / 32) + h] = (uint32_t)(bits >> (32 * h));
        } else {
          uint32_t wv = (uint32_t)bits << ((lane % LPW) * LB);
#pragma unroll
          for (int o = 1; o < LPW; o <<= 1) wv |= __shfl_xor_sync(kFull, wv, o);
          if (lane % LPW == 0) rmask[w0 + lane / LPW] = wv;
        }
      }
      __syncthreads();
      if (warp == 0) {
        int64_t next = s1;
        bool hb = false;
        const int nwords = ntile * (TILE / 32);
        for (int w0 = 0; w0 < nwords; w0 += 32) {
          const uint32_t wv = w0 + lane < nwords ? rmask[w0 + lane] : 0u;
          const int cw = __popc(wv);
          int incl = cw;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
          }
          const int nl = __shfl_sync(kFull, incl, 31);
          int o = incl - cw;
          for (uint32_t bb = wv; bb; bb &= bb - 1) rlst[o++] = (w0 + lane) * 32 + __ffs(bb) - 1;
          __syncwarp();
          const int b = decide_items([&](int x) { return base + rlst[x]; }, nl, T,
                                     hand_back ? theta : -kInf64);
          __syncwarp();
          if (b >= 0) {  // an insertion moved the threshold out of (floor, T]
            const int64_t y = base + rlst[b];
            hb = hand_back && L.thr64 <= theta;
            next = hb ? y : y + 1;  // rose above T: flag again from the next item
            break;
          }
        }
        if (lane == 0) {
          *snext = (long long)next;
          ctl[18] = hb ? 1 : 0;
          *pub_thr = L.thr64;
        }
      }
      __syncthreads();
      back = ctl[18] != 0;
      const int64_t nx = (int64_t)*snext;
      walked += (back ? nx + 1 : nx) - s0;  // (CTA-uniform)
      // restarted after an insertion: short sub-ranges again; else grow
      sub = nx < s1 ? min(2048, sub_cap) : min(2 * sub, sub_cap);
      s0 = back ? nx + 1 : nx;
      // long walks (in-order and overflowed-slice walks of this round
      // together) hand the query to the next round: the filter lists the
      // rest under the current live threshold on all SMs (one CTA walks ~1
      // item per clock; a filter pass streams the whole query in microseconds)
      if (!back && !p.last_round && s0 < to && walked > p.walk_cap) {
        if (tid == 0) ctl[16] = 1;
        break;
      }
    }
    if (tid == 0) *sskip = (long long)((back || ctl[16]) ? s0 - 1 : max(to - 1, (int64_t)*sskip));
    __syncthreads();
  };

  if (st.P < n) {
    if (warp == 0) {
      L.H.load(lane);
      live_update(L, F, p.sigma, k, c.f32, false);
      if (lane == 0) *pub_thr = L.thr64;
    }
    const int NS = p.NR * kFW;  // slices of this query, in database order
    const int32_t* qsl = p.slices + (int64_t)q * NS * kSliceInts;
    const int ptid = tid - 32;  // preparing thread index (warps 1..3)
    // Contiguous list (K3c/K3d): the query's listed entries in database order
    // with their float64 exact scores; warps 1..3 stage chunks (cp.async
    // ring), warp 0 decides.  Count mode: only the entries still under the
    // heap maximum matter (T never increases) and no walk is ever needed.
    // List mode: an insertion that lifts the live threshold above theta
    // starts an in-order walk of the database (all four warps); the list
    // resumes at the first entry after the last walked item.
    const bool cl = st.cl_base >= 0;
    if (cl) {
      const int64_t total = st.cl_count;
      const uint4* cle = p.cl_ent + st.cl_base;
      const double* clx = p.cl_ex + st.cl_base;
      listed += total;
      int64_t e_base = 0;  // the pipeline (re)starts at this entry
      for (;;) {
        const int nch = (int)((total - e_base + kCH - 1) / kCH);
        auto issue_cl = [&](int ch) {
          if (ch < nch) {
            uint4* dst = ring + (ch % kRSlots) * kCH;
            double* dex = ring_e + (ch % kRSlots) * kCH;
            const int64_t e0 = e_base + (int64_t)ch * kCH;
            const int len = (int)min((int64_t)kCH, total - e0);
            for (int i = ptid; i < len; i += kRP) {
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + i)),
                           "l"(cle + e0 + i)
                           : "memory");
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dex + i)),
                           "l"(clx + e0 + i)
                           : "memory");
            }
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
        };
        if (warp > 0) {
          issue_cl(0);
          issue_cl(1);
          issue_cl(2);
          asm volatile("cp.async.wait_group 2;" ::: "memory");
        }
        __syncthreads();
        bool want_walk = false;
        for (int ch = 0; ch < nch; ++ch) {
          if (warp > 0) {
            issue_cl(ch + 3);
            asm volatile("cp.async.wait_group 2;" ::: "memory");  // chunk ch + 1 landed
          } else {
            const uint4* src = ring + (ch % kRSlots) * kCH;
            const double* exs = ring_e + (ch % kRSlots) * kCH;
            const int len = (int)min((int64_t)kCH, total - e_base - (int64_t)ch * kCH);
            for (int w0 = 0; w0 < len; w0 += kWU * 32) {
              int32_t ids[kWU];
              uint2 tl[kWU];
              double exv[kWU];
              bool valid[kWU];
              bool any = false;
#pragma unroll
              for (int u = 0; u < kWU; ++u) {
                const int e = w0 + u * 32 + lane;
                const bool ok = e < len;
                const uint4 ent = ok ? src[e] : make_uint4(0, 0, 0, 0);
                exv[u] = ok ? exs[e] : 0.0;
                // count mode: exact >= T now can never be inserted later
                valid[u] = ok && !(c.count_mode && exv[u] >= L.T64);
                ids[u] = (int32_t)ent.x;
                tl[u] = make_uint2(0u, 0u);
                if (valid[u]) {
                  const unsigned long long fb = (unsigned long long)__double_as_longlong(
                      entry_f64<FP>(make_uint2(ent.z, ent.w), lutf, m, F));
                  tl[u] = make_uint2((uint32_t)fb, (uint32_t)(fb >> 32));
                }
                any |= valid[u];
              }
              if (!__any_sync(kFull, any)) continue;
              const int b2 = replay_window<16>(L, c, lane, ids, tl, exv, valid, sid, sidx, sfv, sfe,
                                               lutf, c.count_mode ? kInf64 : theta, -kInf64);
              if (b2 >= 0) {  // the live threshold rose above theta: walk from the next item
                const int32_t y = __shfl_sync(kFull, ids[b2 >> 5], b2 & 31);
                if (lane == 0) { *walk_from = (long long)y + 1; ctl[3] = 1; }
                break;
              }
            }
            if (lane == 0) *pub_thr = L.thr64;
          }
          __syncthreads();
          if (ctl[3]) { want_walk = true; break; }  // (CTA-uniform)
        }
        if (warp > 0) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (!want_walk) {
          if (tid == 0) *sskip = st.list_end - 1;
          __syncthreads();
          break;
        }
        const int64_t from = (int64_t)*walk_from;
        __syncthreads();
        if (tid == 0) ctl[3] = 0;
        // scratch: two exact-score slots of the (drained) ring
        walk(from, st.list_end, true, reinterpret_cast<uint32_t*>(ring_e),
             reinterpret_cast<int32_t*>(ring_e + kCH), kCH * 8 * 8);
        if (*sskip >= st.list_end - 1 || ctl[16]) break;  // walked to the end / handed over
        if (tid == 0) {  // resume at the first entry after the last walked item
          const int64_t skp = (int64_t)*sskip;
          int64_t lo2 = e_base, hi2 = total;
          while (lo2 < hi2) {
            const int64_t mid = (lo2 + hi2) >> 1;
            if ((int64_t)cle[mid].x <= skp) lo2 = mid + 1; else hi2 = mid;
          }
          *snext = (long long)lo2;
        }
        __syncthreads();
        e_base = (int64_t)*snext;
        __syncthreads();
        if (e_base >= total) {
          if (tid == 0) *sskip = st.list_end - 1;
          __syncthreads();
          break;
        }
      }
    }
    for (int g0 = 0; !cl && g0 < NS && *sskip < n - 1 && !ctl[16]; g0 += kSG) {
      const int ng = min(kSG, NS - g0);
      {  // group meta (counts + page ids) -> shared memory
        // (the first kStageInts ints of every slice row: count + the page ids
        // a list-mode slice can hold)
        constexpr int kPieces = kStageInts / 4;
        for (int i = tid; i < ng * kPieces; i += kRW * 32) {
          const int t2 = i / kPieces, w2 = i - t2 * kPieces;
          const uint4* src =
              reinterpret_cast<const uint4*>(qsl + (int64_t)(g0 + t2) * kSliceInts) + w2;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smeta + 4 * i)),
                       "l"(src)
                       : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
      }
      __syncthreads();
      if (tid == 0) {
        // scum: listed entries before each slice (rescans count 0); chunks:
        // {first virtual entry, length, -1} or {-, -, rescan slice}
        int acc = 0, nc = 0, open = -1, dropped = 0;
        for (int t2 = 0; t2 < ng; ++t2) {
          scum[t2] = acc;
          const int cnt = smeta[t2 * kStageInts];
          // (overflowed, or a count-mode slice longer than the staged page table)
          if (cnt < 0 || cnt > kListPages * kPG) {
            if (nc < kMaxChunks) { chunk[3 * nc] = acc; chunk[3 * nc + 1] = 0; chunk[3 * nc + 2] = t2; ++nc; }
            else dropped = 1;
            open = -1;
            continue;
          }
          int rem = cnt;
          while (rem > 0) {
            if (open < 0 || chunk[3 * open + 1] == kCH) {
              if (nc >= kMaxChunks) break;
              open = nc++;
              chunk[3 * open] = acc;
              chunk[3 * open + 1] = 0;
              chunk[3 * open + 2] = -1;
            }
            const int take = min(rem, kCH - chunk[3 * open + 1]);
            chunk[3 * open + 1] += take;
            acc += take;
            rem -= take;
          }
          dropped |= rem > 0;
        }
        scum[ng] = acc;
        ctl[0] = nc;
        ctl[1] = dropped;
      }
      __syncthreads();
      const int nc = ctl[0];
      if (ctl[1]) {  // cannot happen (static_assert above): fail loudly, never silently
        if (tid == 0) atomicOr(p.error, 4);
        break;
      }
      listed += scum[ng];
      // ---- preparing warps: stage chunk ch (cp.async) ----
      auto issue = [&](int ch) {
        if (ch < nc && chunk[3 * ch + 2] < 0) {
          uint4* dst = ring + (ch % kRSlots) * kCH;
          const int v0 = chunk[3 * ch], len = chunk[3 * ch + 1];
          if (ptid < len) {
            int lo2 = 0, hi2 = ng;  // slice t: scum[t] <= v < scum[t + 1]
            const int v = v0 + ptid;
            while (hi2 - lo2 > 1) {
              const int mid = (lo2 + hi2) >> 1;
              if (scum[mid] <= v) lo2 = mid; else hi2 = mid;
            }
            int ts = lo2;
            int e = v - scum[ts];
            int tcnt = scum[ts + 1] - scum[ts];
            for (int i = ptid; i < len; i += kRP) {
              while (e >= tcnt) {
                e -= tcnt;
                ++ts;
                tcnt = scum[ts + 1] - scum[ts];
              }
              const int32_t* sm = smeta + ts * kStageInts;
              const uint4* src = p.pool + (int64_t)sm[1 + e / kPG] * kPG + (e % kPG);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst + i)),
                           "l"(src)
                           : "memory");
              e += kRP;
            }
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      // ---- preparing warps: float64 fast scores, exact scores of the
      //      entries refined under the published bound ----
      auto prep = [&](int ch) {
        if (ch >= nc || chunk[3 * ch + 2] >= 0) return;
        uint4* src = ring + (ch % kRSlots) * kCH;
        double* ex = ring_e + (ch % kRSlots) * kCH;
        const int len = chunk[3 * ch + 1];
        const double thr = *pub_thr;
        const int64_t skp = (int64_t)*sskip;
        for (int i = ptid; i < len; i += kRP) {
          uint4 ent = src[i];
          const double f = entry_f64<FP>(make_uint2(ent.z, ent.w), lutf, m, F);
          const unsigned long long fb = (unsigned long long)__double_as_longlong(f);
          ent.z = (uint32_t)fb;
          ent.w = (uint32_t)(fb >> 32);
          src[i] = ent;
          ex[i] = __longlong_as_double(0x7ff8000000000000LL);
          if ((f < thr || c.count_mode) && (int64_t)ent.x > skp && !(p.debug & 2))
            plist[atomicAdd((int*)&ctl[2], 1)] = i;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kRP));
        // exact scores of the entries under the published bound (debug bit 3:
        // of every entry).  Rows are read in batches of kXB per thread so
        // their latencies overlap.
        const int nl = (p.debug & 8) ? len : ctl[2];
        constexpr int kXB = 6;
        for (int j0 = ptid; j0 < nl; j0 += kXB * kRP) {
          Row rows[kXB];
          int idx[kXB];
#pragma unroll
          for (int r = 0; r < kXB; ++r) {
            const int jj = j0 + r * kRP;
            idx[r] = jj < nl ? ((p.debug & 8) ? jj : (int)plist[jj]) : -1;
            if (idx[r] >= 0) rows[r] = load_row(p.codes_full, p.KP, (int32_t)src[idx[r]].x);
          }
#pragma unroll
          for (int r = 0; r < kXB; ++r)
            if (idx[r] >= 0) ex[idx[r]] = exact64(lut, m, K, false, rows[r]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kRP));
        if (ptid == 0) ctl[2] = 0;
      };
      if (warp > 0) {
        if (ptid == 0) ctl[2] = 0;
        asm volatile("bar.sync 1, %0;" ::"n"(kRP));
        issue(0);
        issue(1);
        issue(2);
        asm volatile("cp.async.wait_group 2;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"n"(kRP));
        prep(0);
      }
      __syncthreads();
      for (int ch = 0; ch < nc;) {
        const long long tw0 = clock64();
        const bool rerun = ctl[17] != 0;  // (CTA-uniform: set before the last barrier)
        const bool rescan = chunk[3 * ch + 2] >= 0;
        if (warp > 0) {
          if (!rerun) {
            issue(ch + 3);
            asm volatile("cp.async.wait_group 2;" ::: "memory");  // chunk ch+1 landed
            asm volatile("bar.sync 1, %0;" ::"n"(kRP));
            prep(ch + 1);
          }
        } else if (!rescan) {
          const uint4* src = ring + (ch % kRSlots) * kCH;
          const double* exs = ring_e + (ch % kRSlots) * kCH;
          const int len = chunk[3 * ch + 1];
          const int64_t skp = (int64_t)*sskip;
          for (int w0 = 0; w0 < len; w0 += kWU * 32) {
            int32_t ids[kWU];
            uint2 tl[kWU];
            double exv[kWU];
            bool valid[kWU];
            bool any = false;
#pragma unroll
            for (int u = 0; u < kWU; ++u) {
              const int e = w0 + u * 32 + lane;
              const uint4 ent = e < len ? src[e] : make_uint4(0, 0, 0, 0);
              valid[u] = e < len && (int64_t)ent.x > skp;  // walked items are decided
              ids[u] = (int32_t)ent.x;
              tl[u] = make_uint2(ent.z, ent.w);  // float64 fast score (prep)
              exv[u] = valid[u] ? exs[e] : 0.0;
              // count mode: only insertions matter; exact >= T now can never
              // insert again (T never increases)
              if (c.count_mode && valid[u] && exv[u] >= L.T64) valid[u] = false;
              any |= valid[u];
            }
            if (c.count_mode && !__any_sync(kFull, any)) continue;
            // (count mode: the lists hold every possible insertion whatever the
            // live threshold is -- no walks)
            const int b = replay_window<16>(L, c, lane, ids, tl, exv, valid, sid, sidx, sfv, sfe,
                                            lutf, c.count_mode ? kInf64 : theta, -kInf64);
            if (b >= 0) {  // the live threshold rose above theta: walk from the next item
              const int32_t y = __shfl_sync(kFull, ids[b >> 5], b & 31);
              if (lane == 0) { *walk_from = (long long)y + 1; ctl[3] = 1; }
              break;
            }
          }
          if (lane == 0) *pub_thr = L.thr64;
        }
        if (rescan) {  // (CTA-uniform)
          // candidates overflowed this slice's pages: walk its items from the codes
          __syncthreads();
          const int64_t j = g0 + chunk[3 * ch + 2];
          const int64_t lo = max(max(j * SW, st.P), (int64_t)*sskip + 1),
                        hi_ = min((j + 1) * SW, st.list_end);
          if (lo < hi_) {
            if (tid == 0) ++fallback_slices;
            // (a rescan chunk is never staged: its ring slot (8 KiB of mask
            // words, 64k-item sub-ranges) and exact-score slot are free)
            walk(lo, hi_, false, reinterpret_cast<uint32_t*>(ring + (ch % kRSlots) * kCH),
                 reinterpret_cast<int32_t*>(ring_e + (ch % kRSlots) * kCH), kCH * 16 * 8);
            if (warp == 0 && lane == 0 && L.thr64 > theta && hi_ < n && !ctl[16] && !c.count_mode) {
              *walk_from = hi_;  // the lists stop covering the items after the slice
              ctl[3] = 1;
            }
          }
        }
        const long long tw1 = clock64();
        __syncthreads();
        if (warp == 0) { t_work += tw1 - tw0; t_wait += clock64() - tw1; }
        if (ctl[3]) {  // (CTA-uniform) walk until the threshold is back under theta
          const int64_t from = (int64_t)*walk_from;
          __syncthreads();
          if (tid == 0) ctl[3] = 0;
          // scratch: the exact-score slots of chunks ch+2 and ch+3 (their
          // entries may still be landing, but prep fills those slots only in
          // the iterations ch+1 / ch+2); 4 KiB each -> 32k-item sub-ranges
          walk(from, n, true, reinterpret_cast<uint32_t*>(ring_e + ((ch + 2) % kRSlots) * kCH),
               reinterpret_cast<int32_t*>(ring_e + ((ch + 3) % kRSlots) * kCH), kCH * 8 * 8);
          if (tid == 0) ctl[17] = 1;  // decide the rest of chunk ch (ids after the walk)
          __syncthreads();
        } else {
          if (tid == 0) ctl[17] = 0;
          __syncthreads();
          ++ch;
        }
        if (*sskip >= n - 1 || ctl[16]) break;  // (CTA-uniform) walked to the end / stopped
      }
      if (warp > 0) asm volatile("cp.async.wait_all;" ::: "memory");
      if (tid == 0) ctl[17] = 0;
      __syncthreads();
    }
    if (warp == 0) L.H.store(lane);
    // the lists covered a prefix only: the rest goes to the next round
    if (tid == 0 && !ctl[16] && st.list_end < n && !p.last_round) {
      *sskip = st.list_end - 1;
      ctl[16] = 1;
    }
  }
  __syncthreads();
  if (ctl[16]) {
    // a walk ran past p.walk_cap (or the lists covered a prefix only): hand
    // the query to the next round -- the heap (sorted descending), the first
    // undecided item and, as the new list threshold, the live threshold
    // itself (J = 0)
    //
    // Count mode pays only while T - Smin is selective, which takes a
    // near-exact heap (small sigma / low recall leaves T loose).  With the
    // heap of the hand-over, sample the last <= 16k decided items: the query
    // stays in count mode iff the live threshold still passes a long list
    // AND T - Smin passes <= 1/2; else it goes on in list mode (theta from
    // the ladder of A_J, as at the prologue end) and the count kernel covers
    // [P0, cm_end) only.
    bool to_list = false;
    double theta_new = 0.0;
    if (st.count_mode && (!p.force_count || (p.debug & 64))) {  // (debug bit 6: always switch)
      constexpr int kLad = 10;
      const int ladder[kLad] = {0, 1, 2, 4, 8, 16, 32, 64, 1 << 30, 0};
      double* lad_thr = sfv;                            // (the window scratch is free now)
      int* lad_cnt = reinterpret_cast<int*>(sfe);
      const int64_t E = (int64_t)*sskip + 1;
      int64_t S = min((int64_t)16384, E - st.P0);
      if (warp == 0) {
        for (int r = 0; r < kLad - 1; ++r) {
          const double A = heap_AJ(hf, k, min(ladder[r], k - 1), lane, nullptr);
          if (lane == 0) { lad_thr[r] = thr_cover(A, p.sigma, c.f32, false); lad_cnt[r] = 0; }
        }
        if (lane == 0) {
          const double T = he[0];
          lad_thr[kLad - 1] = __dadd_ru(__dsub_ru(T, st.smin), fabs(T) * 1e-12);
          lad_cnt[kLad - 1] = 0;
        }
      }
      __syncthreads();
      int cnt[kLad];
#pragma unroll
      for (int r = 0; r < kLad; ++r) cnt[r] = 0;
      for (int64_t i = E - S + tid; i < E; i += kRW * 32) {
        uint2 tup;
        const double f = fast_at(i, tup);
#pragma unroll
        for (int r = 0; r < kLad; ++r) cnt[r] += f < lad_thr[r] ? 1 : 0;
      }
#pragma unroll
      for (int r = 0; r < kLad; ++r) {
        const int c2 = __reduce_add_sync(kFull, cnt[r]);
        if (lane == 0 && c2) atomicAdd(&lad_cnt[r], c2);
      }
      __syncthreads();
      // (a query already in count mode stays there more readily than one
      // enters it: the in-order list replay of a 100M-item database costs more
      // per listed item than the count pass per streamed item)
      const bool stay = !(p.debug & 64) && S > 0 && (int64_t)lad_cnt[0] * p.count_div * 4 > S &&
                        (double)lad_cnt[0] * (double)(n - E) * 4.0 > (double)p.count_min * (double)S &&
                        (int64_t)lad_cnt[kLad - 1] * 2 <= S;
      if (!stay) {
        to_list = true;
        int J = 0;
        for (int r = 0; r < kLad - 1; ++r)
          if (S > 0 && (int64_t)lad_cnt[r] * p.list_div <= S) J = r;
        if (p.list_j >= 0) {  // (a fixed J: its threshold)
          J = 0;
          for (int r = 0; r < kLad - 1; ++r)
            if (ladder[r] <= p.list_j) J = r;
        }
        theta_new = lad_thr[J];
      }
    }
    for (int i = tid; i < k; i += kRW * 32) {
      p.heap_e[(size_t)q * k + i] = he[i];
      p.heap_f[(size_t)q * k + i] = hf[i];
      p.heap_i[(size_t)q * k + i] = hi[i];
    }
    if (tid == 0) {
      QState ns = st;
      ns.P = (int64_t)*sskip + 1;
      ns.refinements = L.refinements;
      ns.insertions = L.insertions;
      ns.thr = L.thr64;
      if (st.count_mode && to_list) {
        ns.count_mode = 0;
        ns.cm_end = ns.P;  // the count kernel covers [P0, cm_end)
        ns.thr = theta_new;
        ns.mt_valid = 0;
      } else if (st.count_mode) {
        // count mode lists every possible insertion whatever the live
        // threshold does later: fast < T - Smin with T at the hand-over
        const double T = he[0];
        ns.thr = __dadd_ru(__dsub_ru(T, st.smin), fabs(T) * 1e-12);
        float loT;
        certified_bounds(T, K, loT, ns.hiT);
      }
      certified_bounds(ns.thr, F, ns.lo, ns.hi);
      if (ns.mt_valid) {  // sigma == 0: the heap maximum's tuple ties at thr exactly
        const Row r = load_fast_row(p.codes_fast, FP, hi[0]);
        ns.mtup[0] = r.w[0];
        ns.mtup[1] = r.w[1];
      }
      ns.ovf_pages = 0;
      ns.ovf_pool = 0;
      ns.rounds = st.rounds + 1;
      ns.list_end = n;
      ns.dense = 0;
      atomicAdd(&p.round_cnt[p.round + 1], 1);
      ns.walked = st.walked + walked;
      ns.ntraj = L.ntraj;
      p.qs[q] = ns;
    }
    return;
  }
  if (tid == 0) {
    p.qs[q].done = 1;
    p.qs[q].P = n;  // later filter rounds skip this query
    p.qs[q].ntraj = L.ntraj;  // (count mode: the count kernel's segments)
  }
  // output: heap ascending by (score, id) (search.py:156-165)
  for (int i = tid; i < k; i += kRW * 32) {
    const int src = k - 1 - i;
    p.ids[(size_t)q * k + i] = hi[src];
    p.scores[(size_t)q * k + i] = he[src];
  }
  if (tid == 0) {
    if (p.refinements) p.refinements[q] = p.exact_mode ? n : L.refinements;
    if (p.stats) {
      int64_t* s = p.stats + (size_t)q * kStats;
      s[0] = L.insertions;
      s[1] = L.candidates;
      s[2] = st.walked + walked;
      s[3] = st.P0;  // the prologue end (P moves when a query is handed to a new round)
      s[4] = st.pro_cycles;
      s[5] = clock64() - t0;
      s[6] = fallback_slices | ((int64_t)p.qs[q].ovf_pages << 20) | ((int64_t)p.qs[q].ovf_pool << 40);
      s[7] = st.wide | ((int64_t)(st.rounds + 1) << 8);  // wide flag | rounds used << 8
      s[8] = st.pro_cand;
      s[9] = listed;
      s[10] = st.insertions;
      s[11] = p.qs[q].listed_raw;  // count mode: listed before the refine kernel (all rounds)
      s[12] = (p.debug & 4) ? t_work : st.pro_t[0];  // debug bit 2: replay warp-0 timers
      s[13] = (p.debug & 4) ? t_wait : st.pro_t[1];
      s[14] = st.pro_t[2];
      s[15] = p.qs[q].skipped;
    }
  }
}

// ==========================================================================
// K5: refinement count (count-mode queries)
// ==========================================================================
// For a count-mode query the replay decided only the possible insertions and
// recorded the live threshold after each one (TrajEntry: items > pos use thr;
// thr0 before the first).  Every item i >= P0 is refined iff
// fast64(i) < thr(i) (search.py:149) -- a parallel test once the trajectory
// is known.  This kernel streams the fast codes like the filter (coalesced
// 16-byte tile loads, lane-private float32 LUT pages, certified float32 test
// with a float64 decision in the uncertain band), counts the refined items
// into refinements[q] and sets their survivor bits.
template <int FP>
__global__ void __launch_bounds__(kFW * 32, 1) icq_count_kernel(const __grid_constant__ PipeParams p) {
  using G = FGeo<FP>;
  constexpr int IPC = G::IPC, V = G::V, TILE = G::TILE, N = V * IPC;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t dyn_size;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_size));
  if (smem_addr(dsm) != kDynBase || smem_addr(dsm) + dyn_size < G::kSmemEnd) {
    if (tid == 0) atomicOr(p.error, 1);
    return;
  }
  uint32_t Lp[FP];
#pragma unroll
  for (int s = 0; s < FP; ++s)
    Lp[s] = ((uint32_t)(1 + s / G::BPR) << 16) |
            (uint32_t)((s % G::BPR) * 4 * G::R + (lane % G::R) * 4);
  const int K = p.K, m = p.m, F = p.F;
  // (ranges of its own, RSC >= RS items: no slices here, and longer units
  // amortise the per-unit barriers and table staging)
  const int64_t n = p.n, RS = p.RSC, SW = p.RSC / kFW;
  // units: (count-mode query, range), range-major over the batch's count-mode
  // queries only, so that a few such queries still spread over every SM
  const int ncm = p.cm_list[0];
  const int64_t U = (int64_t)ncm * p.NRC;
  const uint4* codes = reinterpret_cast<const uint4*>(p.codes_fast);
  double* lut64f = reinterpret_cast<double*>(dsm);
  // the trajectory entries of the unit's range, staged per unit (insertions are
  // sparse after the prologue: a 1M-item range holds a handful)
  constexpr int kTS = 1024;
  int64_t* s_pos = reinterpret_cast<int64_t*>(dsm + 16384);  // (lut64f: <= 16 KiB)
  double* s_thr = reinterpret_cast<double*>(dsm + 16384 + kTS * 8);  // [kTS + 1]: + the threshold before
  int* s_ctl = reinterpret_cast<int*>(dsm + 16384 + kTS * 16 + 16);
  int cur_q = -1;
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    const int q = p.cm_list[1 + (int)(u % ncm)];
    const int r = (int)(u / ncm);
    const int64_t P0 = p.qs[q].P0;
    // (a query that went on in list mode is counted up to cm_end only)
    const int64_t cend = min(n, p.qs[q].cm_end);
    const int64_t r_lo = (int64_t)r * RS, r_hi = min(cend, r_lo + RS);
    if (P0 >= r_hi) continue;
    const TrajEntry* tr = p.traj + (size_t)q * kMaxTraj;
    const int nt = min(p.qs[q].ntraj, kMaxTraj);
    const double thr0 = p.qs[q].thr0;
    __syncthreads();  // every warp is done with the previous unit's pages and trajectory
    if (warp == kFW - 1) {
      // entries [ta, tb) change the threshold inside (r_start, r_hi): lanes 0/1
      // search the two ends (number of entries with pos < x)
      const int64_t x = lane ? r_hi : max(r_lo, P0);
      int lo2 = 0, hi2 = nt;
      if (lane < 2)
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (tr[mid].pos < x) lo2 = mid + 1; else hi2 = mid;
        }
      const int ta = __shfl_sync(kFull, lo2, 0), tb = __shfl_sync(kFull, lo2, 1);
      const int c = tb - ta;
      if (c <= kTS)
        for (int i = lane; i < c; i += 32) { s_pos[i] = tr[ta + i].pos; s_thr[1 + i] = tr[ta + i].thr; }
      if (lane == 0) {
        s_thr[0] = ta ? tr[ta - 1].thr : thr0;
        s_ctl[0] = ta;
        s_ctl[1] = c <= kTS ? c : -1;  // (-1: too many, read the global array)
      }
    }
    if (q != cur_q) {
      const double* glut = p.lut64 + (size_t)q * K * m;
      for (int i = tid; i < FP * m; i += kFW * 32) {
        const int s = i / m, j = i - s * m;
        const float v = s < F ? __double2float_rn(glut[p.fast_books[s] * m + j]) : 0.f;
        const uint32_t a0 = kPage * (1 + s / G::BPR) + j * 256 + (s % G::BPR) * 4 * G::R;
#pragma unroll
        for (int rr = 0; rr < G::R; rr += 4) sts_f32x4(a0 + rr * 4, v);
      }
      for (int i = tid; i < F * m; i += kFW * 32) {
        const int s = i / m, j = i - s * m;
        lut64f[i] = glut[p.fast_books[s] * m + j];
      }
      cur_q = q;
    }
    __syncthreads();
    uint32_t* surv = p.survivors ? p.survivors + (int64_t)q * p.words : nullptr;
    const int64_t w_lo = r_lo + warp * SW, w_hi = min(w_lo + SW, cend);
    const int64_t start = max(w_lo, P0);
    unsigned long long refined = 0;
    // local view of the trajectory: entry i of the unit (0 <= i < ne), the
    // threshold before entry 0 at index -1
    const int ta = s_ctl[0];
    const bool glob = s_ctl[1] < 0;
    const int ne = glob ? nt - ta : s_ctl[1];
    auto pos_at = [&](int i) -> int64_t { return glob ? tr[ta + i].pos : s_pos[i]; };
    auto thr_before = [&](int i) -> double {  // threshold of items in (pos[i-1], pos[i]]
      if (!glob) return s_thr[i];
      return ta + i ? tr[ta + i - 1].thr : thr0;
    };
    // number of the unit's entries with pos < i (items > pos use the entry's threshold)
    auto seg_of = [&](int64_t i) -> int {
      int lo2 = 0, hi2 = ne;
      while (lo2 < hi2) {
        const int mid = (lo2 + hi2) >> 1;
        if (pos_at(mid) < i) lo2 = mid + 1; else hi2 = mid;
      }
      return lo2;
    };
    int64_t t = w_lo + ((start - w_lo) / TILE) * TILE;
    int sg = seg_of(t);  // then advanced monotonically: each change point is crossed once
    double thr = thr_before(sg);
    int64_t next_pos = sg < ne ? pos_at(sg) : INT64_MAX;
    float lo, hi;
    // integer form of the certified test (fast sums are finite and >= 0, so
    // float order = bit order): x = bits(f) - bits(lo) is negative iff f < lo,
    // and 0 <= x < band iff float32 cannot decide (lo <= f < hi)
    uint32_t lo_b, band_w;
    auto set_thr = [&]() {
      certified_bounds(thr, F, lo, hi);
      lo_b = lo > 0.f ? __float_as_uint(lo) : 0u;  // (NaN / non-positive: nothing is below)
      band_w = (hi > 0.f ? __float_as_uint(hi) : 0u) - lo_b;
    };
    set_thr();
    uint4 a[V];  // the next tile's chunks (register double buffer)
    if (t < w_hi) {
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = ldg_stream(codes + t / IPC + lane + v * 32);
    }
    uint32_t cnt32 = 0;  // fast-path count of this lane (flushed below 2^31)
    for (; t < w_hi; t += TILE) {
      uint4 x[V];
#pragma unroll
      for (int v = 0; v < V; ++v) x[v] = a[v];
      if (t + TILE < w_hi) {
#pragma unroll
        for (int v = 0; v < V; ++v) a[v] = ldg_stream(codes + (t + TILE) / IPC + lane + v * 32);
      }
      // the tile's segment(s): one threshold unless a change point falls inside
      if (next_pos < t) {
        while (sg < ne && pos_at(sg) < t) ++sg;
        thr = thr_before(sg);
        next_pos = sg < ne ? pos_at(sg) : INT64_MAX;
        set_thr();
      }
      const bool split = next_pos < t + TILE - 1;
      const bool full = t >= start && t + TILE <= w_hi;
      if (full && !split && !surv) {
        // fast path: count only.  Pair sums run packed (FADD2), as in the filter.
        uint32_t c = 0, mn = 0xffffffffu;
#pragma unroll
        for (int pr = 0; pr < N / 2; ++pr) {
          float2 acc[FP];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int idx = 2 * pr + h, v = idx / IPC, j = idx % IPC;
            const uint32_t wd[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
#pragma unroll
            for (int s2 = 0; s2 < FP; ++s2) {
              const int byte = j * FP + s2;
              const uint32_t sel = 0x7604u | ((uint32_t)(byte & 3) << 4);
              const float val = lds_f32(__byte_perm(wd[byte >> 2], Lp[s2], sel));
              if (h == 0) acc[s2].x = val; else acc[s2].y = val;
            }
          }
#pragma unroll
          for (int h = 1; h < FP; h *= 2)
#pragma unroll
            for (int s2 = 0; s2 + h < FP; s2 += 2 * h) acc[s2] = __fadd2_rn(acc[s2], acc[s2 + h]);
          const uint32_t x0 = __float_as_uint(acc[0].x) - lo_b, x1 = __float_as_uint(acc[0].y) - lo_b;
          c += (x0 >> 31) + (x1 >> 31);
          mn = min(mn, min(x0, x1));
        }
        if (!__any_sync(kFull, mn < band_w)) {
          cnt32 += c;
          continue;
        }
      }
      // (rare) edge tiles, a threshold change inside the tile, near-ties, and
      // every tile when survivor bits are requested: per-item decisions
      const int64_t i0 = t + (int64_t)lane * N;
      unsigned long long bits = 0;
      // the lane's own threshold: its N consecutive items are walked in
      // order, the threshold moves only where a change point is crossed
      double th = thr;
      float l2 = lo, h2 = hi;
      int sgl = sg;
      int64_t nxt = INT64_MAX;  // items > nxt use the next entry's threshold
      if (split) {
        sgl = seg_of(i0);
        th = thr_before(sgl);
        certified_bounds(th, F, l2, h2);
        nxt = sgl < ne ? pos_at(sgl) : INT64_MAX;
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint32_t wd[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
#pragma unroll
        for (int j = 0; j < IPC; ++j) {
          float f = 0.f;
#pragma unroll
          for (int s2 = 0; s2 < FP; ++s2) {
            const int byte = j * FP + s2;
            const uint32_t sel = 0x7604u | ((uint32_t)(byte & 3) << 4);
            f += lds_f32(__byte_perm(wd[byte >> 2], Lp[s2], sel));
          }
          const int64_t i = i0 + v * IPC + j;
          if (i > nxt) {  // (split tiles only)
            while (sgl < ne && pos_at(sgl) < i) ++sgl;
            th = thr_before(sgl);
            certified_bounds(th, F, l2, h2);
            nxt = sgl < ne ? pos_at(sgl) : INT64_MAX;
          }
          if (i < start || i >= w_hi) continue;
          bool ref = f < l2;
          if (!ref && f < h2) ref = tuple_f64<FP>(chunk_tuple<FP>(x[v], j), lut64f, m, F) < th;
          if (ref) bits |= 1ull << (v * IPC + j);
        }
      }
      refined += (unsigned long long)__popcll(bits);
      if (surv && bits) {  // this lane's items are one contiguous, N-aligned run
        constexpr int W = N >= 32 ? N / 32 : 1;
#pragma unroll
        for (int h = 0; h < W; ++h) {
          const uint32_t wv = N >= 32 ? (uint32_t)(bits >> (32 * h))
                                      : (uint32_t)bits << (int)((i0 & 31));
          if (wv) atomicOr(surv + ((i0 + 32 * h) >> 5), wv);
        }
      }
    }
    refined += cnt32;  // (a warp slice holds < 2^31 items)
#pragma unroll
    for (int o = 16; o; o >>= 1) refined += __shfl_xor_sync(kFull, refined, o);
    if (lane == 0 && refined && p.refinements)
      atomicAdd(reinterpret_cast<unsigned long long*>(p.refinements + q), refined);
  }
}

// --------------------------------------------------------------------------
// host launch
// --------------------------------------------------------------------------
template <int FP>
cudaError_t launch_fp(const PipeParams& p, int filter_ctas, cudaStream_t s, cudaEvent_t* ev) {
  int launched = 0;  // kernels of this batch (icq_kernel_launches)
  using G = FGeo<FP>;
  // kernel attributes once per process (they are per function, not per launch)
  static cudaError_t attr[64];
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [&] {
    attr[dev] = [&] {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(icq_prologue_kernel<FP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kSmemWindow - kDynBase))) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(icq_filter_kernel<FP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kSmemWindow - kDynBase))) != cudaSuccess)
      return e;
    if ((e = cudaFuncSetAttribute(icq_count_kernel<FP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kSmemWindow - kDynBase))) != cudaSuccess)
      return e;
    return cudaFuncSetAttribute(icq_replay_kernel<FP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kSmemWindow - kDynBase));
    }();
  });
  if (attr[dev] != cudaSuccess) return attr[dev];
  const ProLayout pl = pro_layout(p.K, p.m, p.F, p.k);
  const RepLayout rl = rep_layout(p.K, p.m, p.F, p.k);
  cudaError_t e;
  if (ev) cudaEventRecord(ev[0], s);
  icq_prologue_kernel<FP><<<p.Q, kProThreads, pl.total, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++launched;
  if (ev) cudaEventRecord(ev[1], s);
  // filter / replay rounds: a query whose walk ran too long resumes in the
  // next round; finished queries cost the later launches nothing
  // refine / gather: units (query, range group) over a bounded grid (rounds
  // nobody was handed to cost a few thousand CTA exits, not Q x NR)
  const int64_t units = (int64_t)p.Q * p.NRG;
  const unsigned unit_grid = (unsigned)(units < 8192 ? (units < 1 ? 1 : units) : 8192);
  for (int r = 0; r < p.rounds; ++r) {
    PipeParams pr = p;
    pr.round = r;
    pr.last_round = r + 1 == p.rounds ? 1 : 0;
    if (r > 0 && (e = cudaMemsetAsync(p.pool_top, 0, sizeof(int32_t), s)) != cudaSuccess) return e;
    if (r > 0 && (e = cudaMemsetAsync(p.cl_top, 0, sizeof(unsigned long long), s)) != cudaSuccess)
      return e;
    icq_filter_kernel<FP><<<filter_ctas, kFW * 32, G::kSmemEnd - kDynBase, s>>>(pr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++launched;
    if (ev) cudaEventRecord(ev[2 + 3 * r], s);
    if (FP <= 8 && !p.exact_mode && p.count_used && r == 0 && p.NRD > 0) {
      // count-mode queries: the first round lists a prefix, without the fast test
      icq_dense_kernel<FP><<<p.Q * p.NRD, kFW * 32, (size_t)p.KP * p.m * sizeof(float), s>>>(pr);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++launched;
    }
    if (FP <= 8 && !p.exact_mode && p.count_used) {  // count-mode lists: possible insertions only
      icq_refine_kernel<FP><<<unit_grid, kFW * 32, (size_t)p.KP * p.m * sizeof(float), s>>>(pr);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++launched;
    }
    {  // the lists made contiguous per query, with float64 exact scores
      icq_cl_scan_kernel<FP><<<p.Q, 256, 0, s>>>(pr);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      ++launched;
      icq_cl_gather_kernel<FP><<<unit_grid, kFW * 32, (size_t)p.K * p.m * sizeof(double), s>>>(pr);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      ++launched;
    }
    if (ev) cudaEventRecord(ev[3 + 3 * r], s);
    icq_replay_kernel<FP><<<p.Q, kRW * 32, rl.total, s>>>(pr);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++launched;
    if (ev) cudaEventRecord(ev[4 + 3 * r], s);
  }
  for (int r = p.rounds; ev && r < kMaxRounds; ++r) {  // unused rounds: empty intervals
    cudaEventRecord(ev[2 + 3 * r], s);
    cudaEventRecord(ev[3 + 3 * r], s);
    cudaEventRecord(ev[4 + 3 * r], s);
  }
  if (FP <= 8 && !p.exact_mode && p.count_used) {  // refinement count of count-mode queries
    icq_count_kernel<FP><<<filter_ctas, kFW * 32, G::kSmemEnd - kDynBase, s>>>(p);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++launched;
  }
  if (ev) cudaEventRecord(ev[2 + 3 * kMaxRounds], s);
  count_kernel_launches(launched);
  return cudaSuccess;
}

}  // namespace icq

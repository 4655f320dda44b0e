// icq_scan.cu — K2..K5 fused: fast-pass scan, in-order margin pruning,
// refinement and top-k for one query per CTA.
//
// Reference semantics: search_two_step, /root/reference/pkg/src/icq/search.py:112-165
//   heap seeded with ids 0..k-1 scored exactly                      (:141-143)
//   element i >= k refined iff fast[i] < bound + sigma, where bound is the
//   FAST score of the current heap maximum by (exact, id)            (:149, :154)
//   inserted iff exact[i] < exact(heap max) (strict)                 (:152-153)
//   result: the heap sorted ascending by (score, id)                 (:156)
// search_exact (:97-109) is the same kernel with the fast set = all books and
// sigma = 0 (then fast == exact and the prune predicate is the top-k test).
//
// One CTA (288 threads, one per SM) owns one query and walks the database in
// order in two phases:
//
// Phase 1 — dense prologue (insertion-heavy start, ~k*ln(i/k) insertions).
//   All 9 warps score chunks of items exactly in float64 (rows from HBM, the
//   float64 LUT in shared memory); warp 0 then replays the reference loop
//   over the chunk with float64 compares only.  Runs until a whole segment
//   sees few insertions.
//
// Phase 2 — pipelined scan (the streaming hot path).
//   warps 1..8 SCAN   stream the fast-code block (16-byte loads, two segments
//                     of register prefetch), gather |F| float32 entries per item
//                     from lane-private replicated LUT pages (conflict-free:
//                     entry j of book s for lane l sits in bank l; its address
//                     is ONE byte_perm of the code word), publish per-group and
//                     per-warp minima, and compact the items under the replay's
//                     published threshold into an ordered per-warp candidate
//                     list whose full code rows arrive by cp.async; their
//                     float64 fast/exact scores are computed one segment later,
//                     so the order-independent work never waits on memory.
//   warp 0     REPLAY consumes slots strictly in database order against the
//                     LIVE bound: the candidate lists of a segment are decided
//                     32 at a time with certified float32 thresholds (float64
//                     only for near-ties); if an insertion lifts the bound
//                     above the threshold a list was filtered with, the rest of
//                     that segment is re-derived from the codes (exact, rare).
//                     Insertions update a register heap.  Everything compared
//                     is float64 and bitwise the reference's.
//   Slots are handed over with mbarriers (full: 256 scan-thread arrivals
//   after the cp.async rows landed; empty: 32 replay-lane arrivals).
#include "icq_types.cuh"

namespace icq {

template <int FP>
struct Geo {
  static constexpr int R = FP <= 4 ? 32 : (FP == 8 ? 16 : 8);  // replicas per entry
  static constexpr int BPR = 64 / R;                             // book slots per 256-B row
  static constexpr int P = (FP + BPR - 1) / BPR;                 // 64 KiB pages
  static constexpr int IPC = 16 / FP;                            // items per 16-B chunk
  static constexpr int V = FP >= 4 ? 4 : 2;                      // chunks per lane per segment
  static constexpr int NC = kNS * 32 * V;                        // groups (chunks) per segment
  static constexpr int S = NC * IPC;                             // items per segment
};

constexpr int kPubR = 3;             // prefetch threshold covers the next kPubR insertions
constexpr int kDenseStopIns = 6;     // leave the prologue once a segment sees <= this many
constexpr int kReplayBlock = 4;      // segments the replay consumes per probe (< slots)
constexpr int kPrefetchSeg = 6;      // L2 bulk-prefetch distance of the code stream (segments)
#define kInf (__int_as_float(0x7f800000))

// --------------------------------------------------------------------------
// float64 scores in the reference's order (search.py:94, see ref_row_sum)
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

__device__ __forceinline__ Row smem_row(const uint8_t* p, int KP) {
  Row r;
  r.w[0] = r.w[1] = r.w[2] = r.w[3] = 0;
  if (KP == 16) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    r.w[0] = v.x; r.w[1] = v.y; r.w[2] = v.z; r.w[3] = v.w;
  } else if (KP == 8) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    r.w[0] = v.x; r.w[1] = v.y;
  } else {
    r.w[0] = *reinterpret_cast<const uint32_t*>(p);
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

// (exact, id) ordering of the reference heap (search.py:140: keys (-exact, -id))
__device__ __forceinline__ bool key_gt(double e1, int32_t i1, double e2, int32_t i2) {
  // branch-free (no short-circuit): the replay warp's hot compares must not
  // open divergence regions
  const bool gt = e1 > e2, eq = e1 == e2, ig = i1 > i2;
  return gt | (eq & ig);
}

// Replace the maximum (entry 0) of a descending-sorted heap in shared memory.
__device__ void heap_replace_max(double* he, double* hf, int32_t* hi, int k, double e, int32_t id,
                                 double f, int lane) {
  int g = 0;
#pragma unroll 4
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
// entries live in warp-0 registers in a BLOCKED layout (lane l holds entries
// 4l..4l+3): an insertion shifts registers locally, moves only the lane
// boundary entry with one shuffle per field, and finds its position with one
// __reduce_add_sync.  Larger k falls back to shared memory.  A warp-uniform
// copy of the top two entries gives the new maximum (T and bound) after an
// insertion with plain per-lane ALU work.
constexpr int kRegHeapRegs = 4;
constexpr int kTopC = 2;  // larger caches push the replay state out of registers
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
  // max fast score over entries 0..R (R < kRegHeapRegs: lane 0 holds them)
  __device__ __forceinline__ double top_fast_max(int R) const {
    double a = 0.0;
    if (reg) {
      a = f[0];
#pragma unroll
      for (int j = 1; j < kRegHeapRegs; ++j)
        if (j <= R && j < k) a = fmax(a, f[j]);
      a = __shfl_sync(0xffffffffu, a, 0);
    } else {
      a = hf[0];
      for (int j = 1; j <= R && j < k; ++j) a = fmax(a, hf[j]);
    }
    return a;
  }
  // largest fast score over the whole heap (warp-uniform result)
  __device__ __forceinline__ double max_fast_all(int lane) const {
    double a = 0.0;
    if (reg) {
#pragma unroll
      for (int r = 0; r < kRegHeapRegs; ++r)
        if (kRegHeapRegs * lane + r < k) a = fmax(a, f[r]);
    } else {
      for (int i = lane; i < k; i += 32) a = fmax(a, hf[i]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    return a;
  }
  __device__ __forceinline__ void replace_max(double xe, int32_t xid, double xf, int lane) {
    // 1. uniform top cache: drop entry 0, insert x if it ranks inside the prefix
    double le = ue[0];  // smallest cached entry (static indexing keeps it in registers)
    int32_t li = ui[0];
#pragma unroll
    for (int j = 1; j < kTopC; ++j)
      if (j == uc - 1) { le = ue[j]; li = ui[j]; }
    const bool in = uc >= 2 && key_gt(xe, xid, le, li);
    // in place, top down: slot j takes old[j+1] while that still outranks x,
    // then x, then keeps old[j]
#pragma unroll
    for (int j = 0; j < kTopC; ++j) {
      const int jn = j + 1 < kTopC ? j + 1 : j;
      const bool above_gt = (j + 1 < uc) && key_gt(ue[jn], ui[jn], xe, xid);
      const bool here_gt = j == 0 ? true : ((j < uc) && key_gt(ue[j], ui[j], xe, xid));
      if (above_gt) { ue[j] = ue[jn]; uf[j] = uf[jn]; ui[j] = ui[jn]; }
      else if (here_gt && in) { ue[j] = xe; uf[j] = xf; ui[j] = xid; }
    }
    if (!in) --uc;
    // 2. the full sorted array (lanes or shared memory), off the critical path
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
    // new[i] = old[i+1] for i < g, x at g, unchanged above; old[i+1] of the
    // lane's last register is the next lane's first
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

// cp.async helpers (rows of candidate items into the slot)
__device__ __forceinline__ void cp_async_row(uint32_t dst, const void* src, int bytes) {
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// --------------------------------------------------------------------------
// shared context
// --------------------------------------------------------------------------
struct Ctx {
  const ScanParams* p;
  uint8_t* dsm;
  uint32_t dbase;
  double* lut;  // float64 LUT [K][m]
  double* he;
  double* hf;
  int32_t* hi;
  uint32_t ctrl;
  bool pw;
  bool wide;
  __device__ __forceinline__ uint8_t* at(uint32_t abs) const { return dsm + (abs - dbase); }
};

// ctrl block: [0,64) full[8]  [64,128) empty[8]  128 pub_thr  132 prologue flag
constexpr uint32_t kCtrlBytes = 160;
constexpr int kMaxSlots = 8;
// slot meta block: cnt[8] int32, pub[8] float, wmin[8] float
constexpr uint32_t kMetaBytes = 128;

// Replay state (warp 0 only; warp-uniform registers)
struct Live {
  double T64, bound64, thr64;
  float lo, hi;
  int64_t refinements, insertions, candidates, certified;
  int64_t wait_cycles;  // replay time spent waiting for the scan warps
  int64_t t_score, t_decide, t_insert;  // prologue breakdown (warp 0 clocks)
  int64_t fallback_segments;            // segments re-derived from the codes
  int64_t t_active, t_fallback;         // phase-2 replay breakdown (clocks)
  int64_t n_rounds;                     // prologue decision rounds
  WarpHeap H;
};

// float64 state after a heap change (all the prologue needs)
__device__ __forceinline__ void live_update64(Live& L, double sigma) {
  L.T64 = L.H.top_e();
  L.bound64 = L.H.top_f();
  L.thr64 = __dadd_rn(L.bound64, sigma);
}

// + certified float32 thresholds for the phase-2 filter
__device__ __forceinline__ void live_update(Live& L, int F, double sigma, bool wide) {
  live_update64(L, sigma);
  if (wide) {
    L.lo = -kInf;
    L.hi = kInf;
  } else {
    certified_bounds(L.thr64, F, L.lo, L.hi);
  }
}

// Publish the scan warps' candidate-list threshold: the bound stays <= the
// max fast score over the top kPubR+1 heap entries (+ sigma per insertion)
// for the next kPubR insertions, so lists filtered with it stay complete.
__device__ __forceinline__ void publish_prefetch(const Live& L, const Ctx& c, int F, double sigma,
                                                 bool wide, int lane) {
  const double a = L.H.top_fast_max(kPubR);
  float lo2, hi2;
  certified_bounds(__dadd_rn(a, sigma * (kPubR + 1)), F, lo2, hi2);
  if (lane == 0) {
    volatile float* pub = reinterpret_cast<volatile float*>(c.at(c.ctrl + 128));
    *pub = wide ? kInf : fmaxf(hi2, L.hi);
  }
}

__device__ __forceinline__ void record_survivor(uint32_t* surv, int64_t id) {
  if (surv) atomicOr(surv + (id >> 5), 1u << (id & 31));
}

// --------------------------------------------------------------------------
// Phase 1: dense prologue (all warps score, warp 0 decides in float64)
// --------------------------------------------------------------------------
template <int FP>
__device__ __forceinline__ int64_t dense_prologue(const Ctx& c, Live& L, int tid, int warp,
                                                  int lane) {
  using G = Geo<FP>;
  const ScanParams& p = *c.p;
  const int64_t n = p.n;
  const int k = p.k;
  const int C = p.dense_chunk;
  double* df = reinterpret_cast<double*>(c.at(p.off_slots));
  double* de = df + C;
  volatile int32_t* flag = reinterpret_cast<volatile int32_t*>(c.at(c.ctrl + 132));
  uint32_t* surv = p.survivors ? p.survivors + (int64_t)blockIdx.x * p.words : nullptr;
  int64_t pos = k;
  int seg_ins = 0;
  while (pos < n) {
    const int64_t end = min(n, (pos / C + 1) * C);
    const int cnt = (int)(end - pos);
    const long long tc0 = clock64();
    const double fcut = p.sigma == 0.0 ? *reinterpret_cast<volatile double*>(c.at(c.ctrl + 136))
                                       : __longlong_as_double(0x7ff0000000000000LL);
    for (int i0 = 0; i0 < cnt; i0 += kThreads * 8) {
      Row rows[8];  // issue all row loads first, then score (one memory latency per round)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + tid + r * kThreads;
        if (i < cnt) rows[r] = load_row(p.codes_full, p.KP, pos + i);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int i = i0 + tid + r * kThreads;
        if (i < cnt) {
          const double fi = fast64(c.lut, p.m, p.F, c.pw, p.fast_books, rows[r]);
          df[i] = fi;
          // never refined in this chunk (fi >= every reachable bound): no exact score needed
          de[i] = (fi < fcut || !(fcut == fcut)) ? exact64(c.lut, p.m, p.K, c.pw, rows[r])
                                                 : __longlong_as_double(0x7ff0000000000000LL);
        }
      }
    }
    __syncthreads();
    const long long tc1 = clock64();
    L.t_score += tc1 - tc0;
    if (warp == 0) {
      // 128-item windows: the four 32-item sub-batches are tested together
      // (independent ballots), so one serial round covers a whole window up
      // to its first insertion (search.py:148-154 applied in order).
      constexpr int U = 4;
      for (int w0 = 0; w0 < cnt; w0 += 32 * U) {
        double f[U], e[U];
        bool valid[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = w0 + u * 32 + lane;
          valid[u] = i < cnt;
          f[u] = valid[u] ? df[i] : 0.0;
          e[u] = valid[u] ? de[i] : 0.0;
        }
        uint32_t done[U] = {0, 0, 0, 0};
        for (;;) {
          ++L.n_rounds;
          uint32_t rm[U], im[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const bool refined = valid[u] && !((done[u] >> lane) & 1u) && (f[u] < L.thr64);
            rm[u] = __ballot_sync(0xffffffffu, refined);
            im[u] = __ballot_sync(0xffffffffu, refined && (e[u] < L.T64));
          }
          int uf = U;  // first sub-batch holding an insertion
#pragma unroll
          for (int u = U - 1; u >= 0; --u)
            if (im[u]) uf = u;
          int first = 31;
          double ne = 0.0, nf = 0.0;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            uint32_t dec = 0;
            if (u < uf) dec = 0xffffffffu;
            if (u == uf) {
              first = __ffs(im[u]) - 1;
              dec = 0xffffffffu >> (31 - first);
              ne = __shfl_sync(0xffffffffu, e[u], first);
              nf = __shfl_sync(0xffffffffu, f[u], first);
            }
            const int nr = __popc(rm[u] & dec);
            L.refinements += nr;
            L.candidates += nr;
            if (surv && ((rm[u] & dec) >> lane & 1u)) record_survivor(surv, pos + w0 + u * 32 + lane);
            done[u] |= dec;
          }
          if (uf == U) break;
          const long long ti0 = clock64();
          L.H.replace_max(ne, (int32_t)(pos + w0 + uf * 32 + first), nf, lane);
          live_update64(L, p.sigma);
          L.t_insert += clock64() - ti0;
          ++L.insertions;
          ++seg_ins;
        }
      }
      L.t_decide += clock64() - tc1;
      // sigma == 0: the bound never exceeds the heap's largest fast score, so
      // items at or above it need no exact score in the next chunk
      const double hmax = L.H.max_fast_all(lane);
      if (lane == 0) *reinterpret_cast<volatile double*>(c.at(c.ctrl + 136)) = hmax;
      live_update(L, p.F, p.sigma, c.wide);
      publish_prefetch(L, c, p.F, p.sigma, c.wide, lane);
      // stop at a segment boundary once the insertion rate has dropped
      bool more = end < n;
      if (end % G::S == 0) {
        if (seg_ins <= kDenseStopIns) more = false;
        seg_ins = 0;
      }
      if (lane == 0) *flag = more ? 1 : 0;
    }
    __syncthreads();
    pos = end;
    if (!*flag) break;
    __syncthreads();  // chunk buffers are rewritten next round
  }
  return pos;
}

// --------------------------------------------------------------------------
// Phase 2, SCAN warps
// --------------------------------------------------------------------------
template <int FP>
__device__ __forceinline__ void scan_role(const Ctx& c, int w, int lane, int64_t seg0) {
  using G = Geo<FP>;
  constexpr int IPC = G::IPC;
  constexpr int V = G::V;
  constexpr int S = G::S;
  const ScanParams& p = *c.p;
  uint32_t L[FP];
#pragma unroll
  for (int s = 0; s < FP; ++s)
    L[s] = ((uint32_t)(1 + s / G::BPR) << 16) |
           (uint32_t)((s % G::BPR) * 4 * G::R + (lane % G::R) * 4);

  const uint4* codes = reinterpret_cast<const uint4*>(p.codes_fast);
  const int cbase = w * 32 * V + lane;  // chunk (group) v of this lane: cbase + 32 v
  const int64_t nseg = p.nseg;
  const int rowb = p.KP < 4 ? 4 : p.KP;
  const volatile float* pub = reinterpret_cast<const volatile float*>(c.at(c.ctrl + 128));

  uint4 a[V], b[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    a[v] = seg0 < nseg ? ldg_stream(codes + seg0 * G::NC + cbase + 32 * v) : make_uint4(0, 0, 0, 0);
    b[v] = seg0 + 1 < nseg ? ldg_stream(codes + (seg0 + 1) * G::NC + cbase + 32 * v)
                           : make_uint4(0, 0, 0, 0);
  }
  int slot = 0;       // ring position and phase parity, advanced incrementally
  uint32_t par = 0;   // (a runtime modulo costs ~80 cycles per segment)
  for (int64_t t = seg0; t < nseg; ++t, slot = (slot + 1 == p.nb) ? 0 : slot + 1,
               par ^= (slot == 0) ? 1u : 0u) {
    uint4 x[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      x[v] = a[v];
      a[v] = b[v];
    }
    if (t + 2 < nseg) {
#pragma unroll
      for (int v = 0; v < V; ++v) b[v] = ldg_stream(codes + (t + 2) * G::NC + cbase + 32 * v);
    }
    // this warp's chunks of a segment are one contiguous 32*V*16-byte run:
    // pull it into L2 kPrefetchSeg segments ahead so the register prefetch hits L2
    if (lane == 0 && t + kPrefetchSeg < nseg)
      prefetch_l2_bulk(codes + (t + kPrefetchSeg) * G::NC + w * 32 * V, 32 * V * 16);
    float f[V][IPC];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t wd[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
#pragma unroll
      for (int j = 0; j < IPC; ++j) {
        float acc[FP];
#pragma unroll
        for (int s = 0; s < FP; ++s) {
          const int byte = j * FP + s;
          const uint32_t sel = 0x7604u | ((uint32_t)(byte & 3) << 4);
          acc[s] = lds_f32(__byte_perm(wd[byte >> 2], L[s], sel));
        }
#pragma unroll
        for (int h = 1; h < FP; h *= 2)
#pragma unroll
          for (int s = 0; s + h < FP; s += 2 * h) acc[s] = acc[s] + acc[s + h];
        f[v][j] = acc[0];
      }
    }
    const int64_t base = t * S;
    // padding past n never enters the replay; only the last segment has any,
    // and 32-bit local indices keep the (predicated) test cheap
    const int nvalid = (int)min((int64_t)S, p.n - base);
    if (nvalid < S) {
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int j = 0; j < IPC; ++j)
          if ((cbase + 32 * v) * IPC + j >= nvalid) f[v][j] = kInf;
    }
    float lm = kInf;
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int j = 0; j < IPC; ++j) lm = fminf(lm, f[v][j]);
    // non-negative floats order like their bit patterns: one redux for the warp min
    const float wm = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(lm)));

    mbar_wait(c.ctrl + 64 + 8 * slot, par ^ 1u);  // empty[slot]
    const uint32_t sb = p.off_slots + (uint32_t)slot * p.slot_bytes;
    sts_f32(sb + p.so_lmin + (uint32_t)(w * 32 + lane) * 4, lm);

    // ordered candidate list: items with f < pub, in item order (v, lane, j)
    const float pt = *pub;
    int total = 0;
    if (__any_sync(0xffffffffu, lm < pt)) {
      int32_t* eid = reinterpret_cast<int32_t*>(c.at(sb + p.so_eid));
      float* ef32 = reinterpret_cast<float*>(c.at(sb + p.so_ef32));
      // one lane prefix scan for all V chunks: per-chunk hit counts packed in
      // kFB-bit fields (32 lanes * IPC hits fit), 5 shuffle steps in total
      constexpr int kFB = 32 / V;
      constexpr uint32_t kFM = (kFB == 32) ? 0xffffffffu : ((1u << kFB) - 1u);
      uint32_t masks[V];
      uint32_t packed = 0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < IPC; ++j) mask |= (f[v][j] < pt ? 1u : 0u) << j;
        masks[v] = mask;
        packed |= (uint32_t)__popc(mask) << (kFB * v);
      }
      uint32_t incl = packed;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - packed;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        uint32_t mask = masks[v];
        int pos = total + (int)((excl >> (kFB * v)) & kFM);
        total += (int)((tot >> (kFB * v)) & kFM);
        while (mask) {
          const int j = __ffs(mask) - 1;
          mask &= mask - 1;
          if (pos < p.cw) {
            const int e = w * p.cw + pos;
            const int64_t id = base + (int64_t)(cbase + 32 * v) * IPC + j;
            eid[e] = (int32_t)id;
            float fj = f[v][0];
#pragma unroll
            for (int jj = 1; jj < IPC; ++jj)
              if (jj == j) fj = f[v][jj];
            ef32[e] = fj;
            cp_async_row(sb + p.so_erow + (uint32_t)e * 16, p.codes_full + id * p.KP, rowb);
          }
          ++pos;
        }
      }
    }
    if (lane == 0) {
      volatile int32_t* meta = reinterpret_cast<volatile int32_t*>(c.at(sb));
      meta[w] = total;
      reinterpret_cast<volatile float*>(meta)[8 + w] = pt;
      reinterpret_cast<volatile float*>(meta)[16 + w] = wm;
    }
    // full[slot] completes once every scan thread arrived AND its row copies
    // landed — the scan warps never wait for their own cp.async traffic
    mbar_arrive_cp_async(c.ctrl + 8 * slot);
    mbar_arrive(c.ctrl + 8 * slot);
  }
  cp_async_wait<0>();
}

// --------------------------------------------------------------------------
// Phase 2, REPLAY warp
// --------------------------------------------------------------------------
// One decision round over up to 32 items in database order (lane order).
// cand/fv: float32 candidate test input; f64/e64: exact scores if `have`,
// else loaded here.  Returns the lane of the insertion (or -1); lanes up to
// it (or all) are decided and recorded.
struct Decided {
  int first;       // inserting lane or -1
  uint32_t done;   // lanes decided in this round
};

template <bool kCertified>
__device__ __forceinline__ Decided decide_round(Live& L, const Ctx& c, int lane, bool cand,
                                                float fv, int64_t id, bool& have, double& f64,
                                                double& e64, uint32_t* surv) {
  const ScanParams& p = *c.p;
  const uint32_t cmask = __ballot_sync(0xffffffffu, cand);
  Decided d{-1, 0xffffffffu};
  if (!cmask) return d;
  bool refined = false, certified = false;
  if (cand) {
    if (kCertified && !c.wide && fv < L.lo) {
      refined = true;
    } else {
      if (!have) {
        const Row r = load_row(p.codes_full, p.KP, id);
        f64 = fast64(c.lut, p.m, p.F, c.pw, p.fast_books, r);
        e64 = exact64(c.lut, p.m, p.K, c.pw, r);
        have = true;
      }
      certified = true;
      refined = f64 < L.thr64;
    }
    if (refined && !have) {
      const Row r = load_row(p.codes_full, p.KP, id);
      f64 = fast64(c.lut, p.m, p.F, c.pw, p.fast_books, r);
      e64 = exact64(c.lut, p.m, p.K, c.pw, r);
      have = true;
    }
  }
  const bool ins = refined && (e64 < L.T64);
  const uint32_t rmask = __ballot_sync(0xffffffffu, refined);
  const uint32_t imask = __ballot_sync(0xffffffffu, ins);
  const uint32_t cert = __ballot_sync(0xffffffffu, certified);
  const int first = imask ? __ffs(imask) - 1 : 31;
  const uint32_t decided = imask ? (0xffffffffu >> (31 - first)) : 0xffffffffu;
  L.refinements += __popc(rmask & decided);
  L.candidates += __popc(cmask & decided);
  L.certified += __popc(cert & decided);
  if (refined && ((decided >> lane) & 1u)) record_survivor(surv, id);
  d.done = decided;
  if (imask) {
    d.first = first;
    const double ne = __shfl_sync(0xffffffffu, e64, first);
    const double nf = __shfl_sync(0xffffffffu, f64, first);
    const int32_t nid = (int32_t)__shfl_sync(0xffffffffu, (int32_t)id, first);
    L.H.replace_max(ne, nid, nf, lane);
    live_update(L, p.F, p.sigma, c.wide);
    ++L.insertions;
  }
  return d;
}

// Exact fallback for items >= pos of one segment: groups gated by their
// minimum, float32 scores recomputed from the codes with this warp's own
// page replicas, float64 scores from the rows.
template <int FP>
__device__ void replay_fallback(Live& L, const Ctx& c, int lane, int64_t t, uint32_t sb,
                                int64_t pos, uint32_t* surv) {
  using G = Geo<FP>;
  constexpr int IPC = G::IPC;
  constexpr int GPB = 32 / IPC;  // groups per 32-lane batch
  const ScanParams& p = *c.p;
  const int64_t base = t * G::S;
  const uint4* codes = reinterpret_cast<const uint4*>(p.codes_fast);
  const float* lmin = reinterpret_cast<const float*>(c.at(sb + p.so_lmin));
  uint32_t Lp[FP];
#pragma unroll
  for (int s = 0; s < FP; ++s)
    Lp[s] = ((uint32_t)(1 + s / G::BPR) << 16) |
            (uint32_t)((s % G::BPR) * 4 * G::R + (lane % G::R) * 4);
  // float32 fast score of item jj of a 16-byte code chunk (this lane's replica)
  auto item_f32 = [&](const uint4& x, int jj) {
    const uint32_t wd[4] = {x.x, x.y, x.z, x.w};
    float out = kInf;
#pragma unroll
    for (int j2 = 0; j2 < IPC; ++j2) {
      if (j2 == jj) {
        float a2[FP];
#pragma unroll
        for (int s = 0; s < FP; ++s) {
          const int byte = j2 * FP + s;
          const uint32_t sel = 0x7604u | ((uint32_t)(byte & 3) << 4);
          a2[s] = lds_f32(__byte_perm(wd[byte >> 2], Lp[s], sel));
        }
#pragma unroll
        for (int h = 1; h < FP; h *= 2)
#pragma unroll
          for (int s = 0; s + h < FP; s += 2 * h) a2[s] = a2[s] + a2[s + h];
        out = a2[0];
      }
    }
    return out;
  };
  ++L.fallback_segments;
  // groups in 32-group rounds; only those holding items >= pos
  const int g_first = (int)((pos - base) / IPC);
  for (int r0 = (g_first / 32) * 32; r0 < G::NC; r0 += 32) {
    const int gl = r0 + lane;
    // gate chunk gl by the minimum of the scan lane that produced it
    // (chunk gl = w*32V + v*32 + l)
    const float gv = lmin[(gl / (32 * G::V)) * 32 + (gl % 32)];
    uint32_t gm = __ballot_sync(0xffffffffu, gl >= g_first && (c.wide || gv < L.hi));
    while (gm) {
      const int gi = lane / IPC;
      const int j = lane % IPC;
      const int ngrp = min(GPB, __popc(gm));
      const int mygrp = gi < ngrp ? (int)__fns(gm, 0, gi + 1) : -1;
      int lastgrp = (int)__fns(gm, 0, ngrp);
      const int cc = r0 + (mygrp < 0 ? 0 : mygrp);
      const int64_t id = base + (int64_t)cc * IPC + j;
      const bool valid = mygrp >= 0 && id >= pos && id < p.n;
      // recompute the float32 fast score of this item from its code chunk
      const float fv = valid ? item_f32(__ldg(codes + t * G::NC + cc), j) : kInf;
      bool have = false;
      double f64 = 0.0, e64 = 0.0;
      uint32_t done = 0;
      for (;;) {
        const bool cand = valid && !((done >> lane) & 1u) && (c.wide || fv < L.hi);
        const Decided d = decide_round<true>(L, c, lane, cand, fv, id, have, f64, e64, surv);
        done |= d.done;
        if (d.first < 0) break;
        // threshold moved: cut the batch after the inserting item's group
        const int gfirst = __shfl_sync(0xffffffffu, mygrp, d.first);
        done |= __ballot_sync(0xffffffffu, mygrp > gfirst);
        lastgrp = gfirst;
      }
      const uint32_t later = (lastgrp >= 31) ? 0u : (0xffffffffu << (lastgrp + 1));
      gm = later & __ballot_sync(0xffffffffu, gl >= g_first && (c.wide || gv < L.hi));
    }
  }
}

template <int FP>
__device__ void replay_segment(Live& L, const Ctx& c, int lane, int64_t t, uint32_t sb,
                               uint32_t* surv);

template <int FP>
__device__ __forceinline__ void replay_role(const Ctx& c, Live& L, int lane, int64_t seg0) {
  using G = Geo<FP>;
  const ScanParams& p = *c.p;
  const int F = p.F;
  const int64_t n = p.n;
  const bool wide = c.wide;
  uint32_t* surv = p.survivors ? p.survivors + (int64_t)blockIdx.x * p.words : nullptr;
  const int cw = p.cw;

  // Slots are consumed in blocks of kReplayBlock segments: all waits first,
  // then ONE meta probe (lane -> (segment lane/8, scan warp lane%8)) decides
  // whether anything in the block can hold a candidate under the live bound;
  // blocks without candidates cost a few waits and one ballot.
  const int kB = min(kReplayBlock, p.nb);  // never more slots than the ring holds
  int slot0 = 0;
  uint32_t par0 = 0;
  for (int64_t t0 = seg0; t0 < p.nseg; t0 += kB) {
    const int nblk = (int)min((int64_t)kB, p.nseg - t0);
    const long long tw = clock64();
    {
      int s = slot0;
      uint32_t pr = par0;
      for (int j = 0; j < nblk; ++j) {
        mbar_wait(c.ctrl + 8 * s, pr);  // full[s]
        if (++s == p.nb) { s = 0; pr ^= 1u; }
      }
    }
    L.wait_cycles += clock64() - tw;
    const int64_t ins0 = L.insertions;
    const int jl = lane >> 3;  // kNS == 8 warps per segment
    int sl = slot0 + jl;
    if (sl >= p.nb) sl -= p.nb;
    const float pwm = jl < nblk ? __int_as_float(reinterpret_cast<const int32_t*>(
                                      c.at(p.off_slots + (uint32_t)sl * p.slot_bytes))[16 + (lane & 7)])
                                : kInf;
    const bool any = __ballot_sync(0xffffffffu, jl < nblk && (wide || pwm < L.hi)) != 0 &&
                     !(p.debug & 1);
    for (int j = 0; j < nblk; ++j) {
      if (any) replay_segment<FP>(L, c, lane, t0 + j, p.off_slots + (uint32_t)slot0 * p.slot_bytes,
                                  surv);
      __syncwarp();
      mbar_arrive(c.ctrl + 64 + 8 * slot0);  // empty[slot]: hand the slot back at once
      if (++slot0 == p.nb) { slot0 = 0; par0 ^= 1u; }
    }
    if (L.insertions != ins0) publish_prefetch(L, c, F, p.sigma, wide, lane);
  }
}

// One segment of phase 2 in database order (called by the replay warp).
template <int FP>
__device__ void replay_segment(Live& L, const Ctx& c, int lane, int64_t t, uint32_t sb,
                               uint32_t* surv) {
  using G = Geo<FP>;
  const ScanParams& p = *c.p;
  const int F = p.F;
  const int64_t n = p.n;
  const bool wide = c.wide;
  const int cw = p.cw;
  {
    const int64_t base = t * G::S;
    // per-warp meta (uniform): list length, threshold the list was cut at, minimum
    const int32_t* meta = reinterpret_cast<const int32_t*>(c.at(sb));
    const int mcnt = lane < kNS ? meta[lane] : 0;
    const float mpub = lane < kNS ? __int_as_float(meta[8 + lane]) : kInf;
    const float mwm = lane < kNS ? __int_as_float(meta[16 + lane]) : kInf;
    auto incomplete = [&](float hi) {  // warps whose list may miss a candidate at hi
      return __ballot_sync(0xffffffffu, lane < kNS && (wide || mwm < hi) &&
                                            (wide || mpub < hi || mcnt > cw));
    };
    const uint32_t active = __ballot_sync(0xffffffffu, lane < kNS && (wide || mwm < L.hi));
    const long long ta = clock64();
    if (active) {
      if (incomplete(L.hi)) {
        replay_fallback<FP>(L, c, lane, t, sb, base, surv);
        L.t_fallback += clock64() - ta;
      } else {
        // concatenated per-warp lists, in item order; every lane reads the 8
        // list lengths itself (uniform loads) to map lane -> (warp, entry)
        int cnt8[kNS];
#pragma unroll
        for (int q = 0; q < kNS; ++q) cnt8[q] = min(meta[q], cw);
        int total = 0;
#pragma unroll
        for (int q = 0; q < kNS; ++q) total += cnt8[q];
        const int32_t* eid = reinterpret_cast<const int32_t*>(c.at(sb + p.so_eid));
        const float* ef32 = reinterpret_cast<const float*>(c.at(sb + p.so_ef32));
        int64_t fb_from = -1;  // fallback start after an insertion lifts the bound
        for (int b0 = 0; b0 < total; b0 += 32) {
          const int i = b0 + lane;
          int w = 0, start_w = 0, acc = 0;
#pragma unroll
          for (int q = 0; q < kNS; ++q) {
            if (i >= acc && i < acc + cnt8[q]) { w = q; start_w = acc; }
            acc += cnt8[q];
          }
          const bool valid = i < total;
          const int ent = w * cw + (i - start_w);
          const int64_t id = valid ? (int64_t)eid[ent] : 0;
          const float fv = valid ? ef32[ent] : kInf;
          // float64 scores of current candidates from the row the scan warps
          // copied into the slot (others are loaded on demand)
          double f64 = 0.0, e64 = 0.0;
          bool have = false;
          if (valid && (wide || fv < L.hi)) {
            const Row r = smem_row(c.at(sb + p.so_erow + (uint32_t)ent * 16), p.KP);
            f64 = fast64(c.lut, p.m, F, c.pw, p.fast_books, r);
            e64 = exact64(c.lut, p.m, p.K, c.pw, r);
            have = true;
          }
          uint32_t done = 0;
          for (;;) {
            const bool cand = valid && !((done >> lane) & 1u) && (wide || fv < L.hi) && id < n;
            const Decided d = decide_round<true>(L, c, lane, cand, fv, id, have, f64, e64, surv);
            done |= d.done;
            if (d.first < 0) break;
            // the bound moved: lists cut at a lower threshold may now miss items
            if (incomplete(L.hi)) {
              fb_from = __shfl_sync(0xffffffffu, id, d.first) + 1;
              break;
            }
          }
          if (fb_from >= 0) break;
        }
        if (fb_from >= 0 && fb_from < base + G::S) {
          const long long tf = clock64();
          replay_fallback<FP>(L, c, lane, t, sb, fb_from, surv);
          L.t_fallback += clock64() - tf;
        }
      }
      L.t_active += clock64() - ta;
    }
  }
}

// --------------------------------------------------------------------------
// the kernel
// --------------------------------------------------------------------------
template <int FP>
__global__ void __launch_bounds__(kThreads, 1) icq_scan_kernel(const ScanParams p) {
  using G = Geo<FP>;
  extern __shared__ __align__(16) uint8_t dsm[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int q = blockIdx.x;

  // The lane-private pages sit at absolute 64 KiB boundaries; the planned
  // layout assumes the dynamic window starts at kDynBase.
  uint32_t dyn_size;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn_size));
  const uint32_t dbase = smem_addr(dsm);
  if (dbase != kDynBase || dbase + dyn_size < p.smem_end) {
    if (tid == 0) atomicExch(p.error, 1);
    return;
  }
  Ctx c;
  c.p = &p;
  c.dsm = dsm;
  c.dbase = dbase;
  c.lut = reinterpret_cast<double*>(c.at(p.off_lut64));
  c.he = reinterpret_cast<double*>(c.at(p.off_heap_e));
  c.hf = reinterpret_cast<double*>(c.at(p.off_heap_f));
  c.hi = reinterpret_cast<int32_t*>(c.at(p.off_heap_i));
  c.ctrl = p.off_ctrl;
  c.pw = p.n == 1;  // numpy row-sum order, see ref_row_sum

  const int K = p.K, m = p.m, F = p.F, k = p.k;
  const double* glut = p.lut64 + (size_t)q * K * m;

  // 1. float64 LUT -> smem; float32 lane-private replicated pages for the fast books
  for (int i = tid; i < K * m; i += kThreads) c.lut[i] = glut[i];
  bool bad = false;
  for (int i = tid; i < FP * m * G::R; i += kThreads) {
    const int s = i / (m * G::R);
    const int rem = i - s * (m * G::R);
    const int j = rem / G::R;
    const int r = rem - j * G::R;
    float v = 0.f;
    if (s < F) {
      const double x = glut[p.fast_books[s] * m + j];
      // float32 certification needs finite entries with headroom; otherwise
      // the query runs in float64 only ("wide" mode)
      bad |= !(x <= 1.2676506002282294e30);  // 2^100 (also catches NaN)
      v = __double2float_rn(x);
    }
    sts_f32(kPage * (1 + s / G::BPR) + j * 256 + (s % G::BPR) * 4 * G::R + r * 4, v);
  }
  if (tid == 0) {
    for (int s = 0; s < p.nb; ++s) {
      mbar_init(c.ctrl + 8 * s, kNS * 32);   // full: every scan thread arrives
      mbar_init(c.ctrl + 64 + 8 * s, 32);    // empty: every replay lane arrives
    }
  }
  c.wide = __syncthreads_or(bad) != 0;

  // 2. seeds: ids 0..k-1 scored exactly (search.py:141), sorted descending
  //    by (exact, id) -> the sorted array is a valid max-heap.
  constexpr int kSeedPer = 8;
  double se[kSeedPer], sf[kSeedPer];
  int32_t sr[kSeedPer];
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kThreads;
    if (i < k) {
      const Row row = load_row(p.codes_full, p.KP, i);
      se[r] = exact64(c.lut, m, K, c.pw, row);
      sf[r] = fast64(c.lut, m, F, c.pw, p.fast_books, row);
      c.he[i] = se[r];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kThreads;
    if (i < k) {
      int rank = 0;
      for (int j = 0; j < k; ++j) rank += key_gt(c.he[j], j, se[r], i) ? 1 : 0;
      sr[r] = rank;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kThreads;
    if (i < k) {
      c.he[sr[r]] = se[r];
      c.hf[sr[r]] = sf[r];
      c.hi[sr[r]] = i;
    }
  }
  __syncthreads();

  Live L;
  L.refinements = L.insertions = L.candidates = L.certified = L.wait_cycles = 0;
  L.t_score = L.t_decide = L.t_insert = L.fallback_segments = 0;
  L.t_active = L.t_fallback = L.n_rounds = 0;
  L.H.k = k;
  L.H.reg = k <= 32 * kRegHeapRegs;
  L.H.he = c.he;
  L.H.hf = c.hf;
  L.H.hi = c.hi;
  if (warp == 0) {
    L.H.load(lane);
    live_update(L, F, p.sigma, c.wide);
    publish_prefetch(L, c, F, p.sigma, c.wide, lane);
    const double hmax = L.H.max_fast_all(lane);
    if (lane == 0) *reinterpret_cast<volatile double*>(c.at(c.ctrl + 136)) = hmax;
  }
  __syncthreads();
  const long long t_setup = clock64();

  // 3. phase 1: dense prologue over the insertion-heavy start
  const int64_t start = dense_prologue<FP>(c, L, tid, warp, lane);
  const int64_t seg0 = (start + G::S - 1) / G::S;  // start is a segment boundary or n
  const long long t_pro = clock64();

  // 4. phase 2: pipelined scan / replay
  if (warp == 0) {
    replay_role<FP>(c, L, lane, seg0);
  } else {
    scan_role<FP>(c, warp - 1, lane, seg0);
  }
  const long long t_scan = clock64();
  if (warp == 0) L.H.store(lane);
  __syncthreads();

  // 5. output: heap ascending by (score, id) (search.py:156-165)
  for (int i = tid; i < k; i += kThreads) {
    const int src = k - 1 - i;
    p.ids[(size_t)q * k + i] = c.hi[src];
    p.scores[(size_t)q * k + i] = c.he[src];
  }
  if (warp == 0 && lane == 0) {
    if (p.refinements) p.refinements[q] = p.exact_mode ? p.n : L.refinements;
    if (p.stats) {
      int64_t* st = p.stats + (size_t)q * kStats;
      st[0] = L.insertions;
      st[1] = L.candidates;
      st[2] = L.certified;
      st[3] = start;
      st[4] = t_pro - t_setup;       // prologue cycles
      st[5] = t_scan - t_pro;        // phase-2 cycles (replay warp)
      st[6] = L.wait_cycles;         // replay cycles waiting for scan warps
      st[7] = c.wide ? 1 : 0;
      st[8] = L.t_score;
      st[9] = L.t_decide;
      st[10] = L.t_insert;
      st[11] = L.fallback_segments;
      st[12] = p.nseg - seg0;        // phase-2 segments
      st[13] = L.t_active;           // replay cycles in segments with candidates
      st[14] = L.t_fallback;         // ... of which in the exact fallback
      st[15] = L.n_rounds;           // prologue decision rounds
    }
  }
}

// --------------------------------------------------------------------------
// host side: layout planning + launch
// --------------------------------------------------------------------------
template <int FP>
static bool plan_layout(ScanParams& p) {
  using G = Geo<FP>;
  const int K = p.K, m = p.m, k = p.k;
  // regions: A = [kDynBase, 64K), pages, B = [end of used pages, window end)
  const uint32_t pages_end = kPage * G::P + (uint32_t)m * 256;
  struct Region {
    uint32_t cur, end;
  } A{kDynBase, kPage}, B{(pages_end + 15u) & ~15u, kSmemWindow};
  auto place = [&](uint32_t bytes, uint32_t* off) {
    bytes = (bytes + 15u) & ~15u;
    if (A.cur + bytes <= A.end) { *off = A.cur; A.cur += bytes; return true; }
    if (B.cur + bytes <= B.end) { *off = B.cur; B.cur += bytes; return true; }
    return false;
  };
  if (!place((uint32_t)K * m * 8, &p.off_lut64)) return false;
  if (!place(kCtrlBytes, &p.off_ctrl)) return false;
  if (!place((uint32_t)k * 8, &p.off_heap_e)) return false;
  if (!place((uint32_t)k * 8, &p.off_heap_f)) return false;
  if (!place((uint32_t)k * 4, &p.off_heap_i)) return false;
  auto al16 = [](uint32_t x) { return (x + 15u) & ~15u; };
  // slot sub-layout for per-warp candidate lists of `cw` entries
  auto slot_layout = [&](int cw) {
    uint32_t o = kMetaBytes;
    p.so_lmin = o;   o = al16(o + kNS * 32 * 4);
    p.so_eid = o;    o = al16(o + kNS * cw * 4);
    p.so_ef32 = o;   o = al16(o + kNS * cw * 4);
    p.so_erow = o;   o = al16(o + kNS * cw * 16);
    return o;
  };
  // deepest ring first: the replay works off the scan by up to nb segments
  const int cw_pref[] = {32, 16};
  for (int nb = kMaxSlots; nb >= 2; --nb) {
    for (int cw : cw_pref) {
      Region a0 = A, b0 = B;
      const uint32_t sbytes = slot_layout(cw);
      // the ring is one contiguous block; the prologue buffer aliases it
      if (place(sbytes * nb, &p.off_slots)) {
        int C = 2048;
        while (C > 32 && (uint32_t)C * 16 > sbytes * nb) C >>= 1;
        if (C >= 256) {
          p.nb = nb;
          p.cw = cw;
          p.slot_bytes = sbytes;
          p.dense_chunk = C;
          const uint32_t end = B.cur > pages_end ? B.cur : pages_end;
          p.smem_end = end;
          p.dyn_bytes = end - kDynBase;
          return true;
        }
      }
      A = a0;
      B = b0;
    }
  }
  return false;
}

template <int FP>
static cudaError_t launch_fp(ScanParams& p, int Q, cudaStream_t s, int* unsupported) {
  using G = Geo<FP>;
  p.nseg = (p.n + G::S - 1) / G::S;
  if (!plan_layout<FP>(p)) {
    *unsupported = 1;
    return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(icq_scan_kernel<FP>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(kSmemWindow - kDynBase));
  if (e != cudaSuccess) return e;
  icq_scan_kernel<FP><<<Q, kThreads, p.dyn_bytes, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_scan(ScanParams& p, int FP, int Q, cudaStream_t s, int* unsupported) {
  *unsupported = 0;
  if (p.k > kThreads * 8) {
    *unsupported = 1;
    return cudaSuccess;
  }
  switch (FP) {
    case 1: return launch_fp<1>(p, Q, s, unsupported);
    case 2: return launch_fp<2>(p, Q, s, unsupported);
    case 4: return launch_fp<4>(p, Q, s, unsupported);
    case 8: return launch_fp<8>(p, Q, s, unsupported);
    case 16: return launch_fp<16>(p, Q, s, unsupported);
    default: *unsupported = 1; return cudaSuccess;
  }
}

}  // namespace icq

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
// CTA layout (288 threads, one CTA per SM, persistent over the database):
//   warps 1..8  SCAN   stream the fast-code column block (16-byte loads,
//                      register double-prefetch), gather |F| float32 entries
//                      per item from lane-private replicated LUT pages
//                      (conflict-free: entry j of book s for lane l sits in
//                      bank l; its address is ONE byte_perm of the code word),
//                      and publish per-item fast scores + per-group minima
//                      into a ring of segment slots.
//   warp 0      REPLAY consumes slots strictly in database order against the
//                      LIVE bound: groups whose minimum clears the bound are
//                      expanded, candidates are decided with certified float32
//                      thresholds (float64 recomputation only for near-ties),
//                      refined items are scored exactly in float64 from the
//                      shared float64 LUT, and insertions update a sorted heap
//                      in shared memory.  The result is bitwise the reference's.
// Slots are handed over with mbarriers (full: 256 scan-thread arrivals;
// empty: 32 replay-lane arrivals).
#include "icq_types.cuh"

namespace icq {



template <int FP>
struct Geo {
  static constexpr int R = FP <= 4 ? 32 : (FP == 8 ? 16 : 8);  // replicas per entry
  static constexpr int BPR = 64 / R;                             // book slots per 256-B row
  static constexpr int P = (FP + BPR - 1) / BPR;                 // 64 KiB pages
  static constexpr int IPC = 16 / FP;                            // items per 16-B chunk
  static constexpr int S = kNC * IPC;                            // items per segment
  static constexpr uint32_t slot_bytes = (IPC * kValStride + kNC) * 4;
};

// --------------------------------------------------------------------------
// float64 scores in the reference's order (search.py:94 -> numpy pairwise)
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
  return e1 > e2 || (e1 == e2 && i1 > i2);
}

// Replace the maximum (entry 0) of a descending-sorted heap by (e, id, f).
__device__ void heap_replace_max(double* he, double* hf, int32_t* hi, int k, double e, int32_t id,
                                 double f, int lane) {
  int g = 0;
  for (int base = 1; base < k; base += 32) {
    const int i = base + lane;
    const bool gt = i < k && key_gt(he[i], hi[i], e, id);
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

// --------------------------------------------------------------------------
// SCAN warps
// --------------------------------------------------------------------------
template <int FP>
__device__ __forceinline__ void scan_role(const ScanParams& p, int w, int lane, uint32_t ctrl) {
  using G = Geo<FP>;
  constexpr int IPC = G::IPC;
  constexpr int S = G::S;
  uint32_t L[FP];
#pragma unroll
  for (int s = 0; s < FP; ++s)
    L[s] = ((uint32_t)(1 + s / G::BPR) << 16) |
           (uint32_t)((s % G::BPR) * 4 * G::R + (lane % G::R) * 4);

  const uint4* codes = reinterpret_cast<const uint4*>(p.codes_fast);
  const int c0 = w * 64 + lane;  // chunk (group) ids owned by this lane
  const int c1 = c0 + 32;
  const int64_t seg0 = p.k / S;
  const int64_t nseg = p.nseg;

  uint4 a0 = make_uint4(0, 0, 0, 0), a1 = a0, b0 = a0, b1 = a0;
  if (seg0 < nseg) {
    a0 = ldg_stream(codes + seg0 * kNC + c0);
    a1 = ldg_stream(codes + seg0 * kNC + c1);
  }
  if (seg0 + 1 < nseg) {
    b0 = ldg_stream(codes + (seg0 + 1) * kNC + c0);
    b1 = ldg_stream(codes + (seg0 + 1) * kNC + c1);
  }
  int iter = 0;
  for (int64_t t = seg0; t < nseg; ++t, ++iter) {
    const uint4 x0 = a0, x1 = a1;
    a0 = b0;
    a1 = b1;
    if (t + 2 < nseg) {
      b0 = ldg_stream(codes + (t + 2) * kNC + c0);
      b1 = ldg_stream(codes + (t + 2) * kNC + c1);
    }
    float f[2][IPC];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const uint4 x = v ? x1 : x0;
      const uint32_t wd[4] = {x.x, x.y, x.z, x.w};
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
    // items outside [k, n) never enter the prune loop (seeds / padding)
    const int64_t base = t * S;
    if (base < p.k || base + S > p.n) {
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int j = 0; j < IPC; ++j) {
          const int64_t id = base + (int64_t)(v ? c1 : c0) * IPC + j;
          if (id < p.k || id >= p.n) f[v][j] = __int_as_float(0x7f800000);
        }
    }
    const int slot = iter % p.nb;
    const uint32_t par = (uint32_t)(iter / p.nb) & 1u;
    mbar_wait(ctrl + 32 + 8 * slot, par ^ 1u);  // empty[slot]
    const uint32_t vb = p.off_slot[slot];
    const uint32_t gb = vb + IPC * kValStride * 4;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int c = v ? c1 : c0;
      float mn = f[v][0];
#pragma unroll
      for (int j = 0; j < IPC; ++j) {
        sts_f32(vb + (uint32_t)(j * kValStride + c) * 4, f[v][j]);
        mn = fminf(mn, f[v][j]);
      }
      sts_f32(gb + (uint32_t)c * 4, mn);
    }
    mbar_arrive(ctrl + 8 * slot);  // full[slot]
  }
}

// --------------------------------------------------------------------------
// REPLAY warp
// --------------------------------------------------------------------------
struct ReplayState {
  double T64, bound64, thr64;
  float lo, hi;
  int64_t refinements, insertions, candidates, certified;
};

template <int FP>
__device__ __forceinline__ void replay_role(const ScanParams& p, int lane, uint32_t ctrl,
                                            const double* lut, double* he, double* hf,
                                            int32_t* hi, bool wide, int64_t* counters) {
  using G = Geo<FP>;
  constexpr int IPC = G::IPC;
  constexpr int S = G::S;
  const int F = p.F;
  const int K = p.K;
  const int m = p.m;
  const int k = p.k;
  const int64_t n = p.n;
  const bool pw = n == 1;
  uint32_t* surv = p.survivors ? p.survivors + (int64_t)blockIdx.x * p.words : nullptr;

  double T64 = he[0], bound64 = hf[0];
  double thr64 = __dadd_rn(bound64, p.sigma);
  float lo, hi_f;
  certified_bounds(thr64, F, lo, hi_f);
  if (wide) { lo = -__int_as_float(0x7f800000); hi_f = __int_as_float(0x7f800000); }
  int64_t refinements = 0, insertions = 0, candidates = 0, certified = 0;

  const int64_t seg0 = p.k / S;
  int iter = 0;
  for (int64_t t = seg0; t < p.nseg; ++t, ++iter) {
    const int slot = iter % p.nb;
    const uint32_t par = (uint32_t)(iter / p.nb) & 1u;
    mbar_wait(ctrl + 8 * slot, par);  // full[slot]
    const uint32_t vb = p.off_slot[slot];
    const uint32_t gb = vb + IPC * kValStride * 4;
    const int64_t base = t * S;
    for (int r = 0; r < kNC / 32; ++r) {
      const int cg = r * 32 + lane;
      const float g = lds_f32(gb + (uint32_t)cg * 4);
      const int64_t gid0 = base + (int64_t)cg * IPC;
      const bool gvalid = gid0 + IPC > k && gid0 < n;
      uint32_t cm = __ballot_sync(0xffffffffu, gvalid && (wide || g < hi_f));
      while (cm) {
        const int cl = __ffs(cm) - 1;
        const int c = r * 32 + cl;
        // ---- expand group c: lane j <-> item base + c*IPC + j --------------
        const bool act = lane < IPC;
        const int64_t id = base + (int64_t)c * IPC + lane;
        const bool valid = act && id >= k && id < n;
        const float fv = act ? lds_f32(vb + (uint32_t)(lane * kValStride + c) * 4) : 0.f;
        uint32_t done = 0;
        for (;;) {
          const bool cand = valid && !((done >> lane) & 1u) && (wide || fv < hi_f);
          const uint32_t cmask = __ballot_sync(0xffffffffu, cand);
          if (!cmask) break;
          bool refined = false, have_row = false, have_f64 = false;
          double f64 = 0.0, e64 = 0.0;
          Row row;
          if (cand) {
            if (!wide && fv < lo) {
              refined = true;
            } else {
              row = load_row(p.codes_full, p.KP, id);
              have_row = true;
              f64 = fast64(lut, m, F, pw, p.fast_books, row);
              have_f64 = true;
              refined = f64 < thr64;
            }
          }
          const uint32_t cert = __ballot_sync(0xffffffffu, cand && have_f64);
          if (refined) {
            if (!have_row) row = load_row(p.codes_full, p.KP, id);
            have_row = true;
            e64 = exact64(lut, m, K, pw, row);
          }
          const bool ins = refined && (e64 < T64);
          const uint32_t rmask = __ballot_sync(0xffffffffu, refined);
          const uint32_t imask = __ballot_sync(0xffffffffu, ins);
          const int first = imask ? __ffs(imask) - 1 : 31;
          const uint32_t decided = imask ? (0xffffffffu >> (31 - first)) : 0xffffffffu;
          refinements += __popc(rmask & decided);
          candidates += __popc(cmask & decided);
          certified += __popc(cert & decided);
          if (surv && refined && ((decided >> lane) & 1u))
            atomicOr(surv + (id >> 5), 1u << (id & 31));
          done |= decided;
          if (!imask) break;
          // ---- insertion of lane `first` (search.py:152-154) --------------
          if (lane == first && !have_f64) f64 = fast64(lut, m, F, pw, p.fast_books, row);
          const double ne = __shfl_sync(0xffffffffu, e64, first);
          const double nf = __shfl_sync(0xffffffffu, f64, first);
          const int32_t nid = (int32_t)__shfl_sync(0xffffffffu, (int32_t)id, first);
          heap_replace_max(he, hf, hi, k, ne, nid, nf, lane);
          T64 = he[0];
          bound64 = hf[0];
          thr64 = __dadd_rn(bound64, p.sigma);
          if (!wide) certified_bounds(thr64, F, lo, hi_f);
          ++insertions;
        }
        // the bound may have moved: re-test the remaining groups of this round
        const uint32_t above = (cl == 31) ? 0u : (0xffffffffu << (cl + 1));
        cm = __ballot_sync(0xffffffffu, gvalid && (wide || g < hi_f)) & above;
      }
    }
    __syncwarp();
    mbar_arrive(ctrl + 32 + 8 * slot);  // empty[slot]
  }
  if (lane == 0) {
    counters[0] = refinements;
    counters[1] = insertions;
    counters[2] = candidates;
    counters[3] = certified;
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
  auto sptr = [&](uint32_t abs) { return dsm + (abs - dbase); };
  double* lut = reinterpret_cast<double*>(sptr(p.off_lut64));
  double* he = reinterpret_cast<double*>(sptr(p.off_heap_e));
  double* hf = reinterpret_cast<double*>(sptr(p.off_heap_f));
  int32_t* hi = reinterpret_cast<int32_t*>(sptr(p.off_heap_i));
  int64_t* counters = reinterpret_cast<int64_t*>(sptr(p.off_ctrl + 64));
  const uint32_t ctrl = p.off_ctrl;

  const int K = p.K, m = p.m, F = p.F, k = p.k;
  const bool pw = p.n == 1;  // numpy row-sum order, see ref_row_sum
  const double* glut = p.lut64 + (size_t)q * K * m;

  // 1. float64 LUT -> smem; float32 lane-private replicated pages for the fast books
  for (int i = tid; i < K * m; i += kThreads) lut[i] = glut[i];
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
      mbar_init(ctrl + 8 * s, kNS * 32);   // full: every scan thread arrives
      mbar_init(ctrl + 32 + 8 * s, 32);    // empty: every replay lane arrives
    }
  }
  const bool wide = __syncthreads_or(bad) != 0;

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
      se[r] = exact64(lut, m, K, pw, row);
      sf[r] = fast64(lut, m, F, pw, p.fast_books, row);
      he[i] = se[r];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kThreads;
    if (i < k) {
      int rank = 0;
      for (int j = 0; j < k; ++j) rank += key_gt(he[j], j, se[r], i) ? 1 : 0;
      sr[r] = rank;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSeedPer; ++r) {
    const int i = tid + r * kThreads;
    if (i < k) {
      he[sr[r]] = se[r];
      hf[sr[r]] = sf[r];
      hi[sr[r]] = i;
    }
  }
  __syncthreads();

  // 3. persistent scan / replay
  if (warp == 0) {
    replay_role<FP>(p, lane, ctrl, lut, he, hf, hi, wide, counters);
  } else {
    scan_role<FP>(p, warp - 1, lane, ctrl);
  }
  __syncthreads();

  // 4. output: heap ascending by (score, id) (search.py:156-165)
  for (int i = tid; i < k; i += kThreads) {
    const int src = k - 1 - i;
    p.ids[(size_t)q * k + i] = hi[src];
    p.scores[(size_t)q * k + i] = he[src];
  }
  if (tid == 0) {
    if (p.refinements) p.refinements[q] = counters[0];
    if (p.stats) {
      p.stats[(size_t)q * 4 + 0] = counters[1];
      p.stats[(size_t)q * 4 + 1] = counters[2];
      p.stats[(size_t)q * 4 + 2] = counters[3];
      p.stats[(size_t)q * 4 + 3] = wide ? 1 : 0;
    }
  }
}

// --------------------------------------------------------------------------
// host side: layout planning + launch
// --------------------------------------------------------------------------
struct ScanLayout {
  bool ok;
  uint32_t dyn_bytes;
  int nb;
};

template <int FP>
static ScanLayout plan_layout(ScanParams& p) {
  using G = Geo<FP>;
  ScanLayout L{false, 0, 0};
  const int K = p.K, m = p.m, k = p.k;
  // regions: A = [kDynBase, 64K), pages, B = [end of used pages, window end)
  const uint32_t pages_end = kPage * G::P + (uint32_t)m * 256;
  struct Region { uint32_t cur, end; } A{kDynBase, kPage}, B{(pages_end + 15u) & ~15u, kSmemWindow};
  auto place = [&](uint32_t bytes, uint32_t* off) {
    bytes = (bytes + 15u) & ~15u;
    if (A.cur + bytes <= A.end) { *off = A.cur; A.cur += bytes; return true; }
    if (B.cur + bytes <= B.end) { *off = B.cur; B.cur += bytes; return true; }
    return false;
  };
  if (!place((uint32_t)K * m * 8, &p.off_lut64)) return L;
  if (!place(128 + 64, &p.off_ctrl)) return L;
  if (!place((uint32_t)k * 8, &p.off_heap_e)) return L;
  if (!place((uint32_t)k * 8, &p.off_heap_f)) return L;
  if (!place((uint32_t)k * 4, &p.off_heap_i)) return L;
  int nb = 0;
  for (; nb < 3; ++nb)
    if (!place(G::slot_bytes, &p.off_slot[nb])) break;
  if (nb < 2) return L;
  p.nb = nb;
  const uint32_t end = B.cur > pages_end ? B.cur : pages_end;
  p.smem_end = end;
  L.ok = true;
  L.nb = nb;
  L.dyn_bytes = end - kDynBase;
  return L;
}

template <int FP>
static cudaError_t launch_fp(ScanParams& p, int Q, cudaStream_t s, int* unsupported) {
  using G = Geo<FP>;
  p.nseg = (p.n + G::S - 1) / G::S;
  const ScanLayout L = plan_layout<FP>(p);
  if (!L.ok) { *unsupported = 1; return cudaSuccess; }
  cudaError_t e = cudaFuncSetAttribute(icq_scan_kernel<FP>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(kSmemWindow - kDynBase));
  if (e != cudaSuccess) return e;
  icq_scan_kernel<FP><<<Q, kThreads, L.dyn_bytes, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_scan(ScanParams& p, int FP, int Q, cudaStream_t s, int* unsupported) {
  *unsupported = 0;
  if (p.k > kThreads * 8) { *unsupported = 1; return cudaSuccess; }
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

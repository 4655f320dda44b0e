// icq_lut.cu — K1: batched per-query lookup-table construction.
//
// Reference: build_lut, /root/reference/pkg/src/icq/search.py:61-69
//     lut[b, j] = sum_t (float64(c[b, j, t]) - q[t])**2     (numpy pairwise order)
//
// The table is built in float64 by direct difference, in numpy's exact
// summation order, so every entry is bitwise equal to the reference's.  The
// pairwise order is a fixed tree of leaves (<= 128 elements, 8 strided
// accumulators each) that the host precomputes as a postfix program.
//
// Tiling: one CTA computes an 8-query x 32-codeword tile (256 threads, one
// entry each); per leaf the query slab (fp64) and the codeword slab (fp32,
// padded stride -> conflict-free) are staged in shared memory.  The work is
// tiny next to the scan (K*m*d per query) and fp64-pipe bound.
#include "icq_types.cuh"

namespace icq {

constexpr int kLutTQ = 8;    // queries per CTA tile
constexpr int kLutTJ = 32;   // codewords per CTA tile
constexpr int kLeafMax = 128;
constexpr int kLutStack = 16;



__global__ void __launch_bounds__(kLutTQ * kLutTJ) lut_build_kernel(
    const float* __restrict__ books, const double* __restrict__ q, double* __restrict__ lut,
    int32_t KM, int32_t d, int32_t Q, const LutProg* __restrict__ prog, int32_t* __restrict__ err) {
  __shared__ double sq[kLutTQ][kLeafMax];
  __shared__ float sc[kLutTJ][kLeafMax + 1];

  const int tj = threadIdx.x % kLutTJ;
  const int tq = threadIdx.x / kLutTJ;
  const int j0 = blockIdx.x * kLutTJ;
  const int q0 = blockIdx.y * kLutTQ;
  const int jj = j0 + tj;
  const int qq = q0 + tq;

  double stack[kLutStack];
  int sp = 0;
  const int nops = prog->nops;
  for (int o = 0; o < nops; ++o) {
    const int start = prog->op[o];
    if (start < 0) {  // combine: pw(left) + pw(right)
      const double b = stack[--sp];
      const double a = stack[--sp];
      stack[sp++] = __dadd_rn(a, b);
      continue;
    }
    const int L = prog->len[o];
    __syncthreads();
    bool bad = false;
    for (int i = threadIdx.x; i < kLutTQ * L; i += blockDim.x) {
      const int r = i / L, t = i % L;
      const double v = (q0 + r < Q) ? q[(size_t)(q0 + r) * d + start + t] : 0.0;
      bad |= !isfinite(v);
      sq[r][t] = v;
    }
    // search.py:51-52: a non-finite query is a ValidationError (the first
    // codeword tile reports it; the host turns it into ICQ_ERR_VALIDATION)
    if (bad && blockIdx.x == 0 && err) atomicOr(err, 8);
    for (int i = threadIdx.x; i < kLutTJ * L; i += blockDim.x) {
      const int r = i / L, t = i % L;
      sc[r][t] = (j0 + r < KM) ? books[(size_t)(j0 + r) * d + start + t] : 0.f;
    }
    __syncthreads();
    const double* qs = sq[tq];
    const float* cs = sc[tj];
    auto term = [&](int t) {
      const double df = __dsub_rn((double)cs[t], qs[t]);
      return __dmul_rn(df, df);
    };
    double res;
    if (L < 8) {
      res = 0.0;
      for (int t = 0; t < L; ++t) res = __dadd_rn(res, term(t));
    } else {
      double r0 = term(0), r1 = term(1), r2 = term(2), r3 = term(3);
      double r4 = term(4), r5 = term(5), r6 = term(6), r7 = term(7);
      int t = 8;
      const int top = L - (L % 8);
#pragma unroll 2
      for (; t < top; t += 8) {
        r0 = __dadd_rn(r0, term(t + 0));
        r1 = __dadd_rn(r1, term(t + 1));
        r2 = __dadd_rn(r2, term(t + 2));
        r3 = __dadd_rn(r3, term(t + 3));
        r4 = __dadd_rn(r4, term(t + 4));
        r5 = __dadd_rn(r5, term(t + 5));
        r6 = __dadd_rn(r6, term(t + 6));
        r7 = __dadd_rn(r7, term(t + 7));
      }
      res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                      __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
      for (; t < L; ++t) res = __dadd_rn(res, term(t));
    }
    stack[sp++] = res;
  }
  if (qq < Q && jj < KM) lut[(size_t)qq * KM + jj] = __dadd_rn(0.0, stack[0]);
}

// host-side program builder + launcher (called from icq_capi.cu)
static void build_prog_rec(LutProg& p, int lo, int n) {
  if (n <= kLeafMax) {
    p.op[p.nops] = lo;
    p.len[p.nops] = n;
    ++p.nops;
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  build_prog_rec(p, lo, n2);
  build_prog_rec(p, lo + n2, n - n2);
  p.op[p.nops] = -1;
  p.len[p.nops] = 0;
  ++p.nops;
}

bool make_lut_prog(int d, LutProg* out) {
  // leaves <= 128 -> ops < 2 * ceil(d / 64); 256 ops cover d <= 8192
  if (d < 1 || d > 8192) return false;
  out->nops = 0;
  build_prog_rec(*out, 0, d);
  return out->nops <= 256;
}

cudaError_t launch_lut(const float* books, const double* q, double* lut, int K, int m, int d,
                       int Q, const LutProg* prog_dev, int32_t* err, cudaStream_t s) {
  const int KM = K * m;
  dim3 grid((KM + kLutTJ - 1) / kLutTJ, (Q + kLutTQ - 1) / kLutTQ);
  lut_build_kernel<<<grid, kLutTQ * kLutTJ, 0, s>>>(books, q, lut, KM, d, Q, prog_dev, err);
  return cudaGetLastError();
}

}  // namespace icq

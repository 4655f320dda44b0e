// icq_pipeline.cu — dispatch of the prologue -> filter -> replay pipeline over
// the fast-row width FP (kernels in icq_pipeline.cuh, instantiated in
// icq_pipe_fp*.cu so the five variants compile in parallel).
#include <atomic>

#include "icq_common.cuh"

namespace icq {

std::atomic<long long> g_kernel_launches{0};
void count_kernel_launches(int n) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }
long long kernel_launches() { return g_kernel_launches.load(std::memory_order_relaxed); }

template <int FP>
cudaError_t launch_fp(const PipeParams& p, int filter_ctas, cudaStream_t s, cudaEvent_t* ev);
uint32_t pipeline_prologue_smem(int K, int m, int F, int k);
uint32_t pipeline_replay_smem(int K, int m, int F, int k);

cudaError_t launch_pipeline(const PipeParams& p, int FP, int filter_ctas, cudaStream_t s,
                            int* unsupported, cudaEvent_t* ev) {
  *unsupported = 0;
  if (p.k > kProThreads * 8 || pipeline_prologue_smem(p.K, p.m, p.F, p.k) > kSmemWindow - kDynBase ||
      pipeline_replay_smem(p.K, p.m, p.F, p.k) > kSmemWindow - kDynBase) {
    *unsupported = 1;
    return cudaSuccess;
  }
  switch (FP) {
    case 1: return launch_fp<1>(p, filter_ctas, s, ev);
    case 2: return launch_fp<2>(p, filter_ctas, s, ev);
    case 4: return launch_fp<4>(p, filter_ctas, s, ev);
    case 8: return launch_fp<8>(p, filter_ctas, s, ev);
    case 16: return launch_fp<16>(p, filter_ctas, s, ev);
    default: *unsupported = 1; return cudaSuccess;
  }
}

}  // namespace icq

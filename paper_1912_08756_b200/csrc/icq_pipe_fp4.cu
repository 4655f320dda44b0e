// icq_pipe_fp4.cu — pipeline kernels for fast rows of 4 byte(s) per item.
#include "icq_pipeline.cuh"

namespace icq {
template cudaError_t launch_fp<4>(const PipeParams&, int, cudaStream_t, cudaEvent_t*);

uint32_t pipeline_prologue_smem(int K, int m, int F, int k) { return pro_layout(K, m, F, k).total; }
uint32_t pipeline_replay_smem(int K, int m, int F, int k) { return rep_layout(K, m, F, k).total; }
}  // namespace icq

// icq_pipe_fp16.cu — pipeline kernels for fast rows of 16 byte(s) per item.
#include "icq_pipeline.cuh"

namespace icq {
template cudaError_t launch_fp<16>(const PipeParams&, int, cudaStream_t, cudaEvent_t*);
}  // namespace icq

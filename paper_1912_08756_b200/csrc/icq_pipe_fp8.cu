// icq_pipe_fp8.cu — pipeline kernels for fast rows of 8 byte(s) per item.
#include "icq_pipeline.cuh"

namespace icq {
template cudaError_t launch_fp<8>(const PipeParams&, int, cudaStream_t, cudaEvent_t*);
}  // namespace icq

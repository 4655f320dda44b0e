// icq_pipe_fp1.cu — pipeline kernels for fast rows of 1 byte(s) per item.
#include "icq_pipeline.cuh"

namespace icq {
template cudaError_t launch_fp<1>(const PipeParams&, int, cudaStream_t, cudaEvent_t*);
}  // namespace icq

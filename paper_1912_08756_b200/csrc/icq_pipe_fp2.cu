// icq_pipe_fp2.cu — pipeline kernels for fast rows of 2 byte(s) per item.
#include "icq_pipeline.cuh"

namespace icq {
template cudaError_t launch_fp<2>(const PipeParams&, int, cudaStream_t, cudaEvent_t*);
}  // namespace icq

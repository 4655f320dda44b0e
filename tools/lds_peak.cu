// tools/lds_peak.cu -- microbenchmark: shared-memory gather throughput per SM (conflict-free
// lane-private LDS.32, as the filter / count kernels issue it; LDS.64; random banks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lds_peak tools/lds_peak.cu && /tmp/lds_peak
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float lds_f32(uint32_t a) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v; }
__device__ __forceinline__ float2 lds_f32x2(uint32_t a) { float2 v; asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a)); return v; }
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(const uint32_t* codes, float* out, int iters) {
  extern __shared__ __align__(16) uint8_t dsm[];
  float* f = reinterpret_cast<float*>(dsm);
  for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) f[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(dsm);
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) w[i] = codes[(blockIdx.x * blockDim.x + threadIdx.x) * 8 + i];
  float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  const uint32_t lp = base + lane * 4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t x = w[i] + it;
      if (MODE == 0) {  // 4 x LDS.32, lane-private (address = code*128 + lane*4): conflict-free
        acc0 += lds_f32(lp + ((x & 0xffu) << 7));
        acc1 += lds_f32(lp + (((x >> 8) & 0xffu) << 7));
        acc2 += lds_f32(lp + (((x >> 16) & 0xffu) << 7));
        acc3 += lds_f32(lp + (((x >> 24) & 0xffu) << 7));
      } else if (MODE == 1) {  // 4 x LDS.64, lane-private 8-byte slots (code*256 + lane*8)
        const uint32_t lp2 = base + lane * 8;
        float2 a = lds_f32x2(lp2 + ((x & 0xffu) << 8));
        float2 b = lds_f32x2(lp2 + (((x >> 8) & 0xffu) << 8));
        float2 c = lds_f32x2(lp2 + (((x >> 16) & 0x7fu) << 8));
        float2 d = lds_f32x2(lp2 + (((x >> 24) & 0x7fu) << 8));
        acc0 += a.x + a.y; acc1 += b.x + b.y; acc2 += c.x + c.y; acc3 += d.x + d.y;
      } else {  // random banks (conflicts), shared 1 KiB table
        acc0 += lds_f32(base + ((x & 0xffu) << 2));
        acc1 += lds_f32(base + (((x >> 8) & 0xffu) << 2));
        acc2 += lds_f32(base + (((x >> 16) & 0xffu) << 2));
        acc3 += lds_f32(base + (((x >> 24) & 0xffu) << 2));
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
template <int MODE> void run(const char* name, int threads, const uint32_t* codes, float* out) {
  const int iters = 2000; int sms = 148;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE><<<sms, threads, 200 * 1024>>>(codes, out, 10);
  cudaEventRecord(a);
  k<MODE><<<sms, threads, 200 * 1024>>>(codes, out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double lds = (double)threads / 32 * iters * 32;  // warp-level LDS per SM
  printf("%-28s threads %4d: %.3f ms  %.3f LDS warp-instr / clk / SM (1.965 GHz)\n", name, threads, ms, lds / (ms * 1e-3 * 1.965e9));
}
int main() {
  uint32_t* codes; float* out;
  cudaMalloc(&codes, 148 * 1024 * 8 * 4); cudaMalloc(&out, 148 * 1024 * 4);
  uint32_t* h = new uint32_t[148 * 1024 * 8];
  uint32_t s = 12345; for (int i = 0; i < 148 * 1024 * 8; ++i) { s = s * 1664525u + 1013904223u; h[i] = s; }
  cudaMemcpy(codes, h, 148 * 1024 * 8 * 4, cudaMemcpyHostToDevice);
  for (int t : {128, 256, 512, 1024}) { run<0>("LDS.32 lane-private", t, codes, out); }
  for (int t : {128, 256, 512}) { run<1>("LDS.64 lane-private", t, codes, out); }
  for (int t : {512}) { run<2>("LDS.32 random banks", t, codes, out); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

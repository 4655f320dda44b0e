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
// MODE 3: the filter's tile loop: 4 coalesced 16-byte loads of an L2-resident
// code stream (register double buffer) feeding 64 lane-private LDS.32 per tile
__global__ void __launch_bounds__(512, 1) k_tile(const uint4* codes, float* out, int tiles, int ntile_buf) {
  extern __shared__ __align__(16) uint8_t dsm[];
  float* f = reinterpret_cast<float*>(dsm);
  for (int i = threadIdx.x; i < 48 * 1024; i += blockDim.x) f[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lp = (uint32_t)__cvta_generic_to_shared(dsm) + lane * 4;
  const uint4* cp = codes + (size_t)((blockIdx.x * 16 + warp) % 64) * 128 + lane;
  uint4 a[4];
  for (int v = 0; v < 4; ++v) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a[v].x), "=r"(a[v].y), "=r"(a[v].z), "=r"(a[v].w) : "l"(cp + v * 32));
  float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int t = 0; t < tiles; ++t) {
    uint4 x[4];
    for (int v = 0; v < 4; ++v) x[v] = a[v];
    const uint4* np = codes + (size_t)(((blockIdx.x * 16 + warp) * 7 + t + 1) % ntile_buf) * 128 + lane;
    for (int v = 0; v < 4; ++v) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a[v].x), "=r"(a[v].y), "=r"(a[v].z), "=r"(a[v].w) : "l"(np + v * 32));
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint32_t w[4] = {x[v].x, x[v].y, x[v].z, x[v].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc0 += lds_f32(lp + ((w[i] & 0xffu) << 7));
        acc1 += lds_f32(lp + (((w[i] >> 8) & 0xffu) << 7));
        acc2 += lds_f32(lp + (((w[i] >> 16) & 0xffu) << 7));
        acc3 += lds_f32(lp + (((w[i] >> 24) & 0xffu) << 7));
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
void run_tile(const uint4* codes, float* out, int ntile_buf) {
  const int tiles = 2000;
  cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_tile<<<148, 512, 200 * 1024>>>(codes, out, 10, ntile_buf);
  cudaEventRecord(a);
  k_tile<<<148, 512, 200 * 1024>>>(codes, out, tiles, ntile_buf);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double lds = 16.0 * tiles * 64;
  printf("%-28s threads  512: %.3f ms  %.3f LDS warp-instr / clk / SM, %.1f clk per tile-warp (64 LDS + 4 LDG.128, %d KiB stream)\n",
         "tile loop LDG.128 + LDS.32", ms, lds / (ms * 1e-3 * 1.965e9), ms * 1e-3 * 1.965e9 / (16.0 * tiles), ntile_buf * 2);
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
  {
    uint4* cb; cudaMalloc(&cb, (size_t)65536 * 2048);
    cudaMemcpy(cb, codes, 148 * 1024 * 8 * 4, cudaMemcpyDeviceToDevice);
    for (size_t o = 148 * 1024 * 8 * 4; o + 148 * 1024 * 8 * 4 <= (size_t)65536 * 2048; o += 148 * 1024 * 8 * 4)
      cudaMemcpy((char*)cb + o, codes, 148 * 1024 * 8 * 4, cudaMemcpyDeviceToDevice);
    run_tile(cb, out, 1024);    // 2 MiB stream: L2-resident
    run_tile(cb, out, 65536);   // 128 MiB stream
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

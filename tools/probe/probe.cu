// Box probe: FP32 FMA peak, pinned H2D/D2H bandwidth, device properties.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template <int CH>
__global__ void fma_peak(float* out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"name\":\"%s\",\"sms\":%d,\"smem_per_block_optin\":%zu,\"smem_per_sm\":%zu,\"l2\":%d,\"regs_per_sm\":%d,\"cc\":\"%d.%d\",\"clock_khz\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.l2CacheSize,
         p.regsPerMultiprocessor, p.major, p.minor, 0);
  float* d; CK(cudaMalloc(&d, 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 1 << 16, threads = 512, blocks = p.multiProcessorCount * 4;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    fma_peak<16><<<blocks, threads>>>(d, iters, 0.9999f, 1e-4f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * (double)iters * threads * blocks;
    printf("{\"fp32_fma_tflops\":%.2f,\"ms\":%.3f}\n", fl / ms / 1e9, ms);
  }
  // pinned H2D / D2H
  size_t bytes = 1ull << 30;
  void *h, *dv; CK(cudaMallocHost(&h, bytes)); CK(cudaMalloc(&dv, bytes));
  memset(h, 1, bytes);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); cudaMemcpyAsync(dv, h, bytes, cudaMemcpyHostToDevice); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"h2d_gbs\":%.1f}\n", bytes / ms / 1e6);
    cudaEventRecord(e0); cudaMemcpyAsync(h, dv, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"d2h_gbs\":%.1f}\n", bytes / ms / 1e6);
  }
  return 0;
}

// Throughput of legacy warp-level mma.sync TF32 (m16n8k8) on this GPU, vs the
// FP32 FMA pipe: is a 3xTF32 warp-MMA path for K1's contractions worth it?
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void mma_tf32(float* out, int iters, long long* cyc) {
  float acc[NACC][4];
  for (int i = 0; i < NACC; ++i)
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = __float_as_uint(0.5f), b1 = b0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < NACC; ++i)
    for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ffma_ref(float* out, int iters, long long* cyc) {
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 0.001f + i;
  const float a = 1.0001f, b = 0.9999f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], a, b);
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  auto avg = [&]() {
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    return m / 148;
  };
  for (int warps : {4, 8, 16}) {
    const int iters = 4000;
    mma_tf32<8><<<148, 32 * warps>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    double c = avg();
    double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * warps;  // per SM
    printf("mma.sync tf32 m16n8k8: %2d warps/SM: %.1f flop/clk/SM (%.2f x FP32 FMA peak 256)\n", warps, flops / c,
           flops / c / 256.0);
    ffma_ref<<<148, 32 * warps>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    c = avg();
    flops = 2.0 * 16 * 32.0 * iters * warps;
    printf("ffma reference       : %2d warps/SM: %.1f flop/clk/SM\n", warps, flops / c);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

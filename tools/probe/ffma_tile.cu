// Outer-product register-tile FFMA throughput (3 register sources), as in K1 phase B:
// acc[j][t] += w[j] * x[t] with w, x refreshed from shared memory each row.
#include <cstdio>
#include <cuda_runtime.h>
template <int TK, int TN, bool LOADS>
__global__ void __launch_bounds__(256, 1) tile(float* out, int iters) {
  __shared__ float sw[64][16], sx[64][8];
  for (int i = threadIdx.x; i < 64 * 16; i += 256) (&sw[0][0])[i] = 1e-3f * (i % 7);
  for (int i = threadIdx.x; i < 64 * 8; i += 256) (&sx[0][0])[i] = 1e-3f * (i % 5);
  __syncthreads();
  float acc[TK][TN];
  for (int j = 0; j < TK; ++j) for (int t = 0; t < TN; ++t) acc[j][t] = 0.f;
  float w[TK], x[TN];
  for (int j = 0; j < TK; ++j) w[j] = sw[0][j];
  for (int t = 0; t < TN; ++t) x[t] = sx[0][t];
  for (int it = 0; it < iters; ++it) {
    const int r = it & 63;
    if (LOADS) {
#pragma unroll
      for (int j = 0; j < TK; ++j) w[j] = sw[r][(j + threadIdx.x) & 15];
#pragma unroll
      for (int t = 0; t < TN; ++t) x[t] = sx[r][t];
    }
#pragma unroll
    for (int j = 0; j < TK; ++j)
#pragma unroll
      for (int t = 0; t < TN; ++t) acc[j][t] = fmaf(w[j], x[t], acc[j][t]);
  }
  float s = 0.f;
  for (int j = 0; j < TK; ++j) for (int t = 0; t < TN; ++t) s += acc[j][t];
  if (s == 1234.5f) out[0] = s;
}
template <int TK, int TN, bool L>
void run(const char* name, float* d, int blocks) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 1 << 14;
  tile<TK, TN, L><<<blocks, 256>>>(d, iters);
  cudaEventRecord(a);
  tile<TK, TN, L><<<blocks, 256>>>(d, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fl = 2.0 * TK * TN * double(iters) * 256 * blocks;
  printf("%-28s %7.2f TFLOP/s\n", name, fl / ms / 1e9);
}
int main() {
  float* d; cudaMalloc(&d, 4);
  run<13, 7, false>("13x7 regs only", d, 148);
  run<13, 7, true>("13x7 + smem loads", d, 148);
  run<8, 8, false>("8x8 regs only", d, 148);
  run<8, 8, true>("8x8 + smem loads", d, 148);
  run<13, 7, false>("13x7 regs only 2 CTA/SM", d, 296);
  return 0;
}

// mma.sync m16n8k8 tf32 throughput when each MMA's B operand is split on the fly
// (LOP3 + FADD per value, as in K1M) and/or loaded from shared memory.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int NACC>
__global__ void mma_mix(float* out, int iters, long long* cyc) {
  __shared__ float sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1.0f + i * 1e-3f;
  float acc[NACC][4];
  for (int i = 0; i < NACC; ++i)
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  float x0 = 0.5f + threadIdx.x, x1 = 0.25f;
  const int lane = threadIdx.x & 31;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      unsigned b0, b1;
      if (MODE == 0) {  // constant B
        b0 = __float_as_uint(x0);
        b1 = __float_as_uint(x1);
      } else if (MODE == 1) {  // B split on the fly: lo = x - trunc(x)
        const float y0 = x0 + float(i), y1 = x1 + float(it);
        b0 = __float_as_uint(y0 - __uint_as_float(__float_as_uint(y0) & 0xffffe000u));
        b1 = __float_as_uint(y1 - __uint_as_float(__float_as_uint(y1) & 0xffffe000u));
      } else {  // B from shared memory (scalar LDS) + split
        const float y0 = sm[(lane + 37 * i + it) & 2047], y1 = sm[(lane + 37 * i + it + 64) & 2047];
        b0 = __float_as_uint(y0 - __uint_as_float(__float_as_uint(y0) & 0xffffe000u));
        b1 = __float_as_uint(y1 - __uint_as_float(__float_as_uint(y1) & 0xffffe000u));
      }
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(acc[i][0]), "+f"(acc[i][1]), "+f"(acc[i][2]), "+f"(acc[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < NACC; ++i)
    for (int j = 0; j < 4; ++j) s += acc[i][j];
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
#define RUN(M, N)                                                                              \
  for (int warps : {8, 12, 16}) {                                                              \
    const int iters = 1000;                                                                    \
    mma_mix<M, N><<<148, 32 * warps>>>(out, iters, cyc);                                       \
    cudaDeviceSynchronize();                                                                   \
    double c = avg();                                                                          \
    double mmas = double(N) * iters * warps;                                                   \
    printf("mode %d chains %2d warps/SM %2d: %.2f cycles per mma per SMSP\n", M, N, warps, c / (mmas / 4)); \
  }
  RUN(0, 8) RUN(1, 8) RUN(2, 8) RUN(1, 14) RUN(2, 14)
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

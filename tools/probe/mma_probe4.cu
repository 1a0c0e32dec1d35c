// Does shared-memory load traffic slow mma.sync down even when the MMAs do not
// depend on it?  HMMA stream (14 independent chains) + R independent LDS per MMA.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND, int R>  // KIND 0: LDS.32, 1: LDS.64, 2: LDS.128
__global__ void mma_lds(float* out, int iters, long long* cyc) {
  __shared__ __align__(16) float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0f + i * 1e-3f;
  constexpr int N = 14;
  float acc[N][4];
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  unsigned b0 = __float_as_uint(0.5f), b1 = b0 + 7;
  const int lane = threadIdx.x & 31;
  float sink = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 64) & 1023;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int off = base + 128 * ((i * R + r) & 7);
        if (KIND == 0) sink += sm[off + lane];
        if (KIND == 1) {
          const float2 v = *reinterpret_cast<const float2*>(sm + 2 * off + 2 * lane);
          sink += v.x + v.y;
        }
        if (KIND == 2) {
          const float4 v = *reinterpret_cast<const float4*>(sm + (4 * off & 4095) + 4 * lane);
          sink += v.x + v.w;
        }
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
  float s = sink;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < 4; ++j) s += acc[i][j];
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND, int R>
__global__ void lds_only(float* out, int iters, long long* cyc) {
  __shared__ __align__(16) float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0f + i * 1e-3f;
  const int lane = threadIdx.x & 31;
  float sink = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int base = (it * 64) & 1023;
#pragma unroll
    for (int i = 0; i < 14; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int off = base + 128 * ((i * R + r) & 7);
        if (KIND == 0) sink += sm[off + lane];
        if (KIND == 2) {
          const float4 v = *reinterpret_cast<const float4*>(sm + (4 * off & 4095) + 4 * lane);
          sink += v.x + v.w;
        }
      }
  }
  __syncthreads();
  long long t1 = clock64();
  if (sink == 1234.5f) out[0] = sink;
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
  const int iters = 500, warps = 12;
#define RUN(K, R)                                                                                       \
  {                                                                                                     \
    mma_lds<K, R><<<148, 32 * warps>>>(out, iters, cyc);                                                \
    cudaDeviceSynchronize();                                                                            \
    const double c = avg(), mmas = 14.0 * iters * warps / 4;                                            \
    printf("kind %d (%s) x%d per mma: %.2f cycles per mma per SMSP\n", K, K == 0 ? "LDS.32" : K == 1 ? "LDS.64" : "LDS.128", R, c / mmas); \
  }
  RUN(0, 0) RUN(0, 1) RUN(0, 2) RUN(0, 4) RUN(1, 1) RUN(1, 2) RUN(2, 1) RUN(2, 2)
#define RUNL(K, R)                                                                                      \
  {                                                                                                     \
    lds_only<K, R><<<148, 32 * warps>>>(out, iters, cyc);                                               \
    cudaDeviceSynchronize();                                                                            \
    const double c = avg(), n = 14.0 * R * iters * warps;                                               \
    printf("lds only kind %d: %.2f cycles per warp-LDS per SM\n", K, c / n);                            \
  }
  RUNL(0, 2) RUNL(2, 2)
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

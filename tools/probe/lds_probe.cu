// Shared-memory wavefront cost of LDS.128 address patterns on this GPU:
// cycles per warp-level LDS.128 per SM with 8 warps issuing back-to-back.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int pat(int p, int lane) {
  switch (p) {
    case 0: return 0;                                   // broadcast
    case 1: return lane >> 4;                           // 2 distinct (one per half)
    case 2: return lane >> 3;                           // 4 distinct (one per quarter)
    case 3: return lane & 7;                            // 8 consecutive, same in each quarter
    case 4: return (lane & 7) * 13;                     // 8 rows stride 13 float4, same per quarter
    case 5: return lane;                                // 32 consecutive
    case 6: return lane >> 1;                           // 16 distinct
    case 7: return lane >> 2;                           // 8 distinct, 4 lanes share
    case 8: return lane & 3;                            // 4 consecutive, same in every quarter
    case 9: return 9 * (lane >> 4) + 2 * ((lane >> 2) & 3);  // phase-B x loads
    case 10: return (lane & 7) * 13 + 0 * (lane >> 3);  // = 4
    case 11: return (lane >> 3) * 13;                   // 4 rows one per quarter, stride 13
    case 12: return (lane & 15);                        // 16 consecutive, same in each half
    case 13: return (lane & 15) * 13;                   // 16 rows stride 13, same per half
    case 14: return (lane >> 4) * 13;                   // 2 rows one per half
    case 15: return (lane & 1) + 2 * (lane >> 3);       // 8 distinct: 2 per quarter
    default: return 0;
  }
}

__global__ void lds_kernel(float* out, int p, int iters, long long* cyc) {
  __shared__ float4 s[2560];
  for (int i = threadIdx.x; i < 2560; i += blockDim.x) s[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned base = static_cast<unsigned>(__cvta_generic_to_shared(s)) + 16u * pat(p, lane);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      float x, y, z, w;
      asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(base + 16u * 256u * (u & 7)) : "memory");
      acc += (x + y) + (z + w);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int iters = 2000, warps = 8;
  for (int p = 0; p < 16; ++p) {
    lds_kernel<<<148, 32 * warps>>>(out, p, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148;
    printf("pattern %2d: %.2f cycles per warp LDS.128 (SM-wide)\n", p, m / (double(iters) * 16 * warps));
  }
  return 0;
}

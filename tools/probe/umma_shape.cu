// tcgen05.mma kind::tf32 (cta_group::1) issue throughput as a function of the
// MMA shape: M in {64, 128}, N in {8 .. 256}, K = 8 (one 32-byte K step), operands
// K-major without swizzle in shared memory, issued by one thread round-robin over
// NACC independent TMEM accumulators, completion by tcgen05.commit + mbarrier.
// Prints cycles per MMA and MAC/clk/SM — the evidence for which K1 shapes could
// use the 5th-generation tensor core (DESIGN.md §5 "tcgen05 for K <= 56").
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_shape umma_shape.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA %s: %s\n", #x, cudaGetErrorString(e));                  \
      return;                                                              \
    }                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
// shared memory matrix descriptor: start, leading / stride byte offsets, layout (0 = no swizzle)
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
// instruction descriptor: D f32, A/B tf32, K-major both, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

template <int M, int N, int NACC>
__global__ void tput(int reps, long long* out) {
  extern __shared__ __align__(1024) float sm[];
  float* A = sm;          // M x 32 tf32 (4 K steps)
  float* B = A + M * 32;  // N x 32
  __shared__ uint32_t tm;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < (M + N) * 32; i += blockDim.x) sm[i] = 0.001f * (i % 97);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tm)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t d0 = tm;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t ad = desc(su(A) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128);
        const uint64_t bd = desc(su(B) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128);
#pragma unroll
        for (int c = 0; c < NACC; ++c)
          asm volatile(
              "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, "
              "q;\n\t}\n" ::"r"(d0 + uint32_t(c * N)),
              "l"(ad), "l"(bd), "r"(idesc(M, N)), "r"(1));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
          : "=r"(done)
          : "r"(su(&bar)));
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int M, int N, int NACC>
void run(int reps = 256) {
  long long* d;
  long long h = 0;
  CK(cudaMalloc(&d, 8));
  auto k = tput<M, N, NACC>;
  const int smem = (M + N) * 32 * 4;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k<<<1, 128, smem>>>(2, d);  // warm-up
  CK(cudaDeviceSynchronize());
  k<<<1, 128, smem>>>(reps, d);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  const double mmas = double(reps) * 4 * NACC;
  const double cyc = h / mmas;
  printf("M=%3d N=%3d K=8 acc=%d : %6.1f cycles/MMA  %6.0f MAC/clk/SM  (3xTF32: %5.0f useful MAC/clk)\n", M, N, NACC,
         cyc, double(M) * N * 8 / cyc, double(M) * N * 8 / cyc / 3.0);
  cudaFree(d);
}

int main() {
  printf("tcgen05.mma.cta_group::1.kind::tf32, one issuing thread, operands K-major / no swizzle in smem\n");
  run<128, 8, 4>();
  run<128, 16, 4>();
  run<128, 32, 4>();
  run<128, 32, 1>();
  run<128, 64, 4>();
  run<128, 64, 1>();
  run<128, 128, 4>();
  run<128, 128, 1>();
  run<128, 256, 2>();
  run<128, 256, 1>();
  run<64, 32, 4>();
  run<64, 64, 4>();
  run<64, 128, 4>();
  run<64, 256, 2>();
  printf("reference: mma.sync.m16n8k8 tf32 = 510 MAC/clk/SM (tools/probe/mma_probe2.cu), i.e. 170 useful 3xTF32\n");
  return 0;
}

// tcgen05 kind::tf32 issue-to-completion throughput for the K1R / K1T operand
// layouts: A MN-major (128B_BASE32B atoms) vs K-major (no swizzle), B K-major.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); return; } } while (0)
__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t(lay) << 61) | uint64_t((a >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(amn) << 15) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
template <int M, int N, int AMN>
__global__ void tput(int reps, long long* out) {
  extern __shared__ __align__(1024) float sm[];
  float* A = sm;            // M x 32 (K = 32 per group: 4 K steps)
  float* B = A + M * 32;    // N x 32
  __shared__ uint32_t tm;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < (M + N) * 32; i += blockDim.x) sm[i] = 0.001f * (i % 97);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tm)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t d = tm;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int s = 0; s < 4; ++s) {
        uint64_t ad;
        if (AMN) ad = desc(su(A) + uint32_t(2 * s * (M / 32) * 128) * 4u, 512, (M / 32) * 512, 1);
        else ad = desc(su(A) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128, 0);
        const uint64_t bd = desc(su(B) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128, 0);
        for (int p = 0; p < 3; ++p)
          asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n\t}\n"
                       ::"r"(d), "l"(ad), "l"(bd), "r"(idesc(M, N, AMN)), "r"(1));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}\n" : "=r"(done) : "r"(su(&bar)));
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}
template <int M, int N, int AMN>
void run(const char* name, int reps = 200) {
  long long* d; long long h = 0;
  CK(cudaMalloc(&d, 8));
  auto k = tput<M, N, AMN>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (M + N) * 32 * 4));
  k<<<1, 128, (M + N) * 32 * 4>>>(reps, d);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  const double mmas = reps * 12.0;
  printf("%-28s reps %3d: %7.1f cycles per MMA (K=8)   %7.0f fp32-equivalent MAC/clk (3xTF32)\n", name, reps, h / mmas,
         double(M) * N * 8 / 3.0 / (h / mmas));
  cudaFree(d);
}
int main() {
  run<64, 56, 1>("M64 N56  A MN-major SW32B");
  run<64, 56, 0>("M64 N56  A K-major");
  run<128, 112, 1>("M128 N112 A MN-major SW32B");
  run<128, 112, 0>("M128 N112 A K-major");
  run<128, 128, 0>("M128 N128 A K-major");
  run<64, 128, 0>("M64 N128 A K-major");
  // latency of one window's worth (12 MMAs + commit + mbarrier wait), cold and warm
  for (int r : {1, 1, 2, 4}) run<64, 56, 1>("M64 N56 one window", r);
  for (int r : {1, 1, 2}) run<128, 112, 1>("M128 N112 half window", r);
  return 0;
}

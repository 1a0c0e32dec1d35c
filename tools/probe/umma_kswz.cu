// Is a K-major tf32 operand legal in the 128B_BASE32B swizzle (descriptor layout 1), and
// with which byte pattern?  D[128][N] = A[128][32] * B[N][32]^T, A K-major no swizzle,
// B K-major in candidate layouts (128-byte rows along K, 8-row groups 1024 B apart):
//   cand 0: 32-byte chunk ^= row % 4          (the MN-major 128B_BASE32B atom's bytes)
//   cand 1: 32-byte chunk ^= (row / 2) % 4
//   cand 2: 16-byte chunk ^= row % 8, layout 2 (plain SWIZZLE_128B, control)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_kswz umma_kswz.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t(layout) << 61) | uint64_t((a >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ int boff(int cand, int n, int k) {  // float offset of B[n][k], K = 32
  const int row = n & 7, grp = n >> 3;
  int byte = (k & 31) * 4;
  if (cand == 0) byte = ((((k >> 3) & 3) ^ (row & 3)) << 5) | ((k & 7) << 2);
  if (cand == 1) byte = ((((k >> 3) & 3) ^ ((row >> 1) & 3)) << 5) | ((k & 7) << 2);
  if (cand == 2) byte = ((((k >> 2) & 7) ^ row) << 4) | ((k & 3) << 2);
  return (grp * 1024 + row * 128 + byte) / 4;
}
__device__ int aoff(int m, int k) { return ((m >> 3) * 8 + (k >> 2)) * 32 + (m & 7) * 4 + (k & 3); }

template <int N>
__global__ void test(const float* A, const float* B, float* D, int cand, int sbo, int ksteps) {
  extern __shared__ __align__(1024) float smraw[];
  const uint32_t base = su(smraw);
  float* sm = smraw + ((((base + 1023u) & ~1023u) - base) >> 2);
  float* As = sm;            // 128 x 32 (hi only: inputs are tf32-exact)
  float* Bs = sm + 128 * 32;  // N x 32
  __shared__ uint32_t tm;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 32; i += 128) As[aoff(i / 32, i % 32)] = A[i];
  for (int i = tid; i < N * 32; i += 128) Bs[boff(cand, i / 32, i % 32)] = B[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tm)), "r"(256));
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
    const uint32_t layout = cand == 2 ? 2u : 1u;
    for (int s = 0; s < ksteps; ++s) {
      const uint64_t ad = desc(su(As + 2 * s * 32), 128, 8 * 128, 0);
      const uint64_t bd = desc(su(Bs) + 32 * s, 16, sbo, layout);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(idesc(128, N)), "r"(s > 0 ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
                   : "=r"(done) : "r"(su(&bar)));
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + (uint32_t(32 * warp) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main(int argc, char** argv) {
  const int only_cand = argc > 1 ? atoi(argv[1]) : -1, only_sbo = argc > 2 ? atoi(argv[2]) : -1;
  const int ksteps = argc > 3 ? atoi(argv[3]) : 4;
  constexpr int N = 64;
  std::vector<float> A(128 * 32), B(N * 32), D(128 * N);
  for (int i = 0; i < 128 * 32; ++i) A[i] = float(1 + (i * 37) % 13) / 8.0f;  // tf32-exact
  for (int i = 0; i < N * 32; ++i) B[i] = float(1 + (i * 11) % 17) / 16.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (128 + N) * 32 * 4 + 2048;
  cudaFuncSetAttribute(test<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int cand = 0; cand < 3; ++cand)
    for (int sbo : {512, 1024}) {
      if ((only_cand >= 0 && cand != only_cand) || (only_sbo >= 0 && sbo != only_sbo)) continue;
      cudaMemset(dD, 0, D.size() * 4);
      test<N><<<1, 128, smem>>>(dA, dB, dD, cand, sbo, ksteps);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double worst = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          double s = 0;
          for (int k = 0; k < 8 * ksteps; ++k) s += double(A[m * 32 + k]) * B[n * 32 + k];
          worst = std::fmax(worst, std::fabs(D[m * N + n] - s) / s);
        }
      printf("cand %d sbo %4d: %s max rel err %.3e\n", cand, sbo, cudaGetErrorString(e), worst);
      if (e != cudaSuccess) return 1;
    }
  return 0;
}

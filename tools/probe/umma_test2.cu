// tcgen05 probe 2: (a) MN-major tf32 with SWIZZLE_128B 16-byte atoms (shared with a
// K-major SWIZZLE_128B layout of the same bytes), (b) raw fp32 as the "hi" operand
// (does the tensor core truncate?), (c) MMA issue throughput for M128N32K8 / M64N64K8.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t(layout) << 61) | uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(dt), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// SWIZZLE_128B rows of 32 elements (128 B); atoms of 8 rows (1 KB); 16-B chunk index ^= row % 8.
// "row" = index along the 128-B-row dimension (rows of the K-major operand / K-rows of the MN-major one),
// "col" = index within the 32-element row. atoms laid [colatom][rowatom].
__device__ __forceinline__ int off_sw128(int row, int col, int rows) {
  const int r8 = row & 7, c = col & 31;
  return ((col >> 5) * (rows >> 3) + (row >> 3)) * 256 + r8 * 32 + (((c >> 2) ^ r8) << 2) + (c & 3);
}
__device__ __forceinline__ uint32_t wait_bar(uint64_t* mbar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
                 : "=r"(done) : "r"(smem_u32(mbar)), "r"(phase));
  return done;
}

// D[M][N] = A[M][K] B[N][K]^T. mode 0: A K-major SW128 (rows = m, cols = k), B K-major SW128.
// mode 1: A MN-major SW128 (rows = k, cols = m), B K-major SW128. raw_hi: use fp32 unmodified as hi.
template <int M, int N, int K>
__global__ void sw128_test(const float* A, const float* B, float* D, int mode, int raw_hi, int reps, long long* cycles) {
  extern __shared__ __align__(1024) float sm[];
  float* Ahi = sm; float* Alo = Ahi + M * K; float* Bhi = Alo + M * K; float* Blo = Bhi + N * K;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const float x = A[i], h = raw_hi ? x : tf32_hi(x);
    const int o = mode == 0 ? off_sw128(m, k, M) : off_sw128(k, m, K);
    Ahi[o] = h; Alo[o] = x - tf32_hi(x);
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const float x = B[i], h = raw_hi ? x : tf32_hi(x);
    Bhi[off_sw128(n, k, N)] = h; Blo[off_sw128(n, k, N)] = x - tf32_hi(x);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  long long t0 = clock64();
  if (tid == 0) {
    const uint32_t idesc = make_idesc(M, N, mode, 0);
    for (int rep = 0; rep < reps; ++rep)
      for (int s = 0; s < K / 8; ++s) {
        // K-major SW128: K step s covers elements 8s..8s+7 = bytes 32s within the 128-B row (same atom column)
        // descriptor start advances by 32 B inside the swizzled row (CUTLASS advance_umma_desc_lo style)
        uint64_t ad[2], bd[2];
        const float* As[2] = {Ahi, Alo};
        const float* Bs[2] = {Bhi, Blo};
        for (int p = 0; p < 2; ++p) {
          if (mode == 0)
            ad[p] = make_desc(smem_u32(As[p] + ((8 * s) >> 5) * (M / 8) * 256 + ((8 * s) & 31)), 16, 1024, 2);
          else  // MN-major SW128: K step s = rows 8s..8s+7 = one row-atom; LBO = stride between 32-element col atoms
            ad[p] = make_desc(smem_u32(As[p] + s * 256), (K / 8) * 1024, 1024, 2);
          bd[p] = make_desc(smem_u32(Bs[p] + ((8 * s) >> 5) * (N / 8) * 256 + ((8 * s) & 31)), 16, 1024, 2);
        }
        const uint32_t acc = (rep > 0 || s > 0) ? 1u : 0u;
        mma_tf32(tbase, ad[0], bd[0], idesc, acc);
        mma_tf32(tbase, ad[0], bd[1], idesc, 1u);
        mma_tf32(tbase, ad[1], bd[0], idesc, 1u);
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  wait_bar(&mbar, 0);
  if (tid == 0) cycles[0] = clock64() - t0;
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tbase + (uint32_t(warp * 32) << 16) + uint32_t(c)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[(warp * 32 + (tid & 31)) * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128));
}

template <int M, int N, int K>
void run(const char* name, int mode, int raw_hi, int reps) {
  std::vector<float> A(M * K), B(N * K), D(128 * N);
  srand(3);
  for (auto& x : A) x = float(rand()) / RAND_MAX + 0.01f;
  for (auto& x : B) x = float(rand()) / RAND_MAX * 1e-2f + 1e-5f;
  float *dA, *dB, *dD; long long* dc;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4)); CK(cudaMalloc(&dc, 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  auto kern = sw128_test<M, N, K>;
  const size_t smem = size_t(2 * (M + N) * K) * 4;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<1, 128, smem>>>(dA, dB, dD, mode, raw_hi, reps, dc);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long long cyc; CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
  double worst = 0;
  const int rowsM = M;  // M=64 rows live in lanes 32q + (0..15)
  for (int m = 0; m < rowsM; ++m) for (int n = 0; n < N; ++n) {
    double s = 0; for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * double(B[n * K + k]);
    s *= reps;
    const int lane = M == 128 ? m : (m / 16) * 32 + (m % 16);
    worst = std::max(worst, std::fabs(D[lane * N + n] - s) / s);
  }
  const double macs = double(M) * N * K * 3 * reps;
  printf("%-40s err %.3e  %lld cycles  %.0f MAC/cycle\n", name, worst, cyc, macs / cyc);
}
int main() {
  run<128, 32, 64>("K-major SW128 M128N32K64", 0, 0, 1);
  run<128, 32, 64>("MN-major SW128 A, M128N32K64", 1, 0, 1);
  run<128, 32, 64>("K-major SW128, raw fp32 hi", 0, 1, 1);
  run<128, 32, 64>("throughput M128N32 (x200)", 0, 0, 200);
  run<64, 64, 64>("throughput M64N64 (x200)", 0, 0, 200);
  run<128, 64, 64>("throughput M128N64 (x200)", 0, 0, 200);
  run<128, 128, 64>("throughput M128N128 (x200)", 0, 0, 200);
  return 0;
}

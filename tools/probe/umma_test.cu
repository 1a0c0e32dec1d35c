// tcgen05 (UMMA) micro-test: D[M][N] = A[M][K] * B[N][K]^T in 3xTF32 with
// hand-built shared-memory descriptors (no swizzle), operands stored either
// K-major or MN-major, accumulator in TMEM read back with tcgen05.ld 32x32b.
// Prints the max relative error vs an fp64 host product and dumps where each
// D row landed in TMEM (lane) for M = 64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_test umma_test.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// no-swizzle UMMA smem descriptor (start, LBO, SBO in bytes)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
  uint64_t d = uint64_t(layout) << 61;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version (sm100)
  return d;               // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)                    // D format f32
         | (2u << 7) | (2u << 10)     // A, B tf32
         | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// element offsets (in floats) of the canonical no-swizzle layouts
// K-major: core matrix = 8 rows x 4 k (16 B per row); blocks [rowgroup][kchunk]
__device__ __forceinline__ int off_kmajor(int r, int k, int K) { return ((r >> 3) * (K >> 2) + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); }
// MN-major (tf32 needs SWIZZLE_128B_BASE32B): atoms of 32 mn x 4 k rows (512 B),
// atoms [katom][matom], the four 32-byte chunks of a 128-byte row XOR-ed with the row index
__device__ __forceinline__ int off_mnmajor(int r, int k, int R) {
  const int row = k & 3, col = r & 31;
  return ((k >> 2) * (R >> 5) + (r >> 5)) * 128 + row * 32 + (((col >> 3) ^ row) << 3) + (col & 7);
}
__device__ __forceinline__ int off_mnmajor_old(int r, int k, int R) { return ((k >> 3) * (R >> 2) + (r >> 2)) * 32 + (k & 7) * 4 + (r & 3); }

template <int M, int N, int K, int A_MN, int B_MN>
__global__ void umma_test(const float* A, const float* B, float* D, int* lanemap) {
  extern __shared__ __align__(1024) float sm[];
  float* Ahi = sm;
  float* Alo = Ahi + M * K;
  float* Bhi = Alo + M * K;
  float* Blo = Bhi + N * K;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = A[i], h = tf32_hi(x);
    const int o = A_MN ? off_mnmajor(r, k, M) : off_kmajor(r, k, K);
    Ahi[o] = h;
    Alo[o] = x - h;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = B[i], h = tf32_hi(x);
    const int o = B_MN ? off_mnmajor(r, k, N) : off_kmajor(r, k, K);
    Bhi[o] = h;
    Blo[o] = x - h;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // make st.shared visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    constexpr uint32_t idesc = make_idesc(M, N, A_MN, B_MN);
    for (int s = 0; s < K / 8; ++s) {
      uint64_t ad[2], bd[2];
      const float* As[2] = {Ahi, Alo};
      const float* Bs[2] = {Bhi, Blo};
      for (int p = 0; p < 2; ++p) {
        if (A_MN)  // MN-major SW128_32B: K step s = k-atoms 2s, 2s+1; LBO = mn-atom stride, SBO = k-atom stride
          ad[p] = make_desc(smem_u32(As[p] + 2 * s * (M / 32) * 128), 512, (M / 32) * 512, 1);
        else  // K-major: two k-chunks at LBO = 128 B, row groups at SBO
          ad[p] = make_desc(smem_u32(As[p] + (2 * s) * 32), 128, (K / 4) * 128);
        if (B_MN)
          bd[p] = make_desc(smem_u32(Bs[p] + 2 * s * (N / 32) * 128), 512, (N / 32) * 512, 1);
        else
          bd[p] = make_desc(smem_u32(Bs[p] + (2 * s) * 32), 128, (K / 4) * 128);
      }
      mma_tf32(tbase, ad[0], bd[0], idesc, s > 0 ? 1u : 0u);  // hi*hi
      mma_tf32(tbase, ad[0], bd[1], idesc, 1u);              // hi*lo
      mma_tf32(tbase, ad[1], bd[0], idesc, 1u);              // lo*hi
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // every warp reads its 32 lanes, N columns, 8 at a time
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    const uint32_t taddr = tbase + (uint32_t(warp * 32) << 16) + uint32_t(c);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int lane_row = warp * 32 + (tid & 31);
    for (int j = 0; j < 8; ++j) D[lane_row * N + c + j] = __uint_as_float(v[j]);
  }
  (void)lanemap;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128));
}

template <int M, int N, int K, int A_MN, int B_MN>
void run(const char* name) {
  std::vector<float> A(M * K), B(N * K), D(128 * N, 0.f);
  srand(1);
  for (auto& x : A) x = float(rand()) / RAND_MAX * 2.0f + 0.01f;
  for (auto& x : B) x = float(rand()) / RAND_MAX * 1e-3f + 1e-6f;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const size_t smem = size_t(2 * (M + N) * K) * 4;
  auto kern = umma_test<M, N, K, A_MN, B_MN>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  kern<<<1, 128, smem>>>(dA, dB, dD, nullptr);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  // find, for each logical row m, the TMEM lane holding it (match column values)
  double worst = 0.0;
  int mismatched_rows = 0;
  std::vector<int> where(M, -1);
  for (int m = 0; m < M; ++m) {
    std::vector<double> ref(N);
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * double(B[n * K + k]);
      ref[n] = s;
    }
    double best = 1e30;
    int bl = -1;
    for (int l = 0; l < 128; ++l) {
      double e = 0;
      for (int n = 0; n < N; ++n) e = std::max(e, std::fabs(D[l * N + n] - ref[n]) / std::fabs(ref[n]));
      if (e < best) best = e, bl = l;
    }
    where[m] = bl;
    worst = std::max(worst, best);
    if (best > 1e-5) ++mismatched_rows;
  }
  printf("%-34s max rel err %.3e, rows off %d, lanes of rows 0,1,15,16,31,32,63: %d %d %d %d %d %d %d\n", name,
         worst, mismatched_rows, where[0], where[1], where[std::min(15, M - 1)], where[std::min(16, M - 1)],
         where[std::min(31, M - 1)], where[std::min(32, M - 1)], where[M - 1]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}

// MN-major A probe: layout variant L (0: core = 4mn x 8k, blocks [kg][mc]; 1: core = 8mn-rows x 4k? blocks [kc][mg])
// and descriptor (lbo, sbo) chosen on the host.
template <int M, int N, int K>
__global__ void mn_probe(const float* A, const float* B, float* D, int L, uint32_t lbo, uint32_t sbo, int kstep_floats) {
  extern __shared__ __align__(1024) float sm[];
  float* As = sm;
  float* Bs = As + M * K;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    int o;
    if (L == 2) {  // MN-major SW128_32B: atoms of 32 mn x 4 k (512 B), [katom][matom], 32B chunks xor k-row
      const int row = k & 3, col = r & 31;
      o = ((k >> 2) * (M >> 5) + (r >> 5)) * 128 + row * 32 + (((col >> 3) ^ row) << 3) + (col & 7);
    } else {
      o = L == 0 ? off_mnmajor_old(r, k, M) : ((k >> 2) * (M >> 3) + (r >> 3)) * 32 + (r & 7) * 4 + (k & 3);
    }
    As[o] = tf32_hi(A[i]);
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    Bs[off_kmajor(r, k, K)] = tf32_hi(B[i]);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = make_idesc(M, N, 1, 0);
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t ad = make_desc(smem_u32(As + s * kstep_floats), lbo, sbo, L == 2 ? 1u : 0u);
      const uint64_t bd = make_desc(smem_u32(Bs + (2 * s) * 32), 128, (K / 4) * 128);
      mma_tf32(tbase, ad, bd, idesc, s > 0 ? 1u : 0u);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
                 : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    const uint32_t taddr = tbase + (uint32_t(warp * 32) << 16) + uint32_t(c);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[(warp * 32 + (tid & 31)) * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128));
}

void probe_mn() {
  constexpr int M = 128, N = 32, K = 32;
  std::vector<float> A(M * K), B(N * K), D(128 * N);
  srand(2);
  for (auto& x : A) x = float(rand()) / RAND_MAX + 0.01f;
  for (auto& x : B) x = float(rand()) / RAND_MAX + 0.01f;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  auto kern = mn_probe<M, N, K>;
  const size_t smem = size_t(M + N) * K * 4;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  struct V { int L; uint32_t lbo, sbo; int kstep; const char* name; } vs[] = {
    {0, (M / 4) * 128, 128, (M / 4) * 32, "L0 lbo=kg sbo=mc"},
    {0, 128, (M / 4) * 128, (M / 4) * 32, "L0 lbo=mc sbo=kg"},
    {1, (M / 8) * 128, 128, 2 * (M / 8) * 32, "L1 lbo=kc sbo=mg"},
    {1, 128, (M / 8) * 128, 2 * (M / 8) * 32, "L1 lbo=mg sbo=kc"},
    {2, 512, (M / 32) * 512, 2 * (M / 32) * 128, "SW32B lbo=matom sbo=katom"},
    {2, (M / 32) * 512, 512, 2 * (M / 32) * 128, "SW32B lbo=katom sbo=matom"},
  };
  for (auto& v : vs) {
    CK(cudaMemset(dD, 0, D.size() * 4));
    kern<<<1, 128, smem>>>(dA, dB, dD, v.L, v.lbo, v.sbo, v.kstep);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double worst = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
      double s = 0; for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * double(B[n * K + k]);
      worst = std::max(worst, std::fabs(D[m * N + n] - s) / s);
    }
    printf("MN probe %-22s max rel err %.3e  D[0][0]=%g\n", v.name, worst, D[0]);
  }
}

int main() {
  probe_mn();
  run<128, 32, 56, 0, 0>("M128 N32 K56 A:K B:K");
  run<128, 64, 64, 0, 0>("M128 N64 K64 A:K B:K");
  run<128, 32, 64, 1, 0>("M128 N32 K64 A:MN B:K");
  run<128, 64, 32, 0, 1>("M128 N64 K32 A:K B:MN");
  run<64, 64, 64, 0, 0>("M64 N64 K64 A:K B:K");
  run<64, 128, 32, 1, 1>("M64 N128 K32 A:MN B:MN");
  run<128, 96, 32, 1, 1>("M128 N96 K32 A:MN B:MN");
  run<64, 64, 128, 1, 0>("M64 N64 K128 A:MN B:K");
  return 0;
}

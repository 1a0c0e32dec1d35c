// tcgen05.mma kind::tf32 with the A operand in tensor memory ("TS": A from TMEM,
// B from shared memory), the form a K <= 64 tcgen05 solve would use for its
// phase A (A = dictionary rows, resident in TMEM for a whole mini-batch).
//  1. numerics: D[M=128][N] = A[128][K] * B[N][K]^T, 3xTF32 (hi*hi + hi*lo + lo*hi)
//     with A hi / lo written into TMEM by tcgen05.st, checked against fp64;
//  2. issue throughput of TS vs SS (A in smem) for M = 128, N in {16 .. 256};
//  3. occupancy of 2-CTA clusters with ~210 KB of dynamic shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_ts umma_ts.cu
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

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(ad), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(bar)));
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(su(bar)), "r"(parity));
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// K-major no-swizzle: core matrix 8 rows x 4 k (16 B rows), [rowgroup][kchunk]
__device__ __forceinline__ int off_k(int r, int k, int K) { return ((r >> 3) * (K >> 2) + (k >> 2)) * 32 + (r & 7) * 4 + (k & 3); }

// ---- 1. numerics (M = 128, K = 32, N given); 128 threads, A rows = lanes
template <int N>
__global__ void ts_numerics(const float* A, const float* B, float* D) {
  constexpr int M = 128, K = 32;
  extern __shared__ __align__(1024) float sm[];
  float* Bhi = sm;
  float* Blo = Bhi + N * K;
  __shared__ uint32_t tm;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    const float x = B[i], h = tf32_hi(x);
    Bhi[off_k(r, k, K)] = h;
    Blo[off_k(r, k, K)] = x - h;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tm)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t0 = tm;
  // A hi -> columns [128, 160), A lo -> [160, 192) of lane = row (this warp's quarter)
  {
    const int row = tid;
    uint32_t h[32], l[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float x = A[row * K + k], hh = tf32_hi(x);
      h[k] = __float_as_uint(hh);
      l[k] = __float_as_uint(x - hh);
    }
    const uint32_t lane_base = t0 + (uint32_t(32 * warp) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
        "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(lane_base + 128),
        "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]), "r"(h[8]), "r"(h[9]),
        "r"(h[10]), "r"(h[11]), "r"(h[12]), "r"(h[13]), "r"(h[14]), "r"(h[15]), "r"(h[16]), "r"(h[17]), "r"(h[18]),
        "r"(h[19]), "r"(h[20]), "r"(h[21]), "r"(h[22]), "r"(h[23]), "r"(h[24]), "r"(h[25]), "r"(h[26]), "r"(h[27]),
        "r"(h[28]), "r"(h[29]), "r"(h[30]), "r"(h[31]));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
        "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(lane_base + 160),
        "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]), "r"(l[8]), "r"(l[9]),
        "r"(l[10]), "r"(l[11]), "r"(l[12]), "r"(l[13]), "r"(l[14]), "r"(l[15]), "r"(l[16]), "r"(l[17]), "r"(l[18]),
        "r"(l[19]), "r"(l[20]), "r"(l[21]), "r"(l[22]), "r"(l[23]), "r"(l[24]), "r"(l[25]), "r"(l[26]), "r"(l[27]),
        "r"(l[28]), "r"(l[29]), "r"(l[30]), "r"(l[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    constexpr uint32_t id = idesc(M, N);
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t bh = desc(su(Bhi + 2 * s * 32), 128, (K / 4) * 128);
      const uint64_t bl = desc(su(Blo + 2 * s * 32), 128, (K / 4) * 128);
      mma_ts(t0, t0 + 128 + 8 * s, bh, id, s > 0);  // hi*hi
      mma_ts(t0, t0 + 128 + 8 * s, bl, id, 1);      // hi*lo
      mma_ts(t0, t0 + 160 + 8 * s, bh, id, 1);      // lo*hi
    }
    commit_wait(&bar, 0);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // D row = lane, columns 0..N-1
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(t0 + (uint32_t(32 * warp) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t0), "r"(256));
}

template <int N>
void numerics() {
  constexpr int M = 128, K = 32;
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(7);
  for (auto& x : A) x = float(std::exp(-6.0 * rand() / RAND_MAX));  // six decades
  for (auto& x : B) x = float(std::exp(-6.0 * rand() / RAND_MAX));
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  const int smem = 2 * N * K * 4;
  CK(cudaFuncSetAttribute(ts_numerics<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  ts_numerics<N><<<1, 128, smem>>>(dA, dB, dD);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += double(A[m * K + k]) * B[n * K + k];
      worst = fmax(worst, fabs(D[m * N + n] - s) / s);
    }
  printf("TS numerics M=128 N=%3d K=32 3xTF32: max rel err %.3e %s\n", N, worst, worst < 1e-5 ? "OK" : "FAIL");
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}

// ---- 2. throughput: one thread issues reps x 4 K-steps x NACC MMAs
template <int N, int NACC, bool TS>
__global__ void tput(int reps, long long* out) {
  extern __shared__ __align__(1024) float sm[];
  float* A = sm;           // 128 x 32
  float* B = A + 128 * 32;  // N x 32
  __shared__ uint32_t tm;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + N) * 32; i += blockDim.x) sm[i] = 0.001f * (i % 97);
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
    const uint32_t acol = 512 - 32;  // A operand columns (TS)
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t ad = desc(su(A) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128);
        const uint64_t bd = desc(su(B) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128);
#pragma unroll
        for (int c = 0; c < NACC; ++c) {
          if (TS)
            mma_ts(d0 + uint32_t(c * N), d0 + acol + 8 * s, bd, idesc(128, N), 1);
          else
            mma_ss(d0 + uint32_t(c * N), ad, bd, idesc(128, N), 1);
        }
      }
    commit_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int N, int NACC, bool TS>
void run(int reps = 256) {
  long long* d;
  long long h = 0;
  CK(cudaMalloc(&d, 8));
  auto k = tput<N, NACC, TS>;
  const int smem = (128 + N) * 32 * 4;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k<<<1, 128, smem>>>(2, d);
  CK(cudaDeviceSynchronize());
  k<<<1, 128, smem>>>(reps, d);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  const double cyc = double(h) / (double(reps) * 4 * NACC);
  printf("%s M=128 N=%3d K=8 acc=%d : %6.1f cycles/MMA  %6.0f MAC/clk/SM\n", TS ? "TS" : "SS", N, NACC, cyc,
         128.0 * N * 8 / cyc);
  cudaFree(d);
}

// ---- 3. cluster occupancy
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) pair_kernel(float* p) {
  extern __shared__ float sm[];
  if (p) p[threadIdx.x] = sm[threadIdx.x];
}

int main() {
  numerics<32>();
  numerics<64>();
  numerics<112>();
  numerics<128>();
  for (int ts = 0; ts < 2; ++ts) {
    if (ts) {
      run<16, 4, true>(); run<32, 4, true>(); run<32, 1, true>(); run<64, 4, true>(); run<64, 1, true>();
      run<112, 4, true>(); run<128, 4, true>(); run<256, 2, true>();
    } else {
      run<16, 4, false>(); run<32, 4, false>(); run<64, 4, false>(); run<112, 4, false>(); run<128, 4, false>();
      run<256, 2, false>();
    }
  }
  for (int kb : {160, 200, 210, 220, 227}) {
    const int smem = kb * 1024;
    CK(cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    int nc = 0;
    CK(cudaOccupancyMaxActiveClusters(&nc, pair_kernel, &cfg));
    printf("2-CTA clusters, 384 threads, %d KB smem: max active clusters %d (%d SMs)\n", kb, nc, 2 * nc);
  }
  return 0;
}

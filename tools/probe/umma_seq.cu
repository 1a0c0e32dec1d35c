// Timing of K1C's exact MMA sequences (csrc/kernels_tc.cuh) in isolation: phase A of one
// 128-row tile (7 k-steps x 3 TS MMAs, N = 64, B = h K-major with SBO = 1792 B) and the
// phase-B MMAs of one 32-row chunk (4 k-steps x {M128 N112 MN-major SW128_32B A, M128 N64}).
// Variants isolate the B stride, the A source and the accumulator chaining.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_seq umma_seq.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t(layout) << 61) | uint64_t((a >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amn, int bmn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(amn) << 15) | (uint32_t(bmn) << 16) | (uint32_t(N >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
               "l"(ad), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_wait(uint64_t* bar, uint32_t& ph) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(bar)));
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
                 : "=r"(done) : "r"(su(bar)), "r"(ph));
  ph ^= 1;
}

// mode 0: phase A as K1C (TS, SBO 1792); 1: phase A with SBO 1024 (KP = 32 layout);
// 2: phase A SS (A = W from smem, K-major); 3: phase A TS, 3 independent accumulators;
// 4: phase-B chunk as K1C; 5: phase-B chunk, A K-major no swizzle instead of MN-major
__global__ void seq(int mode, int reps, long long* out) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ uint32_t tm;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < 45056; i += blockDim.x) sm[i] = 1e-3f * (i % 89);
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
    const uint32_t t0 = tm;
    uint32_t ph = 0;
    const float* WB = sm;             // 112 x 256 (112 KB)
    const float* Wsm = sm;            // 128 x 56 K-major hi | lo (mode 2, overlays WB)
    const float* H = sm + 28672;      // h hi / lo: 64 x 56 each
    const float* Hl = H + 64 * 56;
    const float* op = sm + 36864;     // chunk A operands (mode 4/5): 2 x 4096
    long long best = 1LL << 60;
    for (int r = 0; r < reps; ++r) {
      const long long c0 = clock64();
      if (mode <= 3) {
        const uint32_t sbo = mode == 1 ? 1024 : 1792;
        const uint32_t id = idesc(128, 64, 0, 0);
        for (int s = 0; s < 7; ++s) {
          const uint64_t bh = desc(su(H + 64 * s), 128, sbo, 0), bl = desc(su(Hl + 64 * s), 128, sbo, 0);
          const uint32_t d = mode == 3 ? 0u : 384u;
          if (mode == 2) {
            const uint64_t ah = desc(su(Wsm + 64 * s), 128, 1792, 0), al = desc(su(Wsm + 4096 + 64 * s), 128, 1792, 0);
            mma_ss(t0 + 384, ah, bh, id, s > 0);
            mma_ss(t0 + 384, ah, bl, id, 1);
            mma_ss(t0 + 384, al, bh, id, 1);
          } else {
            mma_ts(t0 + (mode == 3 ? 256u : d), t0 + 8 * s, bh, id, s > 0);
            mma_ts(t0 + (mode == 3 ? 320u : d), t0 + 8 * s, bl, id, s > 0);
            mma_ts(t0 + (mode == 3 ? 448u : d), t0 + 56 + 8 * s, bh, id, s > 0 || mode != 3);
          }
        }
      } else if (mode >= 6) {
        // 6: full pass of phase B (8 chunks = 64 MMAs) into one D; 7: MMA2 into a second D;
        // 8: phase A both tiles interleaved (42 MMAs, 2 chains); 9: phase A tiles in sequence
        if (mode <= 7) {
          const uint32_t id1 = idesc(128, 112, 1, 0), id2 = idesc(128, 64, 1, 0);
          for (int c = 0; c < 8; ++c)
            for (int s = 0; s < 4; ++s) {
              const uint64_t a0 = desc(su(op + (c & 1) * 2048 + 2 * s * 512), 512, 2048, 1);
              const uint64_t a1 = desc(su(op + 4096 + (c & 1) * 0 + 2 * s * 512), 512, 2048, 1);
              const uint64_t bw = desc(su(WB + 64 * (4 * c + s) % 4096), 128, 8192, 0);
              mma_ss(t0 + 224, a0, bw, id1, c > 0 || s > 0);
              mma_ss(t0 + (mode == 7 ? 352u : 224u), a1, bw, id2, mode == 7 ? (c > 0 || s > 0) : 1);
            }
        } else {
          const uint32_t id = idesc(128, 64, 0, 0);
          for (int s = 0; s < 7; ++s)
            for (int t = 0; t < 2; ++t) {
              if (mode == 9 && t == 1) continue;
              const uint64_t bh = desc(su(H + 64 * s), 128, 1792, 0), bl = desc(su(Hl + 64 * s), 128, 1792, 0);
              const uint32_t d = 384 + 64 * t;
              mma_ts(t0 + d, t0 + 112 * t + 8 * s, bh, id, s > 0);
              mma_ts(t0 + d, t0 + 112 * t + 8 * s, bl, id, 1);
              mma_ts(t0 + d, t0 + 112 * t + 56 + 8 * s, bh, id, 1);
            }
          if (mode == 9)
            for (int s = 0; s < 7; ++s) {
              const uint64_t bh = desc(su(H + 64 * s), 128, 1792, 0), bl = desc(su(Hl + 64 * s), 128, 1792, 0);
              mma_ts(t0 + 448, t0 + 112 + 8 * s, bh, id, s > 0);
              mma_ts(t0 + 448, t0 + 112 + 8 * s, bl, id, 1);
              mma_ts(t0 + 448, t0 + 168 + 8 * s, bh, id, 1);
            }
        }
      } else {
        const uint32_t id1 = idesc(128, 112, mode == 4, 0), id2 = idesc(128, 64, mode == 4, 0);
        for (int s = 0; s < 4; ++s) {
          const uint64_t a0 = mode == 4 ? desc(su(op + 2 * s * 512), 512, 2048, 1) : desc(su(op + 64 * s), 128, 1024, 0);
          const uint64_t a1 = mode == 4 ? desc(su(op + 4096 + 2 * s * 512), 512, 2048, 1)
                                        : desc(su(op + 4096 + 64 * s), 128, 1024, 0);
          const uint64_t bw = desc(su(WB + 64 * s), 128, 8192, 0);
          mma_ss(t0 + 224, a0, bw, id1, s > 0);
          mma_ss(t0 + 224, a1, bw, id2, 1);
        }
      }
      commit_wait(&bar, ph);
      const long long c1 = clock64();
      if (c1 - c0 < best) best = c1 - c0;
    }
    out[mode] = best;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  long long* d;
  long long h[12] = {};
  cudaMalloc(&d, sizeof(h));
  cudaMemset(d, 0, sizeof(h));
  const int smem = 45056 * 4 + 1024;
  cudaFuncSetAttribute(seq, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int m = 0; m < 10; ++m) seq<<<1, 128, smem>>>(m, 20, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err: %s\n", cudaGetErrorString(e));
  const char* names[10] = {"phase A tile, TS, SBO 1792 (K1C)", "phase A tile, TS, SBO 1024", "phase A tile, SS",
                          "phase A tile, TS, 3 accumulators", "phase B chunk (K1C: MN-major SW128_32B A)",
                          "phase B chunk, K-major A", "phase B pass (64 MMAs, one D)", "phase B pass, MMA2 into a 2nd D",
                           "phase A both tiles interleaved (42)", "phase A tiles in sequence (42)"};
  const int nm[10] = {21, 21, 21, 21, 8, 8, 64, 64, 42, 42};
  for (int m = 0; m < 10; ++m)
    printf("%-45s %6lld cycles (%d MMAs: %.1f per MMA)\n", names[m], h[m], nm[m], double(h[m]) / nm[m]);
  return 0;
}

// K1T — the large-K solve (config 4: F=1025, K=256, 56 frames per CTA) with its
// phase B on the 5th-generation tensor cores (tcgen05, accumulators in TMEM).
// Same contract as solve_kernel / solve_large_kernel (SolveArgs).
//
// Per 32-row dictionary window c:
//   phase A  (mma.sync 3xTF32, all 8 warps)  Lam^T = h^T W^T  -> q, r
//   phase B  (tcgen05.mma kind::tf32, one thread)  D[k][n'] += W^T[k][rows] . [Q|R][rows][n']
//            3xTF32 (hi*hi + hi*lo + lo*hi) into two 128-lane TMEM tiles (k 0..127, 128..255),
//            N = 2*NT columns: num (q frames) then den (r frames); the whole pass accumulates in
//            TMEM, so there is no cross-warp reduction and no register pressure from num/den.
//   stats    (mma.sync 3xTF32) [sa|sb][row][k] = [Q|R] h^T on the statistics pass.
// The MMAs of window c run on the tensor cores while the warps compute phase A of window c+1.
//
// Shared-memory operand layouts (tools/probe/umma_test.cu):
//   A = W^T, MN-major (k contiguous) in 128B_BASE32B swizzle atoms of 32 k x 4 rows
//       (512 B; atoms [row atom][k atom]; the 32-byte chunks of a 128-byte atom row XOR-ed
//       with row % 4); hi = the raw fp32 bits (the tensor core truncates to tf32), lo = the
//       remainder; two window buffers (the next window is stored while the MMAs read this one).
//   B = [Q|R], K-major (rows contiguous) in no-swizzle core matrices of 8 n' x 4 rows (128 B).
#pragma once

#include <type_traits>

#include "kernels_large.cuh"

namespace isnmf_dev {

constexpr int kTcThreads = 256;
constexpr int kTcRows = 32;  // dictionary rows per window (the MMA K extent of a window)

template <int NB>
struct LargeTcShape {
  static constexpr int KP = 256;
  static constexpr int NT = 8 * NB;               // frames per CTA
  static constexpr int N2 = 2 * NT;               // MMA N: q frames then r frames
  static constexpr int KB = KP / 8;
  static constexpr int FMB = (NT + 15) / 16;
  static constexpr int TPW = (4 * FMB + 7) / 8;
  static constexpr int KPS = KP + 4;
  static constexpr int WS = KP + 4;               // global W32 row stride
  static constexpr int HROWS = 16 * FMB;
  static constexpr int AW = kTcRows * KP;         // floats of one A (W^T) window copy
  static constexpr int BW = N2 * kTcRows;         // floats of one B ([Q|R]) copy
  static constexpr uint32_t kTmemCols = 256;      // 2 tiles x N2 <= 256 columns
  static constexpr size_t smem_bytes() {
    return sizeof(float) * (size_t(HROWS) * KPS + 4 * size_t(AW) + 2 * size_t(BW)) + 1024;  // + alignment slack
  }
};

// MN-major SW128_32B position of W[row][k] (A = W^T: mn = k over R = 256, K = row)
__device__ __forceinline__ int tc_off_a(int k, int row) {
  const int r4 = row & 3;
  return ((row >> 2) * 8 + (k >> 5)) * 128 + r4 * 32 + ((((k & 31) >> 3) ^ r4) << 3) + (k & 7);
}
// K-major no-swizzle position of [Q|R][n'][row] (K = 32 rows)
__device__ __forceinline__ int tc_off_b(int n, int row) { return ((n >> 3) * 8 + (row >> 2)) * 32 + (n & 7) * 4 + (row & 3); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t(layout) << 61) | uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(a_mn) << 15) | (uint32_t(b_mn) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(
          dtmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
}

// ---- statistics chain (SolveArgs::chain): CTAs b with the same b / chain accumulate one plane.
// A window's [sa|sb] tile (2 x 256 k x 32 rows, 64 KB) is staged in shared memory (the lo copy of
// the dictionary window, which the statistics pass does not use: it splits W on the fly) and goes
// out as TMA bulk copies — rank 0 of a chain stores, the others `cp.reduce.async.bulk ... add.f32`
// (the addition happens in L2) — once the previous rank has published that window in
// chain_flags, so every cell is summed in rank order (bitwise reproducible) and a mini-batch
// leaves gridDim / chain planes for K2 instead of gridDim.
// Plane layout in chain mode: [window][sa|sb][k][32 rows], rows XOR-swizzled by k (tc_stat_off).
constexpr int kTcStatTile = 2 * 256 * kTcRows;  // floats of one window tile
__host__ __device__ __forceinline__ int tc_stat_off(int k, int row) {  // inside one [k][32] half tile
  return k * kTcRows + (row ^ (((k >> 1) & 3) << 3));
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
constexpr uint32_t kTcChainSpan = 4096;  // flag values per launch epoch: window + 1, span - 1 = abandoned
constexpr int kTcChainSpins = 1 << 19;  // bounded wait on the previous rank (ST_CHAIN_TIMEOUT)

template <int NB>
__global__ void __launch_bounds__(kTcThreads, 1) solve_large_tc_kernel(const SolveArgs a) {
  using L = LargeTcShape<NB>;
  constexpr int KP = L::KP, NT = L::NT, N2 = L::N2, KB = L::KB, FMB = L::FMB, TPW = L::TPW, KPS = L::KPS,
                WS = L::WS, HROWS = L::HROWS, AW = L::AW, BW = L::BW;
  pdl_wait();
  const bool chained = a.chain > 1 && a.do_stats && a.stats;
  if (*a.status || (a.halt && *a.halt)) {
    // a successor in the statistics chain must never wait for this CTA
    if (chained && threadIdx.x == 0) st_release_u32(a.chain_flags + blockIdx.x, a.chain_base + kTcChainSpan - 1u);
    return;
  }
  extern __shared__ __align__(16) float smem_raw[];
  // 1024-byte aligned base, as an offset from the shared array (keeps the pointers in the shared space)
  const uint32_t sbase = smem_addr(smem_raw);
  float* smem = smem_raw + ((((sbase + 1023u) & ~1023u) - sbase) >> 2);
  float* Ahi = smem;               // [2][AW]
  float* Alo = Ahi + 2 * AW;       // [2][AW]
  float* Bhi = Alo + 2 * AW;       // [BW]  raw q / r (the tensor core reads the tf32 part)
  float* Blo = Bhi + BW;           // [BW]
  float* Hs = Blo + BW;            // [HROWS][KPS], zero outside (n < nf, k < K)
  __shared__ const float* fptr[64];
  __shared__ double red[kTcThreads / 32];
  __shared__ double meanv[64];
  __shared__ int s_bad;
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t mma_bar;
  const int F = a.F, K = a.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int n0 = blockIdx.x * NT;
  const int nf = min(NT, a.nframes - n0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)),
                 "r"(L::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mma_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    s_bad = 0;
  }
  if (tid < 64) {
    const int64_t fr = tid < nf ? (a.vsel ? a.vsel[n0 + tid] : a.v0 + n0 + tid) : 0;
    fptr[tid] = a.V + fr * a.ldv;
  }
  for (int i = tid; i < HROWS * KPS; i += kTcThreads) Hs[i] = 0.0f;
  for (int i = tid; i < 2 * BW; i += kTcThreads) Bhi[i] = 0.0f;  // (and Blo)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (a.h0_mode == 2) {
    for (int n = warp; n < nf; n += kTcThreads / 32) {
      double s = 0.0;
      for (int f = lane; f < F; f += 32) s += double(fptr[n][f]);
      s = warp_sum_d(s);
      if (lane == 0) meanv[n] = s / double(F);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nf * K; idx += kTcThreads) {
    const int n = idx / K, k = idx - n * K;
    int hbad = 0;
    const int64_t col = a.h0_mode == 1 ? warm_col(a, n0 + n) : 0;
    const float val = solve_h0(a, n0 + n, k, col, a.h0_mode == 1 ? a.T[col] : 0u, a.h0_mode == 2 ? meanv[n] : 0.0, hbad);
    if (a.check_h0 && hbad) s_bad = 1;
    Hs[n * KPS + k] = val;
  }
  __syncthreads();
  const bool bad = s_bad != 0;
  const float eps = a.eps;
  const int nch = (F + kTcRows - 1) / kTcRows;

  // ---- window staging: 32 rows x 256 k of W as 8 float4 per thread, through registers
  float4 wreg[8];
  auto fetch_w = [&](int c) {  // global -> registers (rows past F read as 0)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = tid + kTcThreads * j, row = i >> 6, k0 = 4 * (i & 63);
      const int f = c * kTcRows + row;
      wreg[j] = f < F ? __ldg(reinterpret_cast<const float4*>(a.W32 + size_t(f) * WS + k0))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  // chained statistics pass: the lo copy's space is the staging tile of the window statistics,
  // and phase A takes the remainders from the hi copy on the fly
  bool lo_fly = false;
  auto rem = [](float v) { return v - __uint_as_float(__float_as_uint(v) & 0xffffe000u); };
  auto store_w = [&](int buf) {  // registers -> A hi / lo (MN-major swizzled)
    float* hi = Ahi + buf * AW;
    float* lo = Alo + buf * AW;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = tid + kTcThreads * j, row = i >> 6, k0 = 4 * (i & 63);
      const int o = tc_off_a(k0, row);
      const float4 x = wreg[j];
      *reinterpret_cast<float4*>(hi + o) = x;
      if (!lo_fly) *reinterpret_cast<float4*>(lo + o) = make_float4(rem(x.x), rem(x.y), rem(x.z), rem(x.w));
    }
  };

  // ---- statistics chain state (thread 0 issues and publishes the window tiles)
  const int chain_rank = chained ? int(blockIdx.x) % a.chain : 0;
  float* const stage = Alo;  // [sa|sb][k][32 rows] of one window (kTcStatTile floats = both lo buffers)
  uint32_t chain_pending = 0;  // thread 0: flag value to publish once the outstanding tile has landed
  auto chain_release = [&]() {
    if (chain_pending) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async;" ::: "memory");
      st_release_u32(a.chain_flags + blockIdx.x, chain_pending);
      chain_pending = 0;
    }
  };

  // ---- phase A (mma.sync) of window c: accumulators only; the epilogue writes B later
  const int tile0 = warp * TPW;
  const int fmb = min(tile0, 4 * FMB - 1) / 4;
  float acc[TPW][2][4];
  float vv[TPW][4];
  auto phase_a = [&](int c, auto fly_tag) {
    constexpr bool kFly = decltype(fly_tag)::value;  // remainders of W from the hi copy on the fly
    const int c0 = c * kTcRows, rows = min(kTcRows, F - c0);
    const float* Wc = Ahi + (c & 1) * AW;
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[i][0][e] = acc[i][1][e] = 0.0f;
        const int n = 16 * fmb + g + 8 * (e >> 1), row = 8 * ((tile0 + i) & 3) + 2 * t + (e & 1);
        vv[i][e] = (tile0 + i < 4 * FMB && n < nf && row < rows) ? __ldg(fptr[n] + c0 + row) : 0.0f;
      }
    const float* hrow = Hs + (16 * fmb + g) * KPS + t;
    // W fragments straight from the swizzled window: for row r = 8 rnb + g and
    // k = 32 q + 8 u + t, tc_off_a = base(r) + 128 q + ((u ^ r%4) << 3) + t; the
    // remainder half comes from the lo copy the tensor-core phase B uses
    const float* wbase[TPW];
    const float* lbase[TPW];
    int xo[4];
    {
      const int r4 = g & 3;  // row % 4 (8 rnb is a multiple of 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) xo[u] = ((u ^ r4) << 3) + t;
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int row = 8 * ((tile0 + i) & 3) + g;
        const int b = (row >> 2) * 8 * 128 + r4 * 32;
        wbase[i] = Wc + b;
        lbase[i] = Alo + (c & 1) * AW + b;
      }
    }
#pragma unroll 1
    for (int q = 0; q < KB / 4; ++q) {
      if (kFly && q == 2) chain_release();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kb = 4 * q + u, p = u & 1;
        const float* hp = hrow + 8 * kb;
        uint32_t ah[4], al[4];
        split_tf32(hp[0], ah[0], al[0]);
        split_tf32(hp[8 * KPS], ah[1], al[1]);
        split_tf32(hp[4], ah[2], al[2]);
        split_tf32(hp[8 * KPS + 4], ah[3], al[3]);
        uint32_t bh[TPW][2], bl[TPW][2];
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          const int o = 128 * q + xo[u];
          const float w0 = wbase[i][o], w1 = wbase[i][o + 4];
          bh[i][0] = __float_as_uint(w0);
          bh[i][1] = __float_as_uint(w1);
          bl[i][0] = __float_as_uint(kFly ? rem(w0) : lbase[i][o]);
          bl[i][1] = __float_as_uint(kFly ? rem(w1) : lbase[i][o + 4]);
        }
#pragma unroll
        for (int i = 0; i < TPW; ++i) mma_tf32(acc[i][p], al, bh[i][0], bh[i][1]);
#pragma unroll
        for (int i = 0; i < TPW; ++i) mma_tf32(acc[i][p], ah, bl[i][0], bl[i][1]);
#pragma unroll
        for (int i = 0; i < TPW; ++i) mma_tf32(acc[i][p], ah, bh[i][0], bh[i][1]);
      }
    }
  };
  float divacc = 0.0f;
  auto phase_a_epilogue = [&](int c, bool want_div) {  // q, r -> B (hi raw, lo remainder)
    const int rows = min(kTcRows, F - c * kTcRows);
#pragma unroll
    for (int i = 0; i < TPW; ++i) {
      if (tile0 + i >= 4 * FMB) continue;
      const int rnb = (tile0 + i) & 3;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int n = 16 * fmb + g + 8 * (e >> 1), row = 8 * rnb + 2 * t + (e & 1);
        if (n >= NT) continue;
        const bool valid = n < nf && row < rows;
        const float r = rcp_approx(acc[i][0][e] + acc[i][1][e] + eps);
        const float vpe = vv[i][e] + eps;
        if (want_div && valid) divacc += is_term_ratio(vpe * r);
        const float q = valid ? vpe * r * r : 0.0f, rr = valid ? r : 0.0f;
        const int oq = tc_off_b(n, row), orr = tc_off_b(NT + n, row);
        Bhi[oq] = q;
        Blo[oq] = q - __uint_as_float(__float_as_uint(q) & 0xffffe000u);
        Bhi[orr] = rr;
        Blo[orr] = rr - __uint_as_float(__float_as_uint(rr) & 0xffffe000u);
      }
    }
  };

  uint32_t mma_phase = 0;
  const int passes = bad ? 0 : a.iters + (a.do_stats ? 1 : 0);
  for (int pass = 0; pass < passes; ++pass) {
    const bool stats_pass = pass == a.iters;
    const bool want_div = a.div_first ? pass == 0 : stats_pass;
    if (stats_pass) pdl_trigger();
    lo_fly = stats_pass && chained;
    // prologue: windows 0 and 1 staged, phase A of window 0, B(0)
    fetch_w(0);
    store_w(0);
    if (nch > 1) fetch_w(1);
    __syncthreads();
    if (lo_fly)
      phase_a(0, std::true_type{});
    else
      phase_a(0, std::false_type{});
    phase_a_epilogue(0, want_div);
    if (nch > 1) {
      store_w(1);
      if (nch > 2) fetch_w(2);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    for (int c = 0; c < nch; ++c) {
      const int c0 = c * kTcRows, rows = min(kTcRows, F - c0);
#ifdef ISNMF_PHASE_PROF
      const bool stamp = a.prof && blockIdx.x == 0 && pass == 1 && c < 40;
#define TC_STAMP(i, who) \
  if (stamp && tid == (who)) a.prof[c * 8 + (i)] = clock64()
#else
#define TC_STAMP(i, who)
#endif
      TC_STAMP(0, 32);
      if (!stats_pass) {
        if (tid == 0) {  // phase B of window c on the tensor cores
          asm volatile("tcgen05.fence::after_thread_sync;");
          constexpr uint32_t idesc = umma_idesc_tf32(128, N2, 1, 0);
          const float* ah = Ahi + (c & 1) * AW;
          const float* al = Alo + (c & 1) * AW;
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int s = 0; s < kTcRows / 8; ++s) {
              // A: k atoms 4mt.. (128 k), row atoms 2s, 2s+1; B: row chunks 2s, 2s+1
              const uint32_t aoff = uint32_t(2 * s * 8 * 128 + 4 * mt * 128) * 4u;
              const uint64_t adh = umma_desc(smem_addr(ah) + aoff, 512, 8 * 512, 1);
              const uint64_t adl = umma_desc(smem_addr(al) + aoff, 512, 8 * 512, 1);
              const uint64_t bdh = umma_desc(smem_addr(Bhi) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128, 0);
              const uint64_t bdl = umma_desc(smem_addr(Blo) + uint32_t(2 * s * 32) * 4u, 128, 8 * 128, 0);
              const uint32_t d = tmem + uint32_t(mt * N2);
              umma_tf32(d, adl, bdh, idesc, (c > 0 || s > 0) ? 1u : 0u);
              umma_tf32(d, adh, bdl, idesc, 1u);
              umma_tf32(d, adh, bdh, idesc, 1u);
            }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_addr(&mma_bar)));
        }
      } else if (a.stats) {
        // statistics of window c (mma.sync): [sa|sb][row][k] = sum_n [q|r][row][n] h[n][k]
        constexpr int KNW = 4;  // k blocks of 8 per warp
        float sa[2][KNW][4], sb[2][KNW][4];
#pragma unroll
        for (int rm = 0; rm < 2; ++rm)
#pragma unroll
          for (int j = 0; j < KNW; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) sa[rm][j][e] = sb[rm][j][e] = 0.0f;
#pragma unroll 1
        for (int kb = 0; kb < NB; ++kb) {
          uint32_t hh[KNW][2], hl[KNW][2];
#pragma unroll
          for (int j = 0; j < KNW; ++j) {
            const float* hp = Hs + (8 * kb + t) * KPS + 8 * (warp * KNW + j) + g;
            split_tf32(hp[0], hh[j][0], hl[j][0]);
            split_tf32(hp[4 * KPS], hh[j][1], hl[j][1]);
          }
#pragma unroll
          for (int rm = 0; rm < 2; ++rm) {
            const int r0 = 16 * rm + g, n = 8 * kb + t;
            uint32_t qh[4], ql[4], rh[4], rl[4];
            const int oq[4] = {tc_off_b(n, r0), tc_off_b(n, r0 + 8), tc_off_b(n + 4, r0), tc_off_b(n + 4, r0 + 8)};
#pragma unroll
            for (int e = 0; e < 4; ++e) {  // hi = raw q / r, lo from the remainder copy phase B uses
              qh[e] = __float_as_uint(Bhi[oq[e]]);
              ql[e] = __float_as_uint(Blo[oq[e]]);
              rh[e] = __float_as_uint(Bhi[oq[e] + NT * 32]);  // tc_off_b(NT + n, r) = tc_off_b(n, r) + 32 NT
              rl[e] = __float_as_uint(Blo[oq[e] + NT * 32]);
            }
#pragma unroll
            for (int j = 0; j < KNW; ++j) {
              mma_tf32(sa[rm][j], ql, hh[j][0], hh[j][1]);
              mma_tf32(sb[rm][j], rl, hh[j][0], hh[j][1]);
            }
#pragma unroll
            for (int j = 0; j < KNW; ++j) {
              mma_tf32(sa[rm][j], qh, hl[j][0], hl[j][1]);
              mma_tf32(sb[rm][j], rh, hl[j][0], hl[j][1]);
            }
#pragma unroll
            for (int j = 0; j < KNW; ++j) {
              mma_tf32(sa[rm][j], qh, hh[j][0], hh[j][1]);
              mma_tf32(sb[rm][j], rh, hh[j][0], hh[j][1]);
            }
          }
        }
        if (!chained) {
          const int FP = (F + 3) & ~3;
          ISNMF_DASSERT(a.stats_cap == 0 || int(blockIdx.x) < a.stats_cap);
          float* outA = a.stats + size_t(blockIdx.x) * 2 * FP * KP;
          float* outB = outA + size_t(FP) * KP;
#pragma unroll
          for (int rm = 0; rm < 2; ++rm)
#pragma unroll
            for (int j = 0; j < KNW; ++j)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int row = 16 * rm + g + 8 * (e >> 1), k = 8 * (warp * KNW + j) + 2 * t + (e & 1);
                if (row < rows) {
                  outA[size_t(k) * FP + c0 + row] = sa[rm][j][e];
                  outB[size_t(k) * FP + c0 + row] = sb[rm][j][e];
                }
              }
        } else {
          // the tile of window c - 1 has left the staging space (chain_release in phase A of this
          // window, ahead of the barrier that ended the previous iteration)
#pragma unroll
          for (int rm = 0; rm < 2; ++rm)
#pragma unroll
            for (int j = 0; j < KNW; ++j)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int row = 16 * rm + g + 8 * (e >> 1), k = 8 * (warp * KNW + j) + 2 * t + (e & 1);
                const int o = tc_stat_off(k, row);
                stage[o] = sa[rm][j][e];  // rows past F carry exact zeros (q = r = 0 there)
                stage[KP * kTcRows + o] = sb[rm][j][e];
              }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
          if (tid == 0) {
            const uint32_t target = a.chain_base + uint32_t(c) + 1u;
            const int plane = int(blockIdx.x) / a.chain;
            ISNMF_DASSERT(a.stats_cap == 0 || plane < a.stats_cap);
            float* dst = a.stats + (size_t(plane) * nch + c) * kTcStatTile;
            if (chain_rank > 0) {
              const uint32_t* pf = a.chain_flags + blockIdx.x - 1;
              int spins = 0;
              while (int32_t(ld_acquire_u32(pf) - target) < 0)
                if (++spins > kTcChainSpins) {
                  atomicOr(a.status, ST_CHAIN_TIMEOUT);
                  break;
                }
              asm volatile("fence.proxy.async;" ::: "memory");
            }
            constexpr uint32_t kPiece = kTcStatTile * 4 / 4;  // four 16 KB copies
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t src = smem_addr(stage) + i * kPiece;
              const char* d = reinterpret_cast<const char*>(dst) + i * kPiece;
              if (chain_rank == 0)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(src),
                             "r"(kPiece)
                             : "memory");
              else
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(d),
                             "r"(src), "r"(kPiece)
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            chain_pending = target;
          }
        }
      }
      TC_STAMP(1, 0);
      if (c + 1 < nch) {  // on the warps while the tensor cores run window c
        if (lo_fly)
          phase_a(c + 1, std::true_type{});
        else
          phase_a(c + 1, std::false_type{});
      }
      if (tid == 0) chain_release();     // (the last window's tile; otherwise done inside phase A)
      TC_STAMP(2, 32);
      if (!stats_pass) {
        mbar_wait(&mma_bar, mma_phase);  // window c's MMAs are done with A buffer c & 1 and B
        mma_phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
      } else {
        __syncthreads();  // the statistics are done with B
      }
      TC_STAMP(3, 32);
      if (c + 1 < nch) phase_a_epilogue(c + 1, want_div);
      TC_STAMP(4, 32);
      if (c + 2 < nch) {
        store_w(c & 1);
        if (c + 3 < nch) fetch_w(c + 3);
      }
      TC_STAMP(5, 32);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      TC_STAMP(6, 32);
    }
#undef TC_STAMP
    if (!stats_pass) {
      // h update from TMEM: warp (quarter q = warp & 3, column half ch = warp >> 2) reads
      // lanes 32q.. of both k tiles, num at column n, den at column NT + n
      const int q = warp & 3, ch = warp >> 2;
      constexpr int NG = NT / 4;  // column groups of 4 (NT = 8 NB)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int k = 128 * mt + 32 * q + lane;
        const uint32_t tl = tmem + (uint32_t(32 * q) << 16) + uint32_t(mt * N2);
#pragma unroll 1
        for (int gi = ch; gi < NG; gi += 2) {
          uint32_t vn[4], vd[4];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(vn[0]), "=r"(vn[1]), "=r"(vn[2]), "=r"(vn[3])
                       : "r"(tl + uint32_t(4 * gi)));
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(vd[0]), "=r"(vd[1]), "=r"(vd[2]), "=r"(vd[3])
                       : "r"(tl + uint32_t(NT + 4 * gi)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = 4 * gi + e;
            if (n < nf && k < K) {
              float& h = Hs[n * KPS + k];
              h = h * sqrtf(__uint_as_float(vn[e]) / __uint_as_float(vd[e]));
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
    }
  }

  if (chained && bad && tid == 0) st_release_u32(a.chain_flags + blockIdx.x, a.chain_base + kTcChainSpan - 1u);
  if (a.divpart && !bad) {
    double d = warp_sum_d(double(divacc));
    if (lane == 0) red[warp] = d;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kTcThreads / 32; ++w) s += red[w];
      a.divpart[blockIdx.x] = s;
    }
  }
  if (!bad) write_final_h(a, n0, nf, [&](int n, int k) { return Hs[n * KPS + k]; });
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmemCols));
  if (bad && tid == 0) atomicOr(a.status, ST_NONPOS_INIT);
}

}  // namespace isnmf_dev

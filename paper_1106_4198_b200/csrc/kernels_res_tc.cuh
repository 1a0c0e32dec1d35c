// K1R — the config-3 solve (48 < K <= 64, up to 32 frames per CTA) with the
// dictionary resident in shared memory and phase B on the tcgen05 tensor cores.
// Same contract as solve_kernel (SolveArgs).
//
// The dictionary lives in shared memory once per launch, stored as the tcgen05
// A operand (W^T, MN-major 128B_BASE32B atoms of 32 k x 4 rows, the raw fp32 as
// the tf32 "hi" part); the rows are visited in 32-row windows:
//   phase A  (mma.sync 3xTF32, 8 warps x one 16-frame x 8-row tile) Lam^T = h^T W^T,
//            A = h^T from per-pass hi/lo fragment copies, B = W from the resident
//            copy plus the window's remainder copy -> q, r staged as the phase-B operand
//   phase B  (tcgen05.mma kind::tf32, M = 64 k x N = 2 NT, 3xTF32) D[k][n'] += W^T [Q|R]
//            into one TMEM tile for the whole pass: no cross-warp reduction
//   stats    (mma.sync 3xTF32) [sa|sb][row][k] = [Q|R] h^T on the statistics pass.
// Windows are double buffered (the Q/R operand and W's remainder copy), so the
// MMAs of window c run while the warps compute phase A of window c+1.
#pragma once

#include "kernels_large_tc.cuh"

namespace isnmf_dev {

constexpr int kRsThreads = 256;
constexpr int kRsRows = 32;

template <int NB>  // frames per CTA = 8 NB (NB <= 4)
struct ResTcShape {
  static constexpr int KP = 64;
  static constexpr int NT = 8 * NB;
  static constexpr int N2 = 2 * NT;
  static constexpr int KB = KP / 8;              // 8 k blocks
  static constexpr int FMB = (NT + 15) / 16;     // frame blocks of 16 (phase A M)
  static constexpr int TPW = (FMB * 4 + 7) / 8;  // phase-A tiles per warp per window (<= 1)
  static constexpr int KPS = KP + 4;             // h row stride
  static constexpr int WS = KP + 4;              // global W32 row stride (ws_for(64))
  static constexpr int WL = kRsRows * KP;        // floats of one window remainder copy
  static constexpr int BW = N2 * kRsRows;        // floats of one Q/R operand copy
  static constexpr int HF = FMB * KB * 32 * 4;   // floats of one h fragment copy
  static constexpr uint32_t kTmemCols = 64;
  static size_t smem_bytes(int F) {
    const size_t rp = size_t((F + 7) / 8) * 8;  // rows padded to whole MMA K steps
    return sizeof(float) * (rp * KP + 2 * size_t(WL) + 4 * size_t(BW) + size_t(16 * FMB) * KPS + 2 * size_t(HF)) +
           1024;
  }
};

// MN-major SW128_32B position of W[row][k] for KP = 64 (two 32-k atoms per 4-row atom)
__device__ __forceinline__ int rs_off(int k, int row) {
  const int r4 = row & 3;
  return ((row >> 2) * 2 + (k >> 5)) * 128 + r4 * 32 + ((((k & 31) >> 3) ^ r4) << 3) + (k & 7);
}

template <int NB>
__global__ void __launch_bounds__(kRsThreads, 1) solve_res_tc_kernel(const SolveArgs a) {
  using L = ResTcShape<NB>;
  constexpr int KP = L::KP, NT = L::NT, N2 = L::N2, KB = L::KB, FMB = L::FMB, KPS = L::KPS, WS = L::WS,
                WL = L::WL, BW = L::BW, HF = L::HF;
  static_assert(NB <= 4 && L::TPW == 1, "one phase-A tile per warp");
  pdl_wait();
  if (*a.status || (a.halt && *a.halt)) return;
  extern __shared__ __align__(16) float smem_raw[];
  // 1024-byte aligned base, as an offset from the shared array (keeps the pointers in the shared space)
  const uint32_t sbase = smem_addr(smem_raw);
  float* smem = smem_raw + ((((sbase + 1023u) & ~1023u) - sbase) >> 2);
  const int F = a.F, K = a.K;
  const int RP = (F + 7) / 8 * 8;
  float* Whi = smem;                    // [RP/4 row atoms][2 k atoms][128]
  float* Wlo = Whi + RP * KP;           // [2][WL] window remainder copies
  float* Bhi = Wlo + 2 * WL;            // [2][BW] raw q / r, K-major
  float* Blo = Bhi + 2 * BW;            // [2][BW]
  float* Hs = Blo + 2 * BW;             // [16 FMB][KPS]
  float* Hhi = Hs + 16 * FMB * KPS;     // [HF] h^T fragments (tf32 hi)
  float* Hlo = Hhi + HF;                // [HF] (remainder)
  __shared__ const float* fptr[32];
  __shared__ double red[kRsThreads / 32];
  __shared__ double meanv[32];
  __shared__ int s_bad;
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t mma_bar;
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
  if (tid < 32) {
    const int64_t fr = tid < nf ? (a.vsel ? a.vsel[n0 + tid] : a.v0 + n0 + tid) : 0;
    fptr[tid] = a.V + fr * a.ldv;
  }
  // resident dictionary (rows past F zero), h and its fragment copies zeroed
  for (int i = tid; i < RP * (KP / 4); i += kRsThreads) {
    const int row = i / (KP / 4), k0 = 4 * (i % (KP / 4));
    const float4 x = row < F ? __ldg(reinterpret_cast<const float4*>(a.W32 + size_t(row) * WS + k0))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(Whi + rs_off(k0, row)) = x;
  }
  for (int i = tid; i < 16 * FMB * KPS; i += kRsThreads) Hs[i] = 0.0f;
  for (int i = tid; i < 2 * HF; i += kRsThreads) Hhi[i] = 0.0f;
  for (int i = tid; i < 4 * BW; i += kRsThreads) Bhi[i] = 0.0f;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  if (a.h0_mode == 2) {
    for (int n = warp; n < nf; n += kRsThreads / 32) {
      double s = 0.0;
      for (int f = lane; f < F; f += 32) s += double(fptr[n][f]);
      s = warp_sum_d(s);
      if (lane == 0) meanv[n] = s / double(F);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nf * K; idx += kRsThreads) {
    const int n = idx / K, k = idx - n * K;
    float val;
    if (a.h0_mode == 0) {
      val = a.H0[size_t(n0 + n) * K + k];
    } else if (a.h0_mode == 1) {
      const int64_t col = a.widx ? int64_t(a.widx[n0 + n]) : (a.wbase + n0 + n) % a.wmod;
      const uint32_t tag = a.T[col];
      val = float(double(a.U[size_t(col) * K + k]) * (a.P[size_t(a.c_now) * K + k] / a.P[size_t(tag) * K + k]));
    } else {
      const double mv = meanv[n] > a.epsd ? meanv[n] : a.epsd;
      val = float(mv / a.kst->kmeanw * a.u01[size_t(n0 + n) * K + k]);
    }
    if (a.hscale) val = float(double(val) * a.hscale[k]);
    if (a.check_h0 && !(val > 0.0f)) s_bad = 1;
    Hs[n * KPS + k] = val;
    put_hfrag(Hhi, Hlo, hfrag_index<KB>(n, k), val);
  }
  __syncthreads();
  const bool bad = s_bad != 0;
  const float eps = a.eps;
  const int nwin = (F + kRsRows - 1) / kRsRows;

  // remainder copy of window c's rows (8 floats per thread), in the window-local swizzled layout
  auto make_lo = [&](int c) {
    float* lo = Wlo + (c & 1) * WL;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int i = tid + kRsThreads * j, rl = i >> 4, k0 = 4 * (i & 15);
      const float4 x = *reinterpret_cast<const float4*>(Whi + rs_off(k0, kRsRows * c + rl));
      auto rem = [](float v) { return v - __uint_as_float(__float_as_uint(v) & 0xffffe000u); };
      *reinterpret_cast<float4*>(lo + rs_off(k0, rl)) = make_float4(rem(x.x), rem(x.y), rem(x.z), rem(x.w));
    }
  };

  // phase A of window c (one tile per warp: frames 16 fmb.., rows 8 rnb..)
  const int fmb = warp >> 2, rnb = warp & 3;
  const bool has_tile = fmb < FMB;
  float acc[2][4], vv[4];
  int xo[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) xo[u] = ((u ^ (g & 3)) << 3) + t;
  auto phase_a = [&](int c) {
    const int c0 = c * kRsRows, rows = min(kRsRows, F - c0);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc[0][e] = acc[1][e] = 0.0f;
      const int n = 16 * fmb + g + 8 * (e >> 1), row = 8 * rnb + 2 * t + (e & 1);
      vv[e] = (has_tile && n < nf && row < rows) ? __ldg(fptr[n] + c0 + row) : 0.0f;
    }
    if (!has_tile || 8 * rnb >= rows) return;
    const int row = c0 + 8 * rnb + g;
    const float* wh = Whi + ((row >> 2) * 2) * 128 + (g & 3) * 32;
    const float* wl = Wlo + (c & 1) * WL + ((2 * rnb + (g >> 2)) * 2) * 128 + (g & 3) * 32;
#pragma unroll
    for (int kb = 0; kb < KB; ++kb) {
      const int p = kb & 1, o = (kb >> 2) * 128 + xo[kb & 3];
      uint32_t ah[4], al[4];
      const float4 x = *reinterpret_cast<const float4*>(Hhi + ((fmb * KB + kb) * 32 + lane) * 4);
      const float4 y = *reinterpret_cast<const float4*>(Hlo + ((fmb * KB + kb) * 32 + lane) * 4);
      ah[0] = __float_as_uint(x.x);
      ah[1] = __float_as_uint(x.y);
      ah[2] = __float_as_uint(x.z);
      ah[3] = __float_as_uint(x.w);
      al[0] = __float_as_uint(y.x);
      al[1] = __float_as_uint(y.y);
      al[2] = __float_as_uint(y.z);
      al[3] = __float_as_uint(y.w);
      const uint32_t bh0 = __float_as_uint(wh[o]), bh1 = __float_as_uint(wh[o + 4]);
      const uint32_t bl0 = __float_as_uint(wl[o]), bl1 = __float_as_uint(wl[o + 4]);
      mma_tf32(acc[p], al, bh0, bh1);
      mma_tf32(acc[p], ah, bl0, bl1);
      mma_tf32(acc[p], ah, bh0, bh1);
    }
  };
  float divacc = 0.0f;
  auto phase_a_epilogue = [&](int c, bool want_div) {  // q, r -> Q/R operand buffer c & 1
    if (!has_tile) return;
    const int rows = min(kRsRows, F - c * kRsRows);
    float* bh = Bhi + (c & 1) * BW;
    float* bl = Blo + (c & 1) * BW;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int n = 16 * fmb + g + 8 * (e >> 1), row = 8 * rnb + 2 * t + (e & 1);
      if (n >= NT) continue;
      const bool valid = n < nf && row < rows;
      const float r = rcp_approx(acc[0][e] + acc[1][e] + eps);
      const float vpe = vv[e] + eps;
      if (want_div && valid) divacc += is_term_ratio(vpe * r);
      const float q = valid ? vpe * r * r : 0.0f, rr = valid ? r : 0.0f;
      const int oq = tc_off_b(n, row), orr = oq + 32 * NT;
      bh[oq] = q;
      bl[oq] = q - __uint_as_float(__float_as_uint(q) & 0xffffe000u);
      bh[orr] = rr;
      bl[orr] = rr - __uint_as_float(__float_as_uint(rr) & 0xffffe000u);
    }
  };

  uint32_t mma_phase = 0;
  const int passes = bad ? 0 : a.iters + (a.do_stats ? 1 : 0);
  for (int pass = 0; pass < passes; ++pass) {
    const bool stats_pass = pass == a.iters;
    const bool want_div = a.div_first ? pass == 0 : stats_pass;
    if (stats_pass) pdl_trigger();
    make_lo(0);
    __syncthreads();
    phase_a(0);
    phase_a_epilogue(0, want_div);
    if (nwin > 1) make_lo(1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    for (int c = 0; c < nwin; ++c) {
      const int c0 = c * kRsRows, rows = min(kRsRows, F - c0);
      if (!stats_pass) {
        if (tid == 0) {  // phase B of window c on the tensor cores
          asm volatile("tcgen05.fence::after_thread_sync;");
          constexpr uint32_t idesc = umma_idesc_tf32(64, N2, 1, 0);
          const uint32_t wh = smem_addr(Whi) + uint32_t((c0 >> 2) * 2 * 128) * 4u;
          const uint32_t wl = smem_addr(Wlo + (c & 1) * WL);
          const uint32_t qh = smem_addr(Bhi + (c & 1) * BW), ql = smem_addr(Blo + (c & 1) * BW);
          const int steps = (rows + 7) / 8;
          for (int s = 0; s < steps; ++s) {
            const uint64_t adh = umma_desc(wh + uint32_t(2 * s * 2 * 128) * 4u, 512, 2 * 512, 1);
            const uint64_t adl = umma_desc(wl + uint32_t(2 * s * 2 * 128) * 4u, 512, 2 * 512, 1);
            const uint64_t bdh = umma_desc(qh + uint32_t(2 * s * 32) * 4u, 128, 8 * 128, 0);
            const uint64_t bdl = umma_desc(ql + uint32_t(2 * s * 32) * 4u, 128, 8 * 128, 0);
            umma_tf32(tmem, adl, bdh, idesc, (c > 0 || s > 0) ? 1u : 0u);
            umma_tf32(tmem, adh, bdl, idesc, 1u);
            umma_tf32(tmem, adh, bdh, idesc, 1u);
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_addr(&mma_bar)));
        }
      } else if (a.stats) {
        // statistics of window c (mma.sync): warp -> k block 8 warp.., row blocks 0/1 of 16
        const float* bh = Bhi + (c & 1) * BW;
        const float* bl = Blo + (c & 1) * BW;
        float sa[2][4], sb[2][4];
#pragma unroll
        for (int rm = 0; rm < 2; ++rm)
#pragma unroll
          for (int e = 0; e < 4; ++e) sa[rm][e] = sb[rm][e] = 0.0f;
#pragma unroll
        for (int kb = 0; kb < NB; ++kb) {
          uint32_t hh[2], hl[2];
          const float* hp = Hs + (8 * kb + t) * KPS + 8 * warp + g;
          split_tf32(hp[0], hh[0], hl[0]);
          split_tf32(hp[4 * KPS], hh[1], hl[1]);
#pragma unroll
          for (int rm = 0; rm < 2; ++rm) {
            const int r0 = 16 * rm + g, n = 8 * kb + t;
            const int oq[4] = {tc_off_b(n, r0), tc_off_b(n, r0 + 8), tc_off_b(n + 4, r0), tc_off_b(n + 4, r0 + 8)};
            uint32_t qh[4], ql[4], rh[4], rl[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              qh[e] = __float_as_uint(bh[oq[e]]);
              ql[e] = __float_as_uint(bl[oq[e]]);
              rh[e] = __float_as_uint(bh[oq[e] + 32 * NT]);
              rl[e] = __float_as_uint(bl[oq[e] + 32 * NT]);
            }
            mma_tf32(sa[rm], ql, hh[0], hh[1]);
            mma_tf32(sb[rm], rl, hh[0], hh[1]);
            mma_tf32(sa[rm], qh, hl[0], hl[1]);
            mma_tf32(sb[rm], rh, hl[0], hl[1]);
            mma_tf32(sa[rm], qh, hh[0], hh[1]);
            mma_tf32(sb[rm], rh, hh[0], hh[1]);
          }
        }
        const int FP = (F + 3) & ~3;
        float* outA = a.stats + size_t(blockIdx.x) * 2 * FP * KP;
        float* outB = outA + size_t(FP) * KP;
#pragma unroll
        for (int rm = 0; rm < 2; ++rm)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int row = 16 * rm + g + 8 * (e >> 1), k = 8 * warp + 2 * t + (e & 1);
            if (row < rows) {
              outA[size_t(k) * FP + c0 + row] = sa[rm][e];
              outB[size_t(k) * FP + c0 + row] = sb[rm][e];
            }
          }
      }
      if (c + 1 < nwin) {
        phase_a(c + 1);
        phase_a_epilogue(c + 1, want_div);  // the other Q/R buffer
      }
      if (!stats_pass) {
        mbar_wait(&mma_bar, mma_phase);  // window c's MMAs are done with its buffers
        mma_phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      if (c + 2 < nwin) make_lo(c + 2);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
    }
    if (!stats_pass) {
      // h update from TMEM: the M = 64 tile puts k = 16 q + j in lane 32 q + j; warps w and w+4
      // read quarter q = w & 3, frames split in halves (num at column n, den at NT + n)
      const int q = warp & 3, ch = warp >> 2;
      const int k = 16 * q + lane;
      const uint32_t tl = tmem + (uint32_t(32 * q) << 16);
      constexpr int NG = NT / 4;
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
        if (lane < 16) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = 4 * gi + e;
            if (n < nf && k < K) {
              float& h = Hs[n * KPS + k];
              h = h * sqrtf(__uint_as_float(vn[e]) / __uint_as_float(vd[e]));
              put_hfrag(Hhi, Hlo, hfrag_index<KB>(n, k), h);
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
    }
  }

  if (a.divpart && !bad) {
    double d = warp_sum_d(double(divacc));
    if (lane == 0) red[warp] = d;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kRsThreads / 32; ++w) s += red[w];
      a.divpart[blockIdx.x] = s;
    }
  }
  if (!bad && (a.Hout || a.write_store)) {
    for (int idx = tid; idx < nf * K; idx += kRsThreads) {
      const int n = idx / K, k = idx - n * K;
      const float h = Hs[n * KPS + k];
      if (a.Hout) a.Hout[size_t(n0 + n) * K + k] = h;
      if (a.write_store) {
        const int64_t col = a.widx ? int64_t(a.widx[n0 + n]) : (a.wbase + n0 + n) % a.wmod;
        a.U[size_t(col) * K + k] = h;
        if (k == 0) a.T[col] = a.c_now;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmemCols));
  if (bad && tid == 0) atomicOr(a.status, ST_NONPOS_INIT);
}

}  // namespace isnmf_dev

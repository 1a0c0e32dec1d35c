// K1L — fused mini-batch solve for large K (config 4: F=1025, K=256, 56 frames
// per CTA) on the tensor pipe.  Same contract as solve_kernel (SolveArgs;
// kernels.hpp:62-108, online.hpp:303-361); W (1 MB) does not fit shared memory,
// so it streams through a double-buffered 32-row window (cp.async from L2).
//
// Both contractions run as 3xTF32 mma.sync m16n8k8 (hi*hi + hi*lo + lo*hi, fp32
// accumulate; measured 4x the FP32 FMA rate per product on this part, so 1.33x
// the FMA peak at ~1e-6 relative error):
//   phase A  Lam^T[frame][row] = h^T W^T: tiles (16 frames x 8 rows), K = k;
//   phase B  [num|den][k][frame] += W^T [Q|R]: every warp owns 16*MBW values
//            of k for all frames and all rows, so num/den need no cross-warp
//            reduction (they stay in registers for the whole pass);
//   stats    [A|B]-partials[row][k] = [Q|R] h^T per 32-row chunk.
// hi = the raw fp32 bits (the tensor core reads the tf32 part), lo = x minus
// its tf32 truncation.
#pragma once

#include "kernels.cuh"

namespace isnmf_dev {

constexpr int kLgThreads = 256;  // 8 warps
constexpr int kLgChunk = 32;     // dictionary rows per window

template <int MBW, int NB>
struct LargeShape {
  static constexpr int KP = 128 * MBW;       // k padded: 8 warps x MBW m-blocks of 16
  static constexpr int NT = 8 * NB;          // frames per CTA (<= 64)
  static constexpr int KB = KP / 8;          // k blocks of 8 (phase A K dimension)
  static constexpr int FMB = (NT + 15) / 16; // frame blocks of 16 (phase A M dimension)
  static constexpr int TPW = (4 * FMB + 7) / 8;  // phase-A tiles per warp
  static constexpr int KPS = KP + 4;         // h row stride (= 4 mod 32: phase-A A loads conflict-free)
  static constexpr int WS = KP + 4;          // dictionary row stride (the global W32 layout)
  static constexpr int QRS = 136;            // staging row: q frames [0,64), r [64,128); = 8 mod 32
  static constexpr int HROWS = 16 * FMB;
  static constexpr size_t smem_bytes() {
    return sizeof(float) * (size_t(HROWS) * KPS + 3 * size_t(kLgChunk) * WS + 2 * size_t(kLgChunk) * QRS);
  }
};

__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(x);
  lo = __float_as_uint(x - __uint_as_float(hi & 0xffffe000u));
}

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

template <int MBW, int NB>
__global__ void __launch_bounds__(kLgThreads, 1) solve_large_kernel(const SolveArgs a) {
  using L = LargeShape<MBW, NB>;
  constexpr int KP = L::KP, NT = L::NT, KB = L::KB, FMB = L::FMB, TPW = L::TPW, KPS = L::KPS, WS = L::WS,
                QRS = L::QRS, HROWS = L::HROWS;
  pdl_wait();
  if (*a.status || (a.halt && *a.halt)) return;
  extern __shared__ __align__(16) float smem[];
  float* Hs = smem;                   // [HROWS][KPS], zero outside (n < nf, k < K)
  float* Wb = Hs + HROWS * KPS;        // [3][32][WS]: windows c, c+1 in use, c+2 loading
  float* QRb = Wb + 3 * kLgChunk * WS; // [2][32][QRS]: staging of windows c (phase B) and c+1 (phase A)
  __shared__ const float* fptr[64];
  __shared__ double red[kLgThreads / 32];
  __shared__ double meanv[64];
  __shared__ int s_bad;
  const int F = a.F, K = a.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int n0 = blockIdx.x * NT;
  const int nf = min(NT, a.nframes - n0);
  if (tid < 64) {
    const int64_t fr = tid < nf ? (a.vsel ? a.vsel[n0 + tid] : a.v0 + n0 + tid) : 0;
    fptr[tid] = a.V + fr * a.ldv;
  }
  if (tid == 0) s_bad = 0;
  for (int i = tid; i < HROWS * KPS; i += kLgThreads) Hs[i] = 0.0f;
  __syncthreads();
  if (a.h0_mode == 2) {  // mean of each frame in fp64 (fresh_h_init's v.mean())
    for (int n = warp; n < nf; n += kLgThreads / 32) {
      double s = 0.0;
      for (int f = lane; f < F; f += 32) s += double(fptr[n][f]);
      s = warp_sum_d(s);
      if (lane == 0) meanv[n] = s / double(F);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < nf * K; idx += kLgThreads) {  // h0
    const int n = idx / K, k = idx - n * K;
    int bad = 0;
    const int64_t col = a.h0_mode == 1 ? warm_col(a, n0 + n) : 0;
    const float val = solve_h0(a, n0 + n, k, col, a.h0_mode == 1 ? a.T[col] : 0u, a.h0_mode == 2 ? meanv[n] : 0.0, bad);
    if (a.check_h0 && bad) s_bad = 1;
    Hs[n * KPS + k] = val;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicOr(a.status, ST_NONPOS_INIT);
    return;
  }

  const float eps = a.eps;
  const int nch = (F + kLgChunk - 1) / kLgChunk;
  // dictionary window: rows [c0, c0+32) -> buffer; rows past F are zero (they meet zero q/r)
  auto load_w = [&](int c0, int buf) {
    const int rows = min(kLgChunk, F - c0);
    float* dst = Wb + buf * kLgChunk * WS;
    const float* src = a.W32 + size_t(c0) * WS;
    const int n4 = rows * WS / 4;
    for (int i = tid; i < n4; i += kLgThreads) cp_async16(dst + 4 * i, src + 4 * i);
    for (int i = n4 + tid; i < kLgChunk * WS / 4; i += kLgThreads)
      *reinterpret_cast<float4*>(dst + 4 * i) = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  float divacc = 0.0f;
  const int passes = a.iters + (a.do_stats ? 1 : 0);
  // phase-A tiles of this warp: tile i -> frame block i / 4, row block i % 4
  const int tile0 = warp * TPW;
      // ---------------- phase A of window c: Lam^T = h^T W^T for this warp's tiles, q / r staged
  auto phase_a = [&](int c, bool want_div) {
        const int c0 = c * kLgChunk, rows = min(kLgChunk, F - c0);
        const float* Wc = Wb + (c % 3) * kLgChunk * WS;
        float* QR = QRb + (c & 1) * kLgChunk * QRS;
        float acc[TPW][2][4];  // [tile][k-block parity][fragment]
#pragma unroll
        for (int i = 0; i < TPW; ++i)
#pragma unroll
          for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][p][e] = 0.0f;
        const int fmb = min(tile0, 4 * FMB - 1) / 4;  // the warp's tiles share one frame block
        // V of the outputs (L2 / HBM), in flight during the k loop
        float vv[TPW][4];
#pragma unroll
        for (int i = 0; i < TPW; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = 16 * fmb + g + 8 * (e >> 1), row = 8 * ((tile0 + i) & 3) + 2 * t + (e & 1);
            vv[i][e] = (tile0 + i < 4 * FMB && n < nf && row < rows) ? __ldg(fptr[n] + c0 + row) : 0.0f;
          }
        const float* hrow = Hs + (16 * fmb + g) * KPS + t;
#pragma unroll 1
        for (int kb = 0; kb < KB; kb += 2) {
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const float* hp = hrow + 8 * (kb + p);
            uint32_t ah[4], al[4];
            split_tf32(hp[0], ah[0], al[0]);
            split_tf32(hp[8 * KPS], ah[1], al[1]);
            split_tf32(hp[4], ah[2], al[2]);
            split_tf32(hp[8 * KPS + 4], ah[3], al[3]);
            uint32_t bh[TPW][2], bl[TPW][2];
#pragma unroll
            for (int i = 0; i < TPW; ++i) {
              const int rnb = (tile0 + i) & 3;
              const float* wp = Wc + (8 * rnb + g) * WS + 8 * (kb + p) + t;
              split_tf32(wp[0], bh[i][0], bl[i][0]);
              split_tf32(wp[4], bh[i][1], bl[i][1]);
            }
#pragma unroll
            for (int i = 0; i < TPW; ++i) mma_tf32(acc[i][p], al, bh[i][0], bh[i][1]);
#pragma unroll
            for (int i = 0; i < TPW; ++i) mma_tf32(acc[i][p], ah, bl[i][0], bl[i][1]);
#pragma unroll
            for (int i = 0; i < TPW; ++i) mma_tf32(acc[i][p], ah, bh[i][0], bh[i][1]);
          }
        }
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
          if (tile0 + i >= 4 * FMB) continue;
          const int rnb = (tile0 + i) & 3;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int n = 16 * fmb + g + 8 * (e >> 1), row = 8 * rnb + 2 * t + (e & 1);
            const bool valid = n < nf && row < rows;
            const float v = vv[i][e];
            const float r = rcp_approx(acc[i][0][e] + acc[i][1][e] + eps);
            const float vpe = v + eps;
            if (want_div && valid) divacc += is_term_ratio(vpe * r);
            QR[row * QRS + n] = valid ? vpe * r * r : 0.0f;
            QR[row * QRS + 64 + n] = valid ? r : 0.0f;
          }
        }
        };
  for (int pass = 0; pass < passes; ++pass) {
    const bool stats_pass = pass == a.iters;
    const bool want_div = a.div_first ? pass == 0 : stats_pass;
    if (stats_pass) pdl_trigger();  // K2 may launch onto SMs as CTAs finish
    float num[MBW][NB][4], den[MBW][NB][4];
#pragma unroll
    for (int mb = 0; mb < MBW; ++mb)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) num[mb][nb][e] = den[mb][nb][e] = 0.0f;
    // windows: c in W buffer c % 3 and staging c & 1; phase A of c+1 and phase B of c
    // run between the same two barriers
    load_w(0, 0);
    if (nch > 1) load_w(kLgChunk, 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    phase_a(0, want_div);
    for (int c = 0; c < nch; ++c) {
      const int c0 = c * kLgChunk, rows = min(kLgChunk, F - c0);
      const float* Wc = Wb + (c % 3) * kLgChunk * WS;
      const float* QR = QRb + (c & 1) * kLgChunk * QRS;
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();  // staging c complete, window c+1 visible, window c-1 and staging c+1 free
      if (c + 2 < nch) load_w(c0 + 2 * kLgChunk, (c + 2) % 3);
      if (c + 1 < nch) phase_a(c + 1, want_div);

      if (!stats_pass) {
        // ---------------- phase B: [num|den][k][n] += sum_rows W[row][k] [q|r][row][n]
#pragma unroll 1
        for (int kb = 0; kb < kLgChunk / 8; ++kb) {
          const float* wp = Wc + (8 * kb + t) * WS + g;
          const float* qp = QR + (8 * kb + t) * QRS + g;
          uint32_t qh[NB][2], ql[NB][2], rh[NB][2], rl[NB][2];
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            split_tf32(qp[8 * nb], qh[nb][0], ql[nb][0]);
            split_tf32(qp[4 * QRS + 8 * nb], qh[nb][1], ql[nb][1]);
            split_tf32(qp[64 + 8 * nb], rh[nb][0], rl[nb][0]);
            split_tf32(qp[4 * QRS + 64 + 8 * nb], rh[nb][1], rl[nb][1]);
          }
#pragma unroll
          for (int mb = 0; mb < MBW; ++mb) {
            const int km = 16 * (warp * MBW + mb);
            uint32_t ah[4], al[4];
            split_tf32(wp[km], ah[0], al[0]);
            split_tf32(wp[km + 8], ah[1], al[1]);
            split_tf32(wp[4 * WS + km], ah[2], al[2]);
            split_tf32(wp[4 * WS + km + 8], ah[3], al[3]);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              mma_tf32(num[mb][nb], al, qh[nb][0], qh[nb][1]);
              mma_tf32(den[mb][nb], al, rh[nb][0], rh[nb][1]);
            }
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              mma_tf32(num[mb][nb], ah, ql[nb][0], ql[nb][1]);
              mma_tf32(den[mb][nb], ah, rl[nb][0], rl[nb][1]);
            }
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
              mma_tf32(num[mb][nb], ah, qh[nb][0], qh[nb][1]);
              mma_tf32(den[mb][nb], ah, rh[nb][0], rh[nb][1]);
            }
          }
        }
      } else if (a.stats) {
        // ---------------- statistics of the window rows: [sa|sb][row][k] = sum_n [q|r][row][n] h[n][k]
        constexpr int KNW = 2 * MBW;  // k blocks of 8 per warp
        float sa[2][KNW][4], sb[2][KNW][4];
#pragma unroll
        for (int rm = 0; rm < 2; ++rm)
#pragma unroll
          for (int j = 0; j < KNW; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) sa[rm][j][e] = sb[rm][j][e] = 0.0f;
#pragma unroll 1
        for (int kb = 0; kb < NB; ++kb) {  // frames 8kb .. 8kb+7
          uint32_t hh[KNW][2], hl[KNW][2];
#pragma unroll
          for (int j = 0; j < KNW; ++j) {
            const float* hp = Hs + (8 * kb + t) * KPS + 8 * (warp * KNW + j) + g;
            split_tf32(hp[0], hh[j][0], hl[j][0]);
            split_tf32(hp[4 * KPS], hh[j][1], hl[j][1]);
          }
#pragma unroll
          for (int rm = 0; rm < 2; ++rm) {
            const float* qp = QR + (16 * rm + g) * QRS + 8 * kb + t;
            uint32_t qh[4], ql[4], rh[4], rl[4];
            split_tf32(qp[0], qh[0], ql[0]);
            split_tf32(qp[8 * QRS], qh[1], ql[1]);
            split_tf32(qp[4], qh[2], ql[2]);
            split_tf32(qp[8 * QRS + 4], qh[3], ql[3]);
            split_tf32(qp[64], rh[0], rl[0]);
            split_tf32(qp[8 * QRS + 64], rh[1], rl[1]);
            split_tf32(qp[68], rh[2], rl[2]);
            split_tf32(qp[8 * QRS + 68], rh[3], rl[3]);
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
      }
    }
    if (!stats_pass) {
      __syncthreads();  // every warp is done reading h in this pass
#pragma unroll
      for (int mb = 0; mb < MBW; ++mb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 16 * (warp * MBW + mb) + g + 8 * (e >> 1), n = 8 * nb + 2 * t + (e & 1);
            if (n < nf && k < K) {
              float& h = Hs[n * KPS + k];
              h = h * sqrtf(num[mb][nb][e] / den[mb][nb][e]);
            }
          }
    }
    __syncthreads();  // h updated; window buffer 0 free for the next pass
  }

  if (a.divpart) {
    double d = warp_sum_d(double(divacc));
    if (lane == 0) red[warp] = d;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kLgThreads / 32; ++w) s += red[w];
      a.divpart[blockIdx.x] = s;
    }
  }
  write_final_h(a, n0, nf, [&](int n, int k) { return Hs[n * KPS + k]; });
}

}  // namespace isnmf_dev

// K1M — fused mini-batch solve with every contraction on the tensor pipe, for
// K <= 8*KB (KB <= 7) and up to 16*FG frames per CTA (config 3: F=513, K=50,
// 28 frames per CTA).  Same contract as solve_kernel (SolveArgs; solve_h
// kernels.hpp:62-80, accumulate_sample_stats kernels.hpp:95-108, the
// divergence online.hpp:303-309).
//
// All products are 3xTF32 mma.sync m16n8k8 (lo*hi + hi*lo + hi*hi, fp32
// accumulate, ~1e-6 relative; hi = the raw fp32 bits, which the tensor core
// reads as tf32, lo = x minus its tf32 truncation).  mma.sync measured 8.0
// cycles per m16n8k8 per SM sub-partition with 2 warps x >= 2 chains
// (tools/probe/mma_probe2.cu), i.e. 1.33x the FP32 FMA peak per useful product
// and ~10x fewer issued instructions than FFMA register tiles, which is what
// bounded the FFMA kernel (issue-limited at ~55%).
//
// CTA: NW = 12 warps (8 when shared memory is short) = FG frame groups x RG row
// groups; W resident in shared memory (TMA bulk load, rows padded to 16 with zeros);
// h kept only as a pre-split fragment copy ([fm][kb][hi | lo][lane][4]).
//
// Iterations: warp (fm, rq) owns frames [16fm, 16fm+16) and the rq-th share of
// the dictionary rows in 8-row blocks; per chunk of up to 4 blocks
//   phase A  Lam^T[frame][row] = h^T W^T        (M = 16 frames, N = 8 rows, K = k)
//   q = (v+eps)/Lam^2, r = 1/Lam in registers  (Lam never leaves the registers)
//   phase B  [num|den]^T[frame][k] += [Q|R]^T W (M = 16 frames, N = 8 k, K = 8 rows)
// The C fragment of phase A (frame g / g+8, columns 2t, 2t+1) IS the A fragment
// of phase B once the 8 rows of a block are assigned to the k slots as
// slot t <-> column 2t, slot t+4 <-> column 2t+1, so q and r are never staged.
// Rows inside a block are permuted (column n of phase A is row rho(n),
// rho(g) = g ^ (g >> 2)) so that both phases' dictionary loads are free of
// bank conflicts with a row stride of 8 or 24 mod 32 words.  The RG warps of a
// frame group sum their num/den partials in a fixed order through shared memory
// (bitwise reproducible), then h *= sqrt(num/den); each group synchronises on its
// own named barrier, and every SM sub-partition hosts warps of both groups.
//
// Statistics pass (final h): warps own 16-row blocks and all frames,
//   Lam[row][frame] = W h                      (M = 16 rows, N = 8 frames, K = k)
//   [sa|sb][row][k] = [Q|R] h^T               (M = 16 rows, N = 8 k, K = 8 frames)
// with the same C -> A fragment identity (frame slots 2t, 2t+1), written
// straight to this CTA's statistics planes (no cross-warp reduction).
#pragma once

#include "kernels_large.cuh"

namespace isnmf_dev {


// smallest stride >= n (a multiple of 8) that is 8 or 24 mod 32 words: the
// 64-bit fragment loads of a half warp (8-word groups of 4 rows) hit 32 banks
__host__ __device__ constexpr int mm_stride(int n) {
  int s = (n + 7) & ~7;
  while (s % 32 != 8 && s % 32 != 24) s += 8;
  return s;
}

template <int KB, int FG, int NW>
struct MmShape {
  static constexpr int KP = 8 * KB;   // k padded to the MMA k-block
  static constexpr int NT = 16 * FG;  // frame capacity per CTA
  static constexpr int RG = NW / FG;  // row groups per frame group
  static constexpr int WS = mm_stride(KP);
  static constexpr int HT = mm_stride(NT);
  static constexpr int NREG = 8 * KB;         // num + den accumulator floats per lane
  static constexpr int HF = FG * KB * 32 * 8;  // h^T A fragments, [fm][kb][lane][hi 4 | lo 4]
  // num/den partials [NW][NREG][32] | h^T [KP][HT] (statistics pass)
  static constexpr int RED_FLOATS = NW * NREG * 32 > KP * HT ? NW * NREG * 32 : KP * HT;
  static constexpr int XR_FLOATS = 2 * 2 * 32 * KB * 8;  // K1P exchange [parity][rank][record][num 4 | den 4]
  static size_t smem_bytes(int F, bool pair2 = false) {
    const size_t F16 = size_t((F + 15) & ~15);
    return sizeof(float) * (F16 * WS + HF + RED_FLOATS + (pair2 ? XR_FLOATS : 0));
  }
};

__device__ __forceinline__ int mm_rho(int n) { return n ^ (n >> 2); }

// Timeline stamps of CTA 0 (ISNMF_PHASE_PROF builds): prof[warp * 64 + event] = clock64()
#ifdef ISNMF_PHASE_PROF
#define MM_STAMP(ev)                                                                     \
  do {                                                                                   \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && a.prof && (ev) < 64)                \
      a.prof[(threadIdx.x >> 5) * 64 + (ev)] = clock64();                                \
  } while (0)
#define MM_STAMP_P(prof, ev)                                                             \
  do {                                                                                   \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (prof) && (ev) < 64)                \
      (prof)[(threadIdx.x >> 5) * 64 + (ev)] = clock64();                                \
  } while (0)
#else
#define MM_STAMP(ev)
#define MM_STAMP_P(prof, ev)
#endif

// is_term (kernels.hpp:15-18) of ratio = (v+eps)/Lam as u - log(ratio) with the
// fast log: absolute error ~1e-7 per cell (the series of is_term_ratio only
// buys relative accuracy on terms that are themselves ~1e-7); used for the
// online objective of the statistics pass.  The batch objective of the incoming
// (W, H) (div_first) keeps the series of is_term_ratio (the fast form there makes
// ptxas spill at the 168-register cap of the 12-warp CTA)
__device__ __forceinline__ float is_term_fast(float ratio) {
  const float t = (ratio - 1.0f) - __logf(ratio);
  return t > 0.0f ? t : 0.0f;
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// barrier of one frame group's warps (named barrier 1 + fm; all warps when FG = 1)
template <int FG, int NW>
__device__ __forceinline__ void group_sync_t(int fm) {
  if constexpr (FG == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + fm), "r"(32 * NW / FG) : "memory");
  }
}

// position of h[n][k] in the fragment copy [fm][kb][hi | lo][lane][4]: lane (g, t)
// of block (fm, kb) holds a0 = (g, 2t), a1 = (g+8, 2t), a2 = (g, 2t+1),
// a3 = (g+8, 2t+1); the lo copy is 128 floats on (16-byte lane records,
// conflict-free LDS.128)
template <int KB>
__device__ __forceinline__ int hf_index(int n, int k) {
  ISNMF_DASSERT(k >= 0 && k < 8 * KB && n >= 0);
  const int fm = n >> 4, nn = n & 15, kb = k >> 3, kk = k & 7;
  const int ln = 4 * (nn & 7) + (kk >> 1), ai = (nn >> 3) + 2 * (kk & 1);
  return (fm * KB + kb) * 256 + ln * 4 + ai;
}
__device__ __forceinline__ void put_hf(float* p, float h) {
  uint32_t hi, lo;
  split_tf32(h, hi, lo);
  p[0] = __uint_as_float(hi);
  p[128] = __uint_as_float(lo);
}

__device__ __forceinline__ float2 lds64(const float* p) { return *reinterpret_cast<const float2*>(p); }
// K1M statistics planes: [window of 16 rows][sa | sb][K][16 rows], the rows of a [K][16] tile
// XOR-swizzled by k (2-way instead of 4-way bank conflicts when the C fragments are staged);
// K2 (fold_commit_kernel, stats_tiled = 2) reads float4 row quads of one k
__host__ __device__ __forceinline__ size_t mm_plane_floats(int F, int K) { return size_t((F + 15) >> 4) * 2 * K * 16; }
__host__ __device__ __forceinline__ int mm_plane_off(int k, int row16) { return k * 16 + (row16 ^ (((k >> 1) & 1) << 3)); }

// K1P exchange: st.async into the peer's shared memory with complete_tx on the peer's mbarrier
// (no cluster barrier in the pass loop: barrier.cluster costs ~380 cycles and its acquire
// invalidates L1, where the frames live; a release.cluster arrive costs a MEMBAR.ALL.GPU)
__device__ __forceinline__ void mm_bar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(uint32_t(__cvta_generic_to_shared(bar))), "r"(count));
}
__device__ __forceinline__ uint32_t mm_peer_addr(const void* p, unsigned rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(uint32_t(__cvta_generic_to_shared(p))), "r"(rank));
  return ra;
}
__device__ __forceinline__ void mm_st_async4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   raddr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mm_bar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(uint32_t(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mm_bar_wait(unsigned long long* bar, uint32_t parity) {
  const uint32_t b = uint32_t(__cvta_generic_to_shared(bar));
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
}

// One chunk of NBK 8-row blocks (rows row0 ...) of an iteration pass: phase A,
// q/r in registers, phase B into nd[0] (num^T) / nd[1] (den^T).
template <int KB, int WS, int NBK, bool DIV>
__device__ __forceinline__ void mm_chunk(const float* Ws, const float* pA, const float* pB, bool okA, bool okB,
                                         int row0, int F, float eps, const float* hf, float (&nd)[2][KB][4],
                                         int g, int t, float& divacc) {
  const int rg = mm_rho(g), rp = mm_rho(2 * t), rq = mm_rho(2 * t + 1);
  // V of this lane's cells: c0 (frame g, row rp), c1 (g, rq), c2 (g+8, rp), c3 (g+8, rq)
  float vv[NBK][4];
#pragma unroll
  for (int i = 0; i < NBK; ++i) {
    const int fp = row0 + 8 * i + rp, fq = row0 + 8 * i + rq;
    vv[i][0] = (okA && fp < F) ? __ldg(pA + fp) : 0.0f;
    vv[i][1] = (okA && fq < F) ? __ldg(pA + fq) : 0.0f;
    vv[i][2] = (okB && fp < F) ? __ldg(pB + fp) : 0.0f;
    vv[i][3] = (okB && fq < F) ? __ldg(pB + fq) : 0.0f;
  }
  // ---- phase A: Lam^T (16 frames x 8 rows per block), NBK independent chains
  float acc[NBK][4];
#pragma unroll
  for (int i = 0; i < NBK; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[i][c] = 0.0f;
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
    uint32_t ah[4], al[4];  // h^T A fragments (pre-split): a0 (g, slot t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4)
    {
      const float4 x = *reinterpret_cast<const float4*>(hf + kb * 256);
      const float4 y = *reinterpret_cast<const float4*>(hf + kb * 256 + 128);
      ah[0] = __float_as_uint(x.x);
      ah[1] = __float_as_uint(x.y);
      ah[2] = __float_as_uint(x.z);
      ah[3] = __float_as_uint(x.w);
      al[0] = __float_as_uint(y.x);
      al[1] = __float_as_uint(y.y);
      al[2] = __float_as_uint(y.z);
      al[3] = __float_as_uint(y.w);
    }
    uint32_t bh[NBK][2], bl[NBK][2];
#pragma unroll
    for (int i = 0; i < NBK; ++i) {
      const float2 w = lds64(Ws + (row0 + 8 * i + rg) * WS + 8 * kb + 2 * t);
      split_tf32(w.x, bh[i][0], bl[i][0]);
      split_tf32(w.y, bh[i][1], bl[i][1]);
    }
#pragma unroll
    for (int i = 0; i < NBK; ++i) mma_tf32(acc[i], al, bh[i][0], bh[i][1]);
#pragma unroll
    for (int i = 0; i < NBK; ++i) mma_tf32(acc[i], ah, bl[i][0], bl[i][1]);
#pragma unroll
    for (int i = 0; i < NBK; ++i) mma_tf32(acc[i], ah, bh[i][0], bh[i][1]);
  }
  // ---- q = (v+eps)/Lam^2, r = 1/Lam (zero outside the valid frames / rows)
  float q[NBK][4], r[NBK][4];
#pragma unroll
  for (int i = 0; i < NBK; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int f = row0 + 8 * i + ((c & 1) ? rq : rp);
      const bool valid = ((c < 2) ? okA : okB) && f < F;
      const float rr = rcp_approx(acc[i][c] + eps);
      const float ve = vv[i][c] + eps;
      q[i][c] = valid ? ve * rr * rr : 0.0f;
      r[i][c] = valid ? rr : 0.0f;
      if constexpr (DIV) divacc += valid ? is_term_ratio(ve * rr) : 0.0f;
    }
  // ---- phase B: per block, K = its 8 rows (slot t <-> c0/c2, slot t+4 <-> c1/c3);
  // the dictionary values of block i+1 are loaded while block i's MMAs issue
  float wv[KB][2];
  auto load_wb = [&](int i) {
    const float* wp = Ws + (row0 + 8 * i + rp) * WS + g;
    const float* wq = Ws + (row0 + 8 * i + rq) * WS + g;
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      wv[j][0] = wp[8 * j];
      wv[j][1] = wq[8 * j];
    }
  };
  load_wb(0);
#pragma unroll
  for (int i = 0; i < NBK; ++i) {
    uint32_t qh[4], ql[4], rh[4], rl[4];
    split_tf32(q[i][0], qh[0], ql[0]);
    split_tf32(q[i][2], qh[1], ql[1]);
    split_tf32(q[i][1], qh[2], ql[2]);
    split_tf32(q[i][3], qh[3], ql[3]);
    split_tf32(r[i][0], rh[0], rl[0]);
    split_tf32(r[i][2], rh[1], rl[1]);
    split_tf32(r[i][1], rh[2], rl[2]);
    split_tf32(r[i][3], rh[3], rl[3]);
    uint32_t bh[KB][2], bl[KB][2];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      split_tf32(wv[j][0], bh[j][0], bl[j][0]);
      split_tf32(wv[j][1], bh[j][1], bl[j][1]);
    }
    if (i + 1 < NBK) load_wb(i + 1);
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      mma_tf32(nd[0][j], ql, bh[j][0], bh[j][1]);
      mma_tf32(nd[1][j], rl, bh[j][0], bh[j][1]);
    }
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      mma_tf32(nd[0][j], qh, bl[j][0], bl[j][1]);
      mma_tf32(nd[1][j], rh, bl[j][0], bl[j][1]);
    }
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      mma_tf32(nd[0][j], qh, bh[j][0], bh[j][1]);
      mma_tf32(nd[1][j], rh, bh[j][0], bh[j][1]);
    }
  }
}

// One 16-row block of the statistics pass: Lam = W h, q/r (+ divergence), and
// the block's rows of the statistics planes.
// V of a statistics block's cells: c0 (row g, frame 8nb+2t), c1 (g, 2t+1), c2 (g+8, 2t), c3 (g+8, 2t+1)
template <int NB>
__device__ __forceinline__ void mm_stats_v(float (&vv)[NB][4], const float* const* fptr, int f0, int F, int nf,
                                           int g, int t) {
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    const int na = 8 * nb + 2 * t, nbb = na + 1;
    const bool ra = f0 + g < F, rb = f0 + g + 8 < F;
    vv[nb][0] = (na < nf && ra) ? __ldg(fptr[na] + f0 + g) : 0.0f;
    vv[nb][1] = (nbb < nf && ra) ? __ldg(fptr[nbb] + f0 + g) : 0.0f;
    vv[nb][2] = (na < nf && rb) ? __ldg(fptr[na] + f0 + g + 8) : 0.0f;
    vv[nb][3] = (nbb < nf && rb) ? __ldg(fptr[nbb] + f0 + g + 8) : 0.0f;
  }
}

template <int KB, int FG, int WS, int HT>
__device__ __forceinline__ void mm_stats_block(const float* Ws, const float* Hf, const float* Ht,
                                               const float* const* fptr, int f0, int F, int nf, float eps, int g,
                                               int t, bool want_div, float& divacc, float* outA, float* outB, int FP,
                                               float (&vv)[2 * FG][4], int f0n, long long* prof, int ev,
                                               bool accumulate, int K, float* stg, bool first_block) {
  constexpr int NB = 2 * FG;  // frame blocks of 8
  MM_STAMP_P(prof, ev);
  float acc[NB][4];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[nb][c] = 0.0f;
#pragma unroll
  for (int kb = 0; kb < KB; ++kb) {
    const float2 x = lds64(Ws + (f0 + g) * WS + 8 * kb + 2 * t);
    const float2 y = lds64(Ws + (f0 + g + 8) * WS + 8 * kb + 2 * t);
    uint32_t wh[4], wl[4];
    split_tf32(x.x, wh[0], wl[0]);
    split_tf32(y.x, wh[1], wl[1]);
    split_tf32(x.y, wh[2], wl[2]);
    split_tf32(y.y, wh[3], wl[3]);
    // h (k 8kb+2t, 2t+1) of frames 8nb+g from the pre-split fragment records:
    // frame block 2fm is (a0, a2) of record (fm, kb, lane), block 2fm+1 is (a1, a3)
    uint32_t hh[NB][2], hl[NB][2];
#pragma unroll
    for (int fm = 0; fm < FG; ++fm) {
      const float* rec = Hf + (fm * KB + kb) * 256 + (4 * g + t) * 4;
      const float4 x = *reinterpret_cast<const float4*>(rec);
      const float4 y = *reinterpret_cast<const float4*>(rec + 128);
      hh[2 * fm][0] = __float_as_uint(x.x);
      hh[2 * fm][1] = __float_as_uint(x.z);
      hh[2 * fm + 1][0] = __float_as_uint(x.y);
      hh[2 * fm + 1][1] = __float_as_uint(x.w);
      hl[2 * fm][0] = __float_as_uint(y.x);
      hl[2 * fm][1] = __float_as_uint(y.z);
      hl[2 * fm + 1][0] = __float_as_uint(y.y);
      hl[2 * fm + 1][1] = __float_as_uint(y.w);
    }
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) mma_tf32(acc[nb], wl, hh[nb][0], hh[nb][1]);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) mma_tf32(acc[nb], wh, hl[nb][0], hl[nb][1]);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) mma_tf32(acc[nb], wh, hh[nb][0], hh[nb][1]);
  }
  MM_STAMP_P(prof, ev + 1);
  float q[NB][4], r[NB][4];
#pragma unroll
  for (int nb = 0; nb < NB; ++nb)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int n = 8 * nb + 2 * t + (c & 1), f = f0 + g + 8 * (c >> 1);
      const float vc = vv[nb][c];
      const bool valid = n < nf && f < F;
      const float rr = rcp_approx(acc[nb][c] + eps);
      const float ve = vc + eps;
      q[nb][c] = valid ? ve * rr * rr : 0.0f;
      r[nb][c] = valid ? rr : 0.0f;
      if (want_div) divacc += valid ? is_term_fast(ve * rr) : 0.0f;
    }
  if (f0n >= 0) mm_stats_v<NB>(vv, fptr, f0n, F, nf, g, t);  // the next block's V, behind the MMAs below
  MM_STAMP_P(prof, ev + 2);
  if (!outA) return;
  float sa[KB][4], sb[KB][4];
#pragma unroll
  for (int j = 0; j < KB; ++j)
#pragma unroll
    for (int c = 0; c < 4; ++c) sa[j][c] = sb[j][c] = 0.0f;
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    uint32_t qh[4], ql[4], rh[4], rl[4];
    split_tf32(q[nb][0], qh[0], ql[0]);
    split_tf32(q[nb][2], qh[1], ql[1]);
    split_tf32(q[nb][1], qh[2], ql[2]);
    split_tf32(q[nb][3], qh[3], ql[3]);
    split_tf32(r[nb][0], rh[0], rl[0]);
    split_tf32(r[nb][2], rh[1], rl[1]);
    split_tf32(r[nb][1], rh[2], rl[2]);
    split_tf32(r[nb][3], rh[3], rl[3]);
    uint32_t bh[KB][2], bl[KB][2];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const float2 h = lds64(Ht + (8 * j + g) * HT + 8 * nb + 2 * t);
      split_tf32(h.x, bh[j][0], bl[j][0]);
      split_tf32(h.y, bh[j][1], bl[j][1]);
    }
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      mma_tf32(sa[j], ql, bh[j][0], bh[j][1]);
      mma_tf32(sb[j], rl, bh[j][0], bh[j][1]);
    }
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      mma_tf32(sa[j], qh, bl[j][0], bl[j][1]);
      mma_tf32(sb[j], rh, bl[j][0], bl[j][1]);
    }
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      mma_tf32(sa[j], qh, bh[j][0], bh[j][1]);
      mma_tf32(sb[j], rh, bh[j][0], bh[j][1]);
    }
  }
  MM_STAMP_P(prof, ev + 3);
#ifdef ISNMF_SKIP_STATS_STORE  // timing-only builds: the cost of the plane stores / reductions
  if (sa[0][0] != 12345.678f) return;
#endif
  // The block's [sa | sb] leave as two TMA bulk copies of one [K][16 rows] tile each (plane
  // layout mm_plane_off below): 56 scattered 4-byte stores / reductions per lane cost ~4.5k
  // cycles per block at config 2 (one 32-byte sector request each), a bulk copy moves whole
  // lines.  The warp's staging tile is reused for sa, then sb: its previous copy must have
  // read it (wait_group.read).  A CTA that owns several frame tiles (batch) adds into its
  // plane with cp.reduce.async.bulk add.f32 after the first; every cell has one issuing
  // thread (lane 0 of the warp that owns the block in every tile) and that thread waits for
  // its previous tile's copies to complete before the first of this tile (first_block), so
  // the sums are formed in tile order: deterministic, bitwise reproducible.
  const int K16 = K * 16;
  float* gA = outA + size_t(f0 >> 4) * 2 * K16;  // outA = the plane; the window's sa tile, sb behind it
#pragma unroll
  for (int ab = 0; ab < 2; ++ab) {
    if ((g | t) == 0) {
      if (ab == 0 && first_block)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      else
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      const int k0 = 8 * j + 2 * t, sw = (t & 1) << 3;  // ((k >> 1) & 1) << 3 for k0 and k0 + 1
      const float(&v)[4] = ab ? sb[j] : sa[j];
      if (k0 < K) {
        stg[k0 * 16 + (g ^ sw)] = v[0];
        stg[k0 * 16 + ((g + 8) ^ sw)] = v[2];
      }
      if (k0 + 1 < K) {
        stg[(k0 + 1) * 16 + (g ^ sw)] = v[1];
        stg[(k0 + 1) * 16 + ((g + 8) ^ sw)] = v[3];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if ((g | t) == 0) {
      const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(stg));
      float* dst = gA + ab * K16;
      const uint32_t bytes = uint32_t(K16) * 4u;
      if (accumulate)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst), "r"(src),
                     "r"(bytes)
                     : "memory");
      else
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
}

// MULTI = false: one frame tile per CTA (online mini-batches: grid = tiles); true: CTAs
// loop over several tiles (batch), accumulating their statistics planes and staging the
// next tile — a separate instantiation, so the online kernel keeps its register budget
template <int KB, int FG, int NW, bool MULTI>
__global__ void __launch_bounds__(32 * NW, 1) solve_mma_kernel(const SolveArgs a) {
  using S = MmShape<KB, FG, NW>;
  constexpr int KP = S::KP, NT = S::NT, RG = S::RG, WS = S::WS, HT = S::HT, NREG = S::NREG;
  constexpr int kMmThreads = 32 * NW;
  MM_STAMP(62);
  if constexpr (!MULTI && FG == 1)
    if (a.pair2) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // (waited below)
  if constexpr (!MULTI) {  // warm-store lines of this CTA's frames towards L2, beside the previous K2
    if (a.h0_mode == 1) {
      const int t0 = (FG == 1 && a.pair2) ? int(blockIdx.x >> 1) : int(blockIdx.x);
      const int nfr = min(a.cta_frames, a.nframes - t0 * a.cta_frames);
      if (int(threadIdx.x) < nfr) warm_prefetch(a, t0 * a.cta_frames + int(threadIdx.x));
    }
  }
  pdl_wait();
  MM_STAMP(58);
  // K1P (a.pair2; online, one frame group): a 2-CTA cluster shares the tile's frames, rank r
  // owning the rows of 16-row blocks [r * S16, ...) — the num/den partials of the two row halves
  // are exchanged through distributed shared memory once per pass, so both CTAs apply the same
  // fixed-order update (rank 0 + rank 1) and hold the same h
  constexpr bool kCanPair = !MULTI && FG == 1;
  const bool pair2 = kCanPair && a.pair2 != 0;
  const unsigned crank = pair2 ? cluster_rank() : 0u;
  // K1P: xbar[pass & 1] = the peer's row-half sums of that pass have landed in XR (transaction
  // bytes of its st.async stores; a barrier is reused two passes later, behind our own next send)
  __shared__ __align__(8) unsigned long long xbar[2];
  if constexpr (kCanPair) {
    if (pair2) {  // both CTAs take the same go decision (a status bit set meanwhile must not split them)
      __shared__ int s_go2[2];
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // the peer has started
      if (threadIdx.x == 0) {
        mm_bar_init(&xbar[0], 1);
        mm_bar_init(&xbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
        const int go = !(*a.status || (a.halt && *a.halt));
        s_go2[crank] = go;
        *const_cast<int*>(map_rank(&s_go2[crank], crank ^ 1u)) = go;
      }
      cluster_sync_all();
      if (!(s_go2[0] && s_go2[1])) return;
    } else if (*a.status || (a.halt && *a.halt)) {
      return;
    }
  } else {
    if (*a.status || (a.halt && *a.halt)) return;
  }

  extern __shared__ __align__(16) float smem[];
  const int F = a.F, K = a.K;
  const int F16 = (F + 15) & ~15;
  float* Ws = smem;           // [F16][WS], rows >= F zero
  // h lives only as its pre-split fragment copy (hi = the raw fp32 value), zero
  // outside n < nf, k < K: [FG][KB][hi | lo][32 lanes][4]
  float* Hf = Ws + F16 * WS;
  float* RED = Hf + S::HF;    // [NW][NREG][32] num/den partials | Ht [KP][HT] (statistics pass)
  __shared__ const float* fptr[NT];
  __shared__ double red[kMmThreads / 32];
  __shared__ double meanv[NT];
  __shared__ int64_t colv[NT];  // warm store column of each frame
  __shared__ uint32_t tagv[NT];  // and its commit tag
  __shared__ int s_bad;
  __shared__ __align__(8) unsigned long long wbar;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int ntc = a.cta_frames;
  // frame tiles of ntc frames; CTA b owns tiles b, b + gridDim.x, ... (one tile per CTA
  // for an online mini-batch; the batch path runs one CTA per SM over all N frames, so
  // the dictionary is loaded once per CTA and the statistics planes accumulate in place)
  const int tile0 = pair2 ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int ntiles = MULTI ? (a.nframes + ntc - 1) / ntc : tile0 + 1;

  if (tid == 0) {  // dictionary -> smem by TMA bulk copies, overlapped with the h0 set-up below
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&wbar));
    const uint32_t bytes = uint32_t(F) * WS * 4u;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes));
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(Ws));
    constexpr uint32_t kPiece = 32768;
    for (uint32_t off = 0; off < bytes; off += kPiece) {
      const uint32_t n = bytes - off < kPiece ? bytes - off : kPiece;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       dst + off),
                   "l"(reinterpret_cast<const char*>(a.W32) + off), "r"(n), "r"(bar)
                   : "memory");
    }
  }
  for (int i = tid; i < (F16 - F) * WS; i += kMmThreads) Ws[F * WS + i] = 0.0f;  // pad rows
  double divd = 0.0;  // this lane's divergence over the CTA's tiles
  // multi-tile CTAs with direct h0 (batch): the next tile's H0 rows are staged into
  // shared memory by cp.async and its frames prefetched into L2 during this tile's
  // statistics pass (RED beyond Ht is free then)
  // (every tile but the last stages its successor, so tile i > 0 finds its H0 staged)
  const bool stage_next = MULTI && a.h0_mode == 0 && !a.vsel && int(gridDim.x) < ntiles;
  float* Hstage = RED + ((KP * HT + 31) & ~31);
  for (int tile = tile0; tile < ntiles; tile += gridDim.x) {
  const bool first_tile = !MULTI || tile == int(blockIdx.x);
  MM_STAMP(59);
  const bool staged = stage_next && !first_tile;
  const int n0 = tile * ntc;
  const int nf = min(ntc, a.nframes - n0);
  if (!first_tile) {
    if (staged) cp_async_wait_all();
    __syncthreads();  // the previous tile's readers of fptr / Hf / Ht are done, the staged H0 landed
  }
  if (tid < NT) {
    const int64_t fr = tid < nf ? (a.vsel ? a.vsel[n0 + tid] : a.v0 + n0 + tid) : 0;
    fptr[tid] = a.V + fr * a.ldv;
    if (a.h0_mode == 1 && tid < nf) {  // per-frame warm-store column and tag, off the per-element chain
      const int64_t col = warm_col(a, n0 + tid);
      colv[tid] = col;
      tagv[tid] = a.T[col];
    }
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();

  if (a.h0_mode == 2) {  // mean of each frame in fp64 (fresh_h_init's v.mean())
    for (int n = warp; n < nf; n += kMmThreads / 32) {
      double s = 0.0;
      for (int f = lane; f < F; f += 32) s += double(fptr[n][f]);
      s = warp_sum_d(s);
      if (lane == 0) meanv[n] = s / double(F);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < NT * KP; idx += kMmThreads) {
    const int n = idx / KP, k = idx - n * KP;
    float val = 0.0f;
    if (n < nf && k < K) {
      int bad = 0;
      val = a.h0_mode == 1 ? solve_h0(a, n0 + n, k, colv[n], tagv[n], 0.0, bad)
            : staged       ? scaled_h0(a, Hstage[n * K + k], k, bad)
                           : solve_h0(a, n0 + n, k, 0, 0u, a.h0_mode == 2 ? meanv[n] : 0.0, bad);
      if (a.check_h0 && bad) s_bad = 1;
    }
    put_hf(Hf + hf_index<KB>(n, k), val);
  }
  if (first_tile) {  // wait for the dictionary (phase 0 of wbar)
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&wbar));
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
          : "=r"(done)
          : "r"(bar)
          : "memory");
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicOr(a.status, ST_NONPOS_INIT);
    return;
  }

  MM_STAMP(0);
  const float eps = a.eps;
  float divacc = 0.0f;
  auto group_sync = [](int fm) { group_sync_t<FG, NW>(fm); };
  // iteration passes: warp = RG * fm + rq, so every SM sub-partition (warp % 4)
  // hosts one warp of each frame group; the groups synchronise on their own
  // named barrier, so one group's reduction/update overlaps the other's MMAs.
  // Frame group 1 visits the row groups in reverse: an uneven block split puts
  // its extra block on a different sub-partition than group 0's.
  const int fm = warp / RG, rq = warp % RG;
  const int rgi = (FG == 2 && fm == 1) ? RG - 1 - rq : rq;
  const int NBLK = (F + 7) >> 3;
  // rows of this CTA: all, or (K1P) 16-row blocks [M0, M1) = 8-row blocks [B0, B1)
  const int NB16 = F16 / 16, S16 = (NB16 + 1) / 2;
  const int M0 = pair2 ? int(crank) * S16 : 0, M1 = pair2 ? (crank ? NB16 : S16) : NB16;
  const int B0 = 2 * M0, B1 = pair2 ? min(NBLK, 2 * M1) : NBLK, NBL = B1 - B0;
  const int blk0 = B0 + rgi * NBL / RG, blk1 = B0 + (rgi + 1) * NBL / RG;
  const int nA = 16 * fm + g, nB = nA + 8;
  const bool okA = nA < nf, okB = nB < nf;
  const float* pA = fptr[nA];
  const float* pB = fptr[nB];

  for (int pass = 0; pass < a.iters; ++pass) {
    const float* hf = Hf + fm * KB * 256 + lane * 4;
    float nd[2][KB][4];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int j = 0; j < KB; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) nd[x][j][c] = 0.0f;
    // chunks of 4 blocks (4 independent phase-A chains); DIV: the batch objective of the
    // incoming (W, H) from this pass's Lam (div_first, pass 0)
    auto chunks = [&](auto div) {
      constexpr bool DIV = decltype(div)::value;
      int cb = blk0;
#pragma unroll 1
      for (; cb + 4 <= blk1; cb += 4)
        mm_chunk<KB, WS, 4, DIV>(Ws, pA, pB, okA, okB, 8 * cb, F, eps, hf, nd, g, t, divacc);
      switch (blk1 - cb) {
        case 3: mm_chunk<KB, WS, 3, DIV>(Ws, pA, pB, okA, okB, 8 * cb, F, eps, hf, nd, g, t, divacc); break;
        case 2: mm_chunk<KB, WS, 2, DIV>(Ws, pA, pB, okA, okB, 8 * cb, F, eps, hf, nd, g, t, divacc); break;
        case 1: mm_chunk<KB, WS, 1, DIV>(Ws, pA, pB, okA, okB, 8 * cb, F, eps, hf, nd, g, t, divacc); break;
        default: break;
      }
    };
    if (a.div_first && pass == 0)
      chunks(std::true_type{});
    else
      chunks(std::false_type{});
    MM_STAMP(1 + 4 * pass);
    {  // partials -> shared memory as [warp][num|den][jb][lane][4] (16-byte lane records)
      float* rw = RED + warp * NREG * 32 + lane * 4;
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int j = 0; j < KB; ++j)
          *reinterpret_cast<float4*>(rw + (x * KB + j) * 128) = make_float4(nd[x][j][0], nd[x][j][1], nd[x][j][2],
                                                                            nd[x][j][3]);
    }
    group_sync(fm);
    MM_STAMP(2 + 4 * pass);
    // fixed-order sum over the RG row groups, h *= sqrt(num/den) (kernels.hpp:77); one
    // thread per (k block, lane) record = 4 cells, h read from / written to the fragment copy
    constexpr int RECS = 32 * KB;  // per frame group, over its RG * 32 threads
    const int gt = tid - fm * RG * 32;
    auto rec_sum = [&](int p, float4& num, float4& den) {
      const int ln = p & 31, jb = p >> 5;
      num = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      den = num;
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const float* src = RED + (fm * RG + r) * NREG * 32 + jb * 128 + ln * 4;
        const float4 x = *reinterpret_cast<const float4*>(src);
        const float4 y = *reinterpret_cast<const float4*>(src + KB * 128);
        num.x += x.x;
        num.y += x.y;
        num.z += x.z;
        num.w += x.w;
        den.x += y.x;
        den.y += y.y;
        den.z += y.z;
        den.w += y.w;
      }
    };
    auto rec_update = [&](int p, const float4& num, const float4& den) {
      const int ln = p & 31, jb = p >> 5;
      // C order (c0 (g, 2t), c1 (g, 2t+1), c2 (g+8, 2t), c3 (g+8, 2t+1)) -> record order a0 a2 a1 a3
      float* rec = Hf + (fm * KB + jb) * 256 + ln * 4;
      float4 h = *reinterpret_cast<const float4*>(rec);
      const int n0c = 16 * fm + (ln >> 2), k0c = 8 * jb + 2 * (ln & 3);
      const bool v0 = n0c < nf, v1 = n0c + 8 < nf, e0 = k0c < K, e1 = k0c + 1 < K;
      h.x = (v0 && e0) ? h.x * sqrt_approx(num.x * rcp_approx(den.x)) : h.x;
      h.z = (v0 && e1) ? h.z * sqrt_approx(num.y * rcp_approx(den.y)) : h.z;
      h.y = (v1 && e0) ? h.y * sqrt_approx(num.z * rcp_approx(den.z)) : h.y;
      h.w = (v1 && e1) ? h.w * sqrt_approx(num.w * rcp_approx(den.w)) : h.w;
      uint32_t hi, lo[4];
      split_tf32(h.x, hi, lo[0]);
      split_tf32(h.y, hi, lo[1]);
      split_tf32(h.z, hi, lo[2]);
      split_tf32(h.w, hi, lo[3]);
      *reinterpret_cast<float4*>(rec) = h;
      *reinterpret_cast<float4*>(rec + 128) = make_float4(__uint_as_float(lo[0]), __uint_as_float(lo[1]),
                                                          __uint_as_float(lo[2]), __uint_as_float(lo[3]));
    };
    // fixed-order sum over the RG row groups, h *= sqrt(num/den) (kernels.hpp:77); one
    // thread per (k block, lane) record = 4 cells, h read from / written to the fragment copy
    if (!pair2) {
#pragma unroll
      for (int m = 0; m < (RECS + RG * 32 - 1) / (RG * 32); ++m) {
        const int p = gt + m * RG * 32;
        if (p < RECS) {
          float4 num, den;
          rec_sum(p, num, den);
          rec_update(p, num, den);
        }
      }
    } else if constexpr (kCanPair) {
      // K1P: this CTA's row-half sums -> XR[pass & 1][rank] here and in the peer (st.async over
      // DSMEM, completing transaction bytes on the peer's xbar[pass & 1]); the thread that owns
      // record p waits for the peer's records, then rank 0 + rank 1 in that order in both CTAs.
      // Double-buffered by pass parity: the peer writes a buffer again two passes later, after
      // every record of our pass between has reached it, each sent after its thread's reads here.
      float4* XR = reinterpret_cast<float4*>(RED + S::RED_FLOATS) + (pass & 1) * 2 * 2 * RECS;
      if (gt == 0) mm_bar_expect_tx(&xbar[pass & 1], uint32_t(RECS * 2 * sizeof(float4)));
      const uint32_t rbar = mm_peer_addr(&xbar[pass & 1], crank ^ 1u);
#pragma unroll
      for (int m = 0; m < (RECS + RG * 32 - 1) / (RG * 32); ++m) {
        const int p = gt + m * RG * 32;
        if (p < RECS) {
          float4 num, den;
          rec_sum(p, num, den);
          float4* own = XR + (crank * RECS + p) * 2;
          const uint32_t far = mm_peer_addr(own, crank ^ 1u);
          mm_st_async4(far, num, rbar);
          mm_st_async4(far + 16, den, rbar);
          own[0] = num;
          own[1] = den;
        }
      }
      if (gt < RECS) mm_bar_wait(&xbar[pass & 1], uint32_t(pass >> 1) & 1u);
#pragma unroll
      for (int m = 0; m < (RECS + RG * 32 - 1) / (RG * 32); ++m) {
        const int p = gt + m * RG * 32;
        if (p < RECS) {
          const float4 n0v = XR[p * 2], d0v = XR[p * 2 + 1];
          const float4 n1v = XR[(RECS + p) * 2], d1v = XR[(RECS + p) * 2 + 1];
          rec_update(p, make_float4(n0v.x + n1v.x, n0v.y + n1v.y, n0v.z + n1v.z, n0v.w + n1v.w),
                     make_float4(d0v.x + d1v.x, d0v.y + d1v.y, d0v.z + d1v.z, d0v.w + d1v.w));
        }
      }
    }
    MM_STAMP(3 + 4 * pass);
    group_sync(fm);
    MM_STAMP(4 + 4 * pass);
  }
  __syncthreads();
  MM_STAMP(60);
  float* Ht = RED;  // [KP][HT] = h^T, B operand of the statistics contraction (RED is free now)

  if (a.do_stats) {
    pdl_trigger();  // K2 may launch onto SMs as CTAs finish
    const bool want_div = !a.div_first || a.iters == 0;
    for (int idx = tid; idx < KP * NT; idx += kMmThreads) {
      const int k = idx / NT, n = idx - k * NT;
      Ht[k * HT + n] = Hf[hf_index<KB>(n, k)];
    }
    if (stage_next && tile + int(gridDim.x) < ntiles) {
      const int n1 = (tile + int(gridDim.x)) * ntc, nf1 = min(ntc, a.nframes - n1);
      const float* src = a.H0 + size_t(n1) * K;
      for (int i = tid; i < nf1 * K; i += kMmThreads) cp_async4(Hstage + i, src + i);
      asm volatile("cp.async.commit_group;" ::: "memory");
      const char* v1 = reinterpret_cast<const char*>(a.V + (a.v0 + n1) * a.ldv);
      const size_t vbytes = size_t(nf1) * a.ldv * sizeof(float);
      for (size_t off = size_t(tid) * 128; off < vbytes; off += size_t(kMmThreads) * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(v1 + off));
    }
    __syncthreads();
    // (K1P: the pair's plane, this CTA's rows)
    ISNMF_DASSERT(!a.stats || a.stats_cap == 0 || (pair2 ? tile : int(blockIdx.x)) < a.stats_cap);
    float* plane = a.stats ? a.stats + size_t(pair2 ? tile : int(blockIdx.x)) * mm_plane_floats(F, K) : nullptr;
    // this warp's staging tile [K][16] (behind h^T and the next tile's staged H0 in RED)
    float* stg = Hstage + ((NT * KP + 31) & ~31) + warp * 16 * KP;
    float vv[2 * FG][4];
    if (M0 + warp < M1) mm_stats_v<2 * FG>(vv, fptr, 16 * (M0 + warp), F, nf, g, t);
#pragma unroll 1
    for (int m = M0 + warp; m < M1; m += kMmThreads / 32) {
      const int mn = m + kMmThreads / 32;
      mm_stats_block<KB, FG, WS, HT>(Ws, Hf, Ht, fptr, 16 * m, F, nf, eps, g, t, want_div, divacc, plane, plane,
                                         0, vv, mn < M1 ? 16 * mn : -1, a.prof,
                                         44 + 4 * ((m - M0 - warp) / (kMmThreads / 32)), !first_tile, K, stg,
                                         m == M0 + warp);
    }
    // the staging tiles lie in RED: the copies must have read them before the next tile's
    // partials (or the CTA's exit) — and have completed before the grid ends
    if (plane && lane == 0) {
      if (MULTI && tile + int(gridDim.x) < ntiles)
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      else
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  divd += double(divacc);

  if (!pair2) {
    write_final_h(a, n0, nf, [&](int n, int k) { return Hf[hf_index<KB>(n, k)]; });
  } else {  // K1P: both CTAs hold every frame's h; each writes half of the frames
    const int half = (nf + 1) / 2, f0 = crank ? half : 0, fc = crank ? nf - half : half;
    write_final_h(a, n0 + f0, fc, [&](int n, int k) { return Hf[hf_index<KB>(f0 + n, k)]; });
  }
  }  // tiles

  MM_STAMP(61);
  // divergence partial of this CTA (fixed-order reduction)
  if (a.divpart) {
    ISNMF_DASSERT(a.stats_cap == 0 || int(blockIdx.x) < (pair2 ? 2 : 1) * a.stats_cap);  // divpart: 2 x planes
    const double d = warp_sum_d(divd);
    if (lane == 0) red[warp] = d;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kMmThreads / 32; ++w) s += red[w];
      a.divpart[blockIdx.x] = s;  // (K1P: two partials per pair, 2 * pair + rank)
    }
  }
  if constexpr (kCanPair)
    if (pair2) cluster_sync_all();  // no DSMEM access may reach an exited CTA

  MM_STAMP(63);
}

}  // namespace isnmf_dev

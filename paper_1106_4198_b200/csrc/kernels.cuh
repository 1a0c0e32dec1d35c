// Device kernels of the B200 online / batch IS-NMF engine (sm_100a).
//
// K1  solve_kernel   — fused mini-batch H solver (kernels.hpp:62-80) with the
//                      statistics epilogue (kernels.hpp:95-108, online.hpp:360-361)
//                      and the IS-divergence of the final fit (online.hpp:303-309).
// K2  fold_commit_kernel — deterministic fixed-order reduction of the per-CTA
//                      A/B partials into pending (online.hpp:360-361) and, at a
//                      mini-batch boundary, dictionary_commit (online.hpp:319-336:
//                      update_w kernels.hpp:142-159, l1 renormalisation
//                      model.hpp:73-86, ||dW||_F matrix.hpp:38-41, trace point,
//                      eta stop rule online.hpp:390-396) in one cluster launch.
// K0  fresh_kernel   — reference fresh-restart uniforms: std::mt19937_64 seeded
//                      with splitmix64(mix_seed(seed, t)) (online.hpp:294-301,
//                      rng.hpp:10-34), bit-exact.
//
// Layout in HBM: the fp64 state (W, A, B, pending) is column-major
// F x K like the reference's Eigen matrices (coalesced per-column commit);
// per-CTA statistics partials are [2][KP][F] planes at the same cell offsets;
// W32 is the solver's fp32 copy, row-major [F][WS] with zero pad columns.  See DESIGN.md for the roofline of each kernel.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

namespace isnmf_dev {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kChunk = 32;  // rows of F per warp chunk
constexpr int kQS = 68;     // floats per Q/R staging row: q at [ng 4][8], r at 36 + [ng 4][8]
constexpr int kQR_R = 36;   // r half offset: 32 + 4 skew so the 8 (nd, ng) float4 reads of phase B
                            // hit 8 distinct 16-byte bank groups

enum : uint32_t {
  ST_NONPOS_INIT = 1u,
  ST_INCONSISTENT = 2u,
  ST_NONFINITE_W = 4u,
  ST_ZERO_COLUMN = 8u,
  ST_DIVERGED = 16u,
  ST_CHAIN_TIMEOUT = 32u,  // a statistics-chain predecessor never published its window (K1T)
};

// Device-resident scalar state of an online / batch context.
struct DevState {
  unsigned long long t;              // samples seen (online.hpp:226)
  unsigned long long commits;        // online.hpp:234
  unsigned long long pending_count;  // online.hpp:239
  unsigned long long trace_base;     // commits at the last trace clear
  unsigned long long origin_ns;      // clock origin for trace seconds
  double pending_div;                // online.hpp:238
  double last_delta;                 // online.hpp:233
  double last_obj;                   // online.hpp:240
  double kmeanw;                     // K * mean(W) (fresh_h_init, online.hpp:296-297)
  double prev_obj;                   // batch: previous objective (batch.hpp:129)
  unsigned int status;               // error bits (ST_*)
  unsigned int halt;                 // eta stop rule fired
  unsigned int ticket;               // last-block-done counter of fold_commit_kernel
  unsigned int pad;                  // error bits of the running fold_commit_kernel
};

// Optional per-phase cycle instrumentation (build with -DISNMF_PHASE_PROF):
// per warp, cycles spent in each phase are added to a.prof[(block*8+warp)*8 + phase].
#ifdef ISNMF_PHASE_PROF
#define PROF_T0() long long prof_t = clock64()
#define PROF_MARK(ph)                                                                   \
  do {                                                                                  \
    const long long prof_n = clock64();                                                 \
    if (lane == 0 && a.prof) a.prof[(blockIdx.x * kWarps + warp) * 8 + (ph)] += prof_n - prof_t; \
    prof_t = prof_n;                                                                    \
  } while (0)
#else
#define PROF_T0()
#define PROF_MARK(ph)
#endif

// Programmatic dependent launch (the online engine launches K1 and K2 with
// programmatic stream serialization): pdl_wait blocks until the preceding grid
// has completed and its memory is visible (a no-op for a normal launch);
// pdl_trigger lets the next grid start its launch before this one finishes.
// Device-side checks of the debug build (make debug -> lib_debug/, -DISNMF_DEBUG):
// a failed check prints its location and traps, so a bad index surfaces as a loud
// error (compute-sanitizer is closed on this pool).  Compiled out otherwise.
#ifdef ISNMF_DEBUG
#define ISNMF_DASSERT(cond)                                                                          \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("ISNMF_DASSERT %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #cond, blockIdx.x, \
             threadIdx.x);                                                                           \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define ISNMF_DASSERT(cond) \
  do {                      \
  } while (0)
#endif

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// is_term (kernels.hpp:15-18) in fp32, taking ratio = 1 + u = (v+eps)/lam
// computed as a product: a series for |u| < 1/4 (where u - log1p(u) cancels),
// u - log(ratio) elsewhere, so ratios far below 1 (v at the 1e-9 floor) keep
// full relative accuracy instead of rounding u to -1.  Relative error <~1e-6.
__device__ __forceinline__ float is_term_ratio(float ratio) {
  const float u = ratio - 1.0f;
  float p = -1.0f / 12.0f;
  p = fmaf(p, u, 1.0f / 11.0f);
  p = fmaf(p, u, -1.0f / 10.0f);
  p = fmaf(p, u, 1.0f / 9.0f);
  p = fmaf(p, u, -1.0f / 8.0f);
  p = fmaf(p, u, 1.0f / 7.0f);
  p = fmaf(p, u, -1.0f / 6.0f);
  p = fmaf(p, u, 1.0f / 5.0f);
  p = fmaf(p, u, -1.0f / 4.0f);
  p = fmaf(p, u, 1.0f / 3.0f);
  p = fmaf(p, u, -1.0f / 2.0f);
  const float series = -(u * u) * p;
  const float direct = u - __logf(ratio);
  const float t = fabsf(u) < 0.25f ? series : direct;
  return t > 0.0f ? t : 0.0f;
}

__device__ __forceinline__ double is_term_d(double u) {
  const double t = u - log1p(u);
  return t > 0.0 ? t : 0.0;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// K1 — fused solve.
// ---------------------------------------------------------------------------
struct SolveArgs {
  const float* W32;  // [F][SolveShape::WS], pad columns zero
  int ws;            // row stride of W32 (floats)
  const float* WB;   // K1C: W^T hi | lo in its K-major halves (pc_off_wb), nullable otherwise
  int F, K;
  const float* V;  // frames; block-local frame n is V + frame(n) * ldv
  int64_t ldv;
  const int64_t* vsel;  // frame(n) = vsel[n] (nullable)
  int64_t v0;           // frame(n) = v0 + n when vsel == nullptr
  int nframes;
  int cta_frames;  // frames per CTA of runtime-shaped kernels (K1M); set by launch_solve
  int pair2;       // K1M, one frame group: the frames' rows split over a 2-CTA cluster (K1P)
  int iters;
  float eps;
  double epsd;
  int h0_mode;  // 0 direct H0, 1 warm store (U, T, P), 2 fresh (u01, kmeanw)
  const float* H0;
  double* U;
  uint32_t* T;
  const double* P;
  uint32_t c_now;
  const uint64_t* widx;  // store column of frame n (nullable -> (wbase + n) mod wmod)
  int64_t wbase;
  int64_t wmod;
  const double* u01;
  const DevState* kst;  // kmeanw for fresh
  const double* hscale;  // optional per-k multiplier on h0 (batch rescale)
  float* Hout;           // [nframes][K] (nullable)
  int write_store;
  int do_stats;   // extra pass with the final h: divergence (+ statistics when stats != nullptr)
  int div_first;  // divergence from pass 0 (the incoming h) instead of the final pass
  int check_h0;   // flag h0 <= 0 as NonPositiveInit (solve_h, kernels.hpp:67)
  float* stats;     // [gridDim][2][KP][FP], FP = F rounded up to 4
  double* divpart;  // [gridDim]
  int stats_cap;    // planes / divergence partials allocated (debug checks; 0 = unchecked)
  // K1T statistics chain: CTAs b with the same b / chain share plane b / chain; rank b % chain
  // adds its window tile (rank 0 stores, the others red.add) once rank - 1 has published that
  // window through chain_flags[b - 1][warp] >= chain_base + window + 1 (fixed order per cell)
  int chain;                   // CTAs per plane (<= 1: one plane per CTA)
  uint32_t chain_base;         // 64 x the launch's chain epoch
  uint32_t* chain_flags;       // [gridDim][8 warps]
  unsigned int* status;
  const unsigned int* halt;
  long long* prof;  // phase cycle counters (ISNMF_PHASE_PROF builds only)
};

// ---------------------------------------------------------------------------
// Warm activation store — the reference's fp64 warm_h (online.hpp:229, 348-358).
// U[col][k] is fp64, T[col] the commit at which column col was last written; its
// value now is U * P[c_now][k] / P[T][k] (P = prefix products of the column
// scales, so the rescale of every stored H at each commit, model.hpp:84, costs
// O(K)).  The solver works in fp32, whose range does not cover every value the
// fp64 reference keeps: an atom that a frame does not use decays geometrically
// under the MM update, visit after visit (fp32 would flush it to 0 and the next
// visit would raise NonPositiveInit where the reference does not).  Such an h
// enters the solver as kWarmFloor — W * 2^-80 is ~1e-12 of the smallest Lam
// (eps = 1e-12) and leaves Lam's fp32 value unchanged, so the update factors
// sqrt(num/den) are the ones the true value sees — and the store keeps
// h0 * (h / kWarmFloor) in fp64.
// ---------------------------------------------------------------------------
constexpr float kWarmFloor = 0x1p-80f;

__device__ __forceinline__ int64_t warm_col(const SolveArgs& a, int n) {  // n = launch-local frame
  ISNMF_DASSERT(n >= 0 && n < a.nframes);
  const int64_t col = a.widx ? int64_t(a.widx[n]) : (a.wbase + n) % a.wmod;
  ISNMF_DASSERT(col >= 0 && col < a.wmod);
  return col;
}
// L2 prefetch of the tag and the U row of launch-local frame n: safe before the PDL wait (L2 is
// the coherence point: a later load sees whatever a launch still in flight writes), and it turns
// the two dependent HBM round trips of the prologue (tag, then U) into L2 hits
__device__ __forceinline__ void warm_prefetch(const SolveArgs& a, int n) {
  const int64_t col = warm_col(a, n);
  asm volatile("prefetch.global.L2 [%0];" ::"l"(a.T + col));
  const char* u = reinterpret_cast<const char*>(a.U + size_t(col) * a.K);
  const int bytes = a.K * int(sizeof(double));
  for (int off = 0; off < bytes + 127; off += 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(u + (off < bytes ? off : bytes - 1)));
}
__device__ __forceinline__ double warm_value(const SolveArgs& a, int64_t col, uint32_t tag, int k) {
  ISNMF_DASSERT(tag <= a.c_now && k >= 0 && k < a.K);
  return a.U[size_t(col) * a.K + k] * (a.P[size_t(a.c_now) * a.K + k] / a.P[size_t(tag) * a.K + k]);
}

// a direct or fresh h0 times the optional per-atom scale (batch: the last commit's
// column scales); flags h0 <= 0 (NonPositiveInit)
__device__ __forceinline__ float scaled_h0(const SolveArgs& a, float val, int k, int& bad) {
  if (a.hscale) val = float(double(val) * a.hscale[k]);
  if (!(val > 0.0f)) bad = 1;
  return val;
}

// h0 of launch-local frame n, atom k (n < nframes, k < K) as the solver's fp32
// start value; sets bad when the reference's solve_h would raise NonPositiveInit
// (h0 <= 0 or NaN, kernels.hpp:67).  meanv = the frame's mean (fresh mode only).
__device__ __forceinline__ float solve_h0(const SolveArgs& a, int n, int k, int64_t col, uint32_t tag,
                                          double meanv, int& bad) {
  float val;
  if (a.h0_mode == 1) {
    const double h0 = warm_value(a, col, tag, k);
    if (!(h0 > 0.0)) bad = 1;
    val = h0 < double(kWarmFloor) && h0 > 0.0 ? kWarmFloor : float(h0);
  } else {
    if (a.h0_mode == 0) {
      val = a.H0[size_t(n) * a.K + k];
    } else {
      const double mv = meanv > a.epsd ? meanv : a.epsd;
      val = float(mv / a.kst->kmeanw * a.u01[size_t(n) * a.K + k]);
    }
    val = scaled_h0(a, val, k, bad);
  }
  return val;
}

// Writes the final h of atom k to store column col (tag = the column's tag when
// the launch started; T is re-tagged separately, after every U write of the CTA).
__device__ __forceinline__ void warm_put(const SolveArgs& a, int64_t col, uint32_t tag, int k, float h) {
  const double h0 = warm_value(a, col, tag, k);
  a.U[size_t(col) * a.K + k] = h0 < double(kWarmFloor) ? h0 * (double(h) / double(kWarmFloor)) : double(h);
}

// Epilogue of every K1 variant: Hout and the warm store for the CTA's frames
// [n0, n0 + nf); hval(n, k) reads the final h.  Every thread of the CTA calls it.
template <class HVal>
__device__ __forceinline__ void write_final_h(const SolveArgs& a, int n0, int nf, HVal hval) {
  if (!a.Hout && !a.write_store) return;
  const int K = a.K;
  for (int idx = threadIdx.x; idx < nf * K; idx += blockDim.x) {
    const int n = idx / K, k = idx - n * K;
    const float h = hval(n, k);
    if (a.Hout) a.Hout[size_t(n0 + n) * K + k] = h;
    if (a.write_store) {
      const int64_t col = warm_col(a, n0 + n);
      warm_put(a, col, a.T[col], k, h);
    }
  }
  if (a.write_store) {
    __syncthreads();  // every U write of this CTA has read its column's old tag
    for (int n = threadIdx.x; n < nf; n += blockDim.x) a.T[warm_col(a, n0 + n)] = a.c_now;
  }
}

template <int TK>
struct KMap {
  static constexpr int M = TK / 4;
  static constexpr int TT = TK - 4 * M;
  __host__ __device__ static constexpr int k_of(int kg, int j) {
    return j < 4 * M ? 4 * (4 * (j / 4) + kg) + (j & 3) : 16 * M + kg * TT + (j - 4 * M);
  }
  __host__ __device__ static constexpr void inv(int k, int& kg, int& j) {
    if (k < 16 * M) {
      const int c = k >> 2;
      kg = c & 3;
      j = 4 * (c >> 2) + (k & 3);
    } else {
      const int off = k - 16 * M;
      kg = off / (TT > 0 ? TT : 1);
      j = 4 * M + off % (TT > 0 ? TT : 1);
    }
  }
};

template <int TK, int TN>
struct SolveShape {
  static constexpr int KP = 4 * TK;
  static constexpr int NT = 4 * TN;
  // dictionary row stride in smem: an odd number of float4s, so the 8 rows a
  // quarter-warp reads in phase A hit 8 distinct 16-byte bank groups
  static constexpr int WS = ((KP / 4) % 2 == 1) ? KP : KP + 4;
  static constexpr int cells = TK * TN;
  // per-lane num/den partial stride: odd, so scalar stores of 32 lanes are conflict-free
  static constexpr int PBS = (cells % 2 == 1) ? cells : cells + 1;
  static constexpr int union_floats =
      (kWarps * kChunk * kQS > kWarps * 32 * PBS) ? kWarps * kChunk * kQS : kWarps * 32 * PBS;
  // phase A on the tensor pipe (3xTF32 mma.sync m16n8k8, Lam^T = h^T W^T):
  // frames are the M dimension (MB blocks of 16), k the K dimension (KB blocks of 8)
  static constexpr int MB = (NT + 15) / 16;
  static constexpr int KB = (KP + 7) / 8;
  static constexpr int HF = MB * KB * 32 * 4;  // A fragments of h (one of hi / lo)
  static size_t smem_bytes(int F) { return sizeof(float) * (size_t(F) * WS + NT * KP + 2 * HF + union_floats); }
};

// Position of h[k][n] in the A-fragment copy (m16n8k8 tf32, row-major A = h^T):
// thread (g, t) of block (mb, kb) holds A[g][t], A[g+8][t], A[g][t+4], A[g+8][t+4].
template <int KB>
__device__ __forceinline__ int hfrag_index(int n, int k) {
  const int mb = n >> 4, r = n & 15, kb = k >> 3, c = k & 7;
  const int lane = 4 * (r & 7) + (c & 3), e = (r >> 3) + 2 * (c >> 2);
  return ((mb * KB + kb) * 32 + lane) * 4 + e;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// h -> the hi / lo fragment copies (hi = tf32(h), lo = h - hi)
__device__ __forceinline__ void put_hfrag(float* Hhi, float* Hlo, int idx, float h) {
  const float hi = tf32_rna(h);
  Hhi[idx] = hi;
  Hlo[idx] = h - hi;
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Loads the lane's TK dictionary values of one row (k-set of group kg).
template <int TK>
__device__ __forceinline__ void load_wk(const float* wr, int kg, float (&w)[TK]) {
  using KM = KMap<TK>;
#pragma unroll
  for (int q = 0; q < KM::M; ++q) {
    const float4 t = *reinterpret_cast<const float4*>(wr + 4 * (4 * q + kg));
    w[4 * q + 0] = t.x;
    w[4 * q + 1] = t.y;
    w[4 * q + 2] = t.z;
    w[4 * q + 3] = t.w;
  }
#pragma unroll
  for (int e = 0; e < KM::TT; ++e) w[4 * KM::M + e] = wr[16 * KM::M + kg * KM::TT + e];
}

template <int TN>
__device__ __forceinline__ void load_x(const float* xr, float (&x)[TN]) {
  if constexpr (TN >= 4) {
    const float4 a = *reinterpret_cast<const float4*>(xr);
    x[0] = a.x;
    x[1] = a.y;
    x[2] = a.z;
    x[3] = a.w;
    if constexpr (TN > 4) {
      const float4 b = *reinterpret_cast<const float4*>(xr + 4);
#pragma unroll
      for (int t = 4; t < TN; ++t) x[t] = (t == 4 ? b.x : t == 5 ? b.y : t == 6 ? b.z : b.w);
    }
  } else {
#pragma unroll
    for (int t = 0; t < TN; ++t) x[t] = xr[t];
  }
}

// Lane -> role maps.  An LDS.128 costs 2 shared-memory wavefronts when every
// aligned lane quad reads at most 2 distinct 16-byte addresses and 4 otherwise
// (measured, tools/probe/lds_probe.cu), so each quad spans 2 values of each of
// the two operand indices: phase A (row group rg 0..7, frame group fg 0..3)
// and phase B (k group kg 0..3, frame group ng 0..3, nd = num/den).
__device__ __forceinline__ int pa_rg(int lane) { return ((lane >> 1) & 1) | (((lane >> 2) & 3) << 1); }
__device__ __forceinline__ int pa_fg(int lane) { return (lane & 1) | (((lane >> 4) & 1) << 1); }
__device__ __forceinline__ int pb_kg(int lane) { return (lane & 1) | (((lane >> 2) & 1) << 1); }
__device__ __forceinline__ int pb_ng(int lane) { return ((lane >> 1) & 1) | (((lane >> 3) & 1) << 1); }
__device__ __forceinline__ int pb_lane(int kg, int ng, int nd) {
  return (kg & 1) | ((ng & 1) << 1) | ((kg >> 1) << 2) | ((ng >> 1) << 3) | (nd << 4);
}

// V values of a full chunk for this lane's phase-A cells (rows rg+8i, frames fg*TN+j).
template <int TN>
__device__ __forceinline__ void load_v(float (&vv)[4][TN], const float* const* fptr, int c0, int nf, int lane) {
  const int rg = pa_rg(lane), fg = pa_fg(lane);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = fg * TN + j;
      vv[i][j] = n < nf ? __ldg(fptr[n] + c0 + rg + 8 * i) : 0.0f;
    }
}

// Phase A of one warp chunk: lam = W h + eps for `rows` rows x NT frames;
// q = (v+eps)/lam^2 and r = 1/lam are staged into the warp's Q/R rows
// ([row][nd][ng][8], padding lanes of invalid frames hold 0).  For a full
// chunk vv holds the V values of this lane's cells (rows rg+8i, frames
// fg*TN+j), loaded one chunk ahead by load_v so the L2 latency hides behind
// phase B; a tail chunk (rows < 32) takes one (row, frame) cell per lane and
// vt = V of cell `lane` when rows * NT <= 32 (loaded once per launch).
template <int TK, int TN>
__device__ __forceinline__ void phase_a(const float* Ws, const float* Hs, float* QR, const float* const* fptr,
                                        int c0, int rows, int nf, float eps, int lane, float vt) {
  using S = SolveShape<TK, TN>;
  constexpr int KP = S::KP, NT = S::NT, WS = S::WS;
  if (rows == kChunk) {
    const int rg = pa_rg(lane), fg = pa_fg(lane);  // 8 row groups x 4 frame groups
    // V of this lane's cells (an L2 hit after the first pass), in flight during the k loop
    float vv[4][TN];
    load_v<TN>(vv, fptr, c0, nf, lane);
    float acc[4][TN];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
    const float* wrow = Ws + (c0 + rg) * WS;
    const float* hrow = Hs + fg * TN * KP;
    // software-pipelined over k quads with ping-pong register sets: the 4 + TN
    // float4 loads of quad kc+1 are in flight while the 16*TN FMAs of quad kc issue
    constexpr int NQ = KP / 4;
    float4 wa[4], ha[TN], wb[4], hb[TN];
    auto load = [&](int kc, float4(&w4)[4], float4(&h4)[TN]) {
#pragma unroll
      for (int i = 0; i < 4; ++i) w4[i] = *reinterpret_cast<const float4*>(wrow + 8 * i * WS + 4 * kc);
#pragma unroll
      for (int j = 0; j < TN; ++j) h4[j] = *reinterpret_cast<const float4*>(hrow + j * KP + 4 * kc);
    };
    // one k at a time across all 4*TN accumulators: consecutive FMAs are independent
    auto fma4 = [&](const float4(&w4)[4], const float4(&h4)[TN]) {
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(w4[i].x, h4[j].x, acc[i][j]);
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(w4[i].y, h4[j].y, acc[i][j]);
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(w4[i].z, h4[j].z, acc[i][j]);
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][j] = fmaf(w4[i].w, h4[j].w, acc[i][j]);
    };
    load(0, wa, ha);
#pragma unroll 1
    for (int kc = 0; kc < NQ; kc += 2) {
      load(kc + 1 < NQ ? kc + 1 : kc, wb, hb);
      fma4(wa, ha);
      if (kc + 1 >= NQ) break;
      load(kc + 2 < NQ ? kc + 2 : kc, wa, ha);
      fma4(wb, hb);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float* qrow = QR + (rg + 8 * i) * kQS + fg * 8;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const bool valid = fg * TN + j < nf;
        const float r = rcp_approx(acc[i][j] + eps);
        const float q = (vv[i][j] + eps) * r * r;
        qrow[j] = valid ? q : 0.0f;
        qrow[kQR_R + j] = valid ? r : 0.0f;
      }
    }
  } else {
    // tail rows (F not a multiple of 32 per warp): one (row, frame) cell per lane,
    // the k loop unrolled so every load is in flight before the FMA chain
    for (int cell = lane; cell < rows * NT; cell += 32) {
      const int rl = cell / NT, n = cell - rl * NT;
      const float* wr = Ws + (c0 + rl) * WS;
      const float* hr = Hs + n * KP;
      float acc = 0.0f;
#pragma unroll
      for (int kc = 0; kc < KP / 4; ++kc) {
        const float4 w4 = *reinterpret_cast<const float4*>(wr + 4 * kc);
        const float4 h4 = *reinterpret_cast<const float4*>(hr + 4 * kc);
        acc = fmaf(w4.x, h4.x, acc);
        acc = fmaf(w4.y, h4.y, acc);
        acc = fmaf(w4.z, h4.z, acc);
        acc = fmaf(w4.w, h4.w, acc);
      }
      const bool valid = n < nf;
      const float v = !valid ? 0.0f : (rows * NT <= 32 ? vt : __ldg(fptr[n] + c0 + rl));
      const float r = rcp_approx(acc + eps);
      const float q = (v + eps) * r * r;
      float* qrow = QR + rl * kQS + (n / TN) * 8 + (n % TN);
      qrow[0] = valid ? q : 0.0f;
      qrow[kQR_R] = valid ? r : 0.0f;
    }
  }
}

// Phase A of a full 32-row chunk on the tensor pipe: Lam^T (frames x rows) =
// h^T W^T + eps in 3xTF32 (lo*hi + hi*lo + hi*hi, fp32 accumulate: ~1e-6
// relative), then q = (v+eps)/Lam^2 and r = 1/Lam staged as in phase_a.
// A = h^T from the fragment copies (one LDS.128 per block), B = W^T read
// straight from the row-major dictionary (b0 = W[row g][8kb+t], b1 = ..+4);
// hi = the raw fp32 bits (the tensor core reads the tf32 part), lo = x minus
// its tf32 truncation.  C: c0/c1 = (frame g, rows 2t, 2t+1), c2/c3 = frame g+8.
// The work is split in steps (one k block each) so phase B of the previous
// chunk can interleave them: the HMMA pipe runs beside the FFMA pipe.
template <int TK, int TN>
struct MmaA {
  using S = SolveShape<TK, TN>;
  static constexpr int KP = S::KP, NT = S::NT, WS = S::WS, MB = S::MB, KB = S::KB;
  float acc[MB][4][4];
  uint32_t ahi[MB][4], alo[MB][4], bh[4][2], bl[4][2];  // operands of the current k block

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < 4; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[mb][nb][e] = 0.0f;
  }
  // operands of k block kb: A fragments (hi, lo) and W (raw = hi, remainder = lo)
  __device__ __forceinline__ void load(const float* Ws, const float* Hhi, const float* Hlo, int c0, int kb,
                                       int lane) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      const float4 x = *reinterpret_cast<const float4*>(Hhi + ((mb * KB + kb) * 32 + lane) * 4);
      const float4 y = *reinterpret_cast<const float4*>(Hlo + ((mb * KB + kb) * 32 + lane) * 4);
      ahi[mb][0] = __float_as_uint(x.x);
      ahi[mb][1] = __float_as_uint(x.y);
      ahi[mb][2] = __float_as_uint(x.z);
      ahi[mb][3] = __float_as_uint(x.w);
      alo[mb][0] = __float_as_uint(y.x);
      alo[mb][1] = __float_as_uint(y.y);
      alo[mb][2] = __float_as_uint(y.z);
      alo[mb][3] = __float_as_uint(y.w);
    }
    const float* wrow = Ws + (c0 + g) * WS + t + 8 * kb;
#pragma unroll
    for (int nb = 0; nb < 4; ++nb) {
      const float w0 = wrow[8 * nb * WS];
      const float w1 = (KP % 8 == 0 || kb + 1 < KB) ? wrow[8 * nb * WS + 4] : 0.0f;  // k >= KP reads nothing
      bh[nb][0] = __float_as_uint(w0);
      bh[nb][1] = __float_as_uint(w1);
      bl[nb][0] = __float_as_uint(w0 - __uint_as_float(__float_as_uint(w0) & 0xffffe000u));
      bl[nb][1] = __float_as_uint(w1 - __uint_as_float(__float_as_uint(w1) & 0xffffe000u));
    }
  }
  // one of the three products (0: lo*hi, 1: hi*lo, 2: hi*hi) for every (mb, nb) block
  __device__ __forceinline__ void sweep(int s) {
#pragma unroll
    for (int nb = 0; nb < 4; ++nb)
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        if (s == 0) mma_tf32(acc[mb][nb], alo[mb], bh[nb][0], bh[nb][1]);
        if (s == 1) mma_tf32(acc[mb][nb], ahi[mb], bl[nb][0], bl[nb][1]);
        if (s == 2) mma_tf32(acc[mb][nb], ahi[mb], bh[nb][0], bh[nb][1]);
      }
  }
  __device__ __forceinline__ void step(const float* Ws, const float* Hhi, const float* Hlo, int c0, int kb,
                                       int lane) {
    load(Ws, Hhi, Hlo, c0, kb, lane);
    sweep(0);
    sweep(1);
    sweep(2);
  }
  // V of this lane's output cells (frames g + 8*h8 + 16*mb, rows 8nb + 2t + e)
  static __device__ __forceinline__ void load_v(float (&v)[MB][2][4][2], const float* const* fptr, int c0, int nf,
                                                int lane) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int h8 = 0; h8 < 2; ++h8) {
        const int n = 16 * mb + g + 8 * h8;
        const bool valid = n < nf;
        const float* vp = fptr[valid ? n : 0] + c0 + 2 * t;
#pragma unroll
        for (int nb = 0; nb < 4; ++nb) {
          v[mb][h8][nb][0] = valid ? __ldg(vp + 8 * nb) : 0.0f;
          v[mb][h8][nb][1] = valid ? __ldg(vp + 8 * nb + 1) : 0.0f;
        }
      }
  }
  // q, r of the chunk into QR
  __device__ __forceinline__ void finish(const float (&v)[MB][2][4][2], float* QR, int nf, float eps,
                                         int lane) const {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int mb = 0; mb < MB; ++mb)
#pragma unroll
      for (int h8 = 0; h8 < 2; ++h8) {
        const int n = 16 * mb + g + 8 * h8;
        if (n >= NT) continue;
        const bool valid = n < nf;
        float* qp = QR + 2 * t * kQS + (n / TN) * 8 + (n % TN);
#pragma unroll
        for (int nb = 0; nb < 4; ++nb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float r = rcp_approx(acc[mb][nb][2 * h8 + e] + eps);
            const float q = (v[mb][h8][nb][e] + eps) * r * r;
            qp[(8 * nb + e) * kQS] = valid ? q : 0.0f;
            qp[(8 * nb + e) * kQS + kQR_R] = valid ? r : 0.0f;
          }
      }
  }
};

template <int TK, int TN>
__device__ __forceinline__ void phase_a_mma(const float* Ws, const float* Hhi, const float* Hlo, float* QR,
                                            const float* const* fptr, int c0, int nf, float eps, int lane) {
  using M = MmaA<TK, TN>;
  M m;
  float v[M::MB][2][4][2];
  M::load_v(v, fptr, c0, nf, lane);  // in flight during the k loop
  m.zero();
#pragma unroll 1
  for (int kb = 0; kb < M::KB; ++kb) m.step(Ws, Hhi, Hlo, c0, kb, lane);
  m.finish(v, QR, nf, eps, lane);
}

// IS divergence of the staged chunk (online.hpp:303-309 / kernels.hpp:52-53):
// 1 + u = (v+eps)/lam = q / r, branch-free, four independent partial sums.
template <int TN>
__device__ __forceinline__ float chunk_divergence(const float* QR, int rows, int nf, int lane) {
  constexpr int NT = 4 * TN;
  float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  const int cells = rows * NT;
#pragma unroll 4
  for (int cell = lane; cell < cells; cell += 32) {
    const int rl = cell / NT, n = cell - rl * NT;
    const float* qp = QR + rl * kQS + (n / TN) * 8 + (n % TN);
    const float q = qp[0], r = qp[kQR_R];
    const float t = (n < nf) ? is_term_ratio(q * rcp_approx(r)) : 0.0f;
    s[(cell >> 5) & 3] += t;
  }
  return (s[0] + s[1]) + (s[2] + s[3]);
}

template <int TK, int TN>
__global__ void __launch_bounds__(kThreads, 1) solve_kernel(const SolveArgs a) {
  using S = SolveShape<TK, TN>;
  using KM = KMap<TK>;
  constexpr int KP = S::KP, NT = S::NT, PBS = S::PBS, WS = S::WS;
  pdl_wait();
  if (*a.status || (a.halt && *a.halt)) return;

  extern __shared__ __align__(16) float smem[];
  const int F = a.F, K = a.K;
  float* Ws = smem;           // [F][WS]
  float* Hs = Ws + F * WS;    // [NT][KP]
  float* Hhi = Hs + NT * KP;  // h^T A-fragments for the tensor-pipe phase A: tf32 hi
  float* Hlo = Hhi + S::HF;   //   and the fp32 remainder
  float* UN = Hlo + S::HF;    // union: per-warp Q/R staging | per-lane num/den partials
  __shared__ const float* fptr[NT];
  __shared__ double red[kWarps];
  __shared__ double meanv[NT];
  __shared__ int s_bad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.x * NT;
  const int nf = min(NT, a.nframes - n0);
  PROF_T0();

  __shared__ __align__(8) unsigned long long wbar;
  if (tid == 0) {  // dictionary -> smem by TMA bulk copies, overlapped with the h0 set-up below
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&wbar));
    const uint32_t bytes = uint32_t(F) * WS * 4u;  // multiple of 16 (WS % 4 == 0)
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
  if (tid < NT) {
    const int64_t fr = tid < nf ? (a.vsel ? a.vsel[n0 + tid] : a.v0 + n0 + tid) : 0;
    fptr[tid] = a.V + fr * a.ldv;
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();

  if (a.h0_mode == 2) {  // mean of each frame in fp64 (fresh_h_init's v.mean())
    for (int n = warp; n < nf; n += kWarps) {
      double s = 0.0;
      for (int f = lane; f < F; f += 32) s += double(fptr[n][f]);
      s = warp_sum_d(s);
      if (lane == 0) meanv[n] = s / double(F);
    }
    __syncthreads();
  }

  for (int i = tid; i < 2 * S::HF; i += kThreads) Hhi[i] = 0.0f;  // padding frames / k stay 0
  __syncthreads();
  // h0 -> Hs (+ fragment copies)
  for (int idx = tid; idx < NT * KP; idx += kThreads) {
    const int n = idx / KP, k = idx - n * KP;
    float val = 0.0f;
    if (n < nf && k < K) {
      int bad = 0;
      const int64_t col = a.h0_mode == 1 ? warm_col(a, n0 + n) : 0;
      val = solve_h0(a, n0 + n, k, col, a.h0_mode == 1 ? a.T[col] : 0u, a.h0_mode == 2 ? meanv[n] : 0.0, bad);
      if (a.check_h0 && bad) s_bad = 1;
    }
    Hs[idx] = val;
    put_hfrag(Hhi, Hlo, hfrag_index<S::KB>(n, k), val);
  }
  {  // wait for the dictionary (phase 0 of wbar)
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

  PROF_MARK(0);  // prologue: W -> smem, h0
  const int r0 = (warp * F) / kWarps, r1 = ((warp + 1) * F) / kWarps;
  // full 32-row chunks of this warp, visited cyclically; V is prefetched one ahead
  const int nfull = (r1 - r0) / kChunk;
  // V of the tail chunk's cell `lane` (constant over the passes)
  float vt = 0.0f;
  {
    const int tr = r1 - r0 - nfull * kChunk;
    if (tr > 0 && tr * NT <= 32 && lane < tr * NT) {
      const int rl = lane / NT, n = lane - rl * NT;
      if (n < nf) vt = __ldg(fptr[n] + r0 + nfull * kChunk + rl);
    }
  }
  float* QR = UN + warp * (kChunk * kQS);
  const float eps = a.eps;
  float divacc = 0.0f;
  // phase-B lane roles: 4 k groups x 4 frame groups x {num, den}
  const int kg = pb_kg(lane), ng = pb_ng(lane), nd = lane >> 4;

  for (int pass = 0; pass < a.iters; ++pass) {
    float accB[TK][TN];
#pragma unroll
    for (int j = 0; j < TK; ++j)
#pragma unroll
      for (int t = 0; t < TN; ++t) accB[j][t] = 0.0f;

    // chunk 0's phase A runs alone; phase A of every further full chunk runs
    // on the tensor pipe interleaved with phase B of the chunk before it
    MmaA<TK, TN> mA;
    if (nfull > 0) phase_a_mma<TK, TN>(Ws, Hhi, Hlo, QR, fptr, r0, nf, eps, lane);
    for (int c0 = r0; c0 < r1; c0 += kChunk) {
      const int rows = min(kChunk, r1 - c0);
      if (rows < kChunk) phase_a<TK, TN>(Ws, Hs, QR, fptr, c0, rows, nf, eps, lane, vt);
      __syncwarp();
      if (a.div_first && pass == 0) divacc += chunk_divergence<TN>(QR, rows, nf, lane);
      PROF_MARK(1);  // phase A
      // ---------------- phase B: num += W^T q, den += W^T r (this warp's rows)
      const float* wr = Ws + c0 * WS;
      const float* xr = QR + nd * kQR_R + ng * 8;
      const bool overlap = c0 + kChunk < r0 + nfull * kChunk;  // the next chunk is a full one
      if (overlap) {
        // 4 rows of phase B per iteration with one k block of the next chunk's
        // MMA phase A in the same basic block, so the scheduler can interleave
        // HMMA with FFMA (in-order issue: a separate HMMA burst would stall the
        // FFMAs behind it)
        constexpr int KB = MmaA<TK, TN>::KB;
        static_assert(KB <= kChunk / 4, "one k block per 4-row step");
        mA.zero();
        auto row = [&](int rl) {
          float w[TK], x[TN];
          load_wk<TK>(wr + rl * WS, kg, w);
          load_x<TN>(xr + rl * kQS, x);
#pragma unroll
          for (int j = 0; j < TK; ++j)
#pragma unroll
            for (int t = 0; t < TN; ++t) accB[j][t] = fmaf(w[j], x[t], accB[j][t]);
        };
        // each 4-row step carries one k block: its three MMA sweeps sit between rows
#pragma unroll 1
        for (int it = 0; it < KB; ++it) {
          mA.load(Ws, Hhi, Hlo, c0 + kChunk, it, lane);
          row(4 * it);
          mA.sweep(0);
          row(4 * it + 1);
          mA.sweep(1);
          row(4 * it + 2);
          mA.sweep(2);
          row(4 * it + 3);
        }
        float vn[MmaA<TK, TN>::MB][2][4][2];  // V of the next chunk, in flight under the last rows
        MmaA<TK, TN>::load_v(vn, fptr, c0 + kChunk, nf, lane);
#pragma unroll 1
        for (int rl = 4 * KB; rl < kChunk; ++rl) row(rl);
        __syncwarp();  // phase B is done with this chunk's Q/R
        mA.finish(vn, QR, nf, eps, lane);
      } else {  // loads of row rl+1 issued before the FMAs of row rl
        float w[TK], x[TN];
        load_wk<TK>(wr, kg, w);
        load_x<TN>(xr, x);
#pragma unroll 2
        for (int rl = 0; rl < rows; ++rl) {
          float wn[TK], xn[TN];
          const int rn = rl + 1 < rows ? rl + 1 : rl;
          load_wk<TK>(wr + rn * WS, kg, wn);
          load_x<TN>(xr + rn * kQS, xn);
#pragma unroll
          for (int j = 0; j < TK; ++j)
#pragma unroll
            for (int t = 0; t < TN; ++t) accB[j][t] = fmaf(w[j], x[t], accB[j][t]);
#pragma unroll
          for (int j = 0; j < TK; ++j) w[j] = wn[j];
#pragma unroll
          for (int t = 0; t < TN; ++t) x[t] = xn[t];
        }
      }
      __syncwarp();
      PROF_MARK(2);  // phase B
    }

    // ---------------- cross-warp num/den reduction (fixed order) + MM update
    __syncthreads();  // every warp is done with its Q/R staging (aliases UN)
    PROF_MARK(3);  // wait at the end-of-pass barrier
    {
      float* pb = UN + (warp * 32 + lane) * PBS;
#pragma unroll
      for (int j = 0; j < TK; ++j)
#pragma unroll
        for (int t = 0; t < TN; ++t) pb[j * TN + t] = accB[j][t];
    }
    __syncthreads();
    // compile-time trip count: every thread's loads of all its items are independent
    constexpr int MI = (KP * NT + kThreads - 1) / kThreads;
#pragma unroll
    for (int m = 0; m < MI; ++m) {
      const int p = tid + m * kThreads;
      const int k = p / NT, n = p - k * NT;  // NT is a compile-time constant
      if (k < K && n < nf) {
        int kgp, jp;
        KM::inv(k, kgp, jp);
        const int ngp = n / TN, tp = n - ngp * TN;
        const float* p0 = UN + pb_lane(kgp, ngp, 0) * PBS + jp * TN + tp;
        float num = 0.0f, den = 0.0f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          num += p0[w * 32 * PBS];
          den += p0[(w * 32 + 16) * PBS];
        }
        float& h = Hs[n * KP + k];
        h = h * sqrtf(num / den);
        put_hfrag(Hhi, Hlo, hfrag_index<S::KB>(n, k), h);
      }
    }
    __syncthreads();
    PROF_MARK(4);  // partials + MM update
  }

  if (a.do_stats) {
    pdl_trigger();  // K2 may launch onto SMs as CTAs finish
    const bool want_div = !a.div_first || a.iters == 0;
    const int rgs = lane & 7, kgs = lane >> 3;
    for (int c0 = r0; c0 < r1; c0 += kChunk) {
      const int rows = min(kChunk, r1 - c0);
      if (rows == kChunk)
        phase_a_mma<TK, TN>(Ws, Hhi, Hlo, QR, fptr, c0, nf, eps, lane);
      else
        phase_a<TK, TN>(Ws, Hs, QR, fptr, c0, rows, nf, eps, lane, vt);
      __syncwarp();
      if (want_div) divacc += chunk_divergence<TN>(QR, rows, nf, lane);
      PROF_MARK(5);  // stats pass phase A + divergence
      if (a.stats) {
        // statistics: sa[f,k] = sum_n q[f,n] h[k,n], sb[f,k] = sum_n r[f,n] h[k,n]
        float sa[4][TK], sb[4][TK];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < TK; ++j) sa[i][j] = sb[i][j] = 0.0f;
        // pipelined over frames with ping-pong register sets: the loads of frame
        // n+1 issue before the FMAs of frame n.  Rows past `rows` (tail chunk)
        // accumulate stale staging values that are never stored.
        const float* qr = QR + rgs * kQS;
        float ha[TK], qa[4], ra[4], hb[TK], qb[4], rb[4];
        auto load = [&](int n, float(&hk)[TK], float(&q)[4], float(&r)[4]) {
          const int off = (n / TN) * 8 + (n % TN);
          load_wk<TK>(Hs + n * KP, kgs, hk);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            q[i] = qr[8 * i * kQS + off];
            r[i] = qr[8 * i * kQS + kQR_R + off];
          }
        };
        auto fma_frame = [&](const float(&hk)[TK], const float(&q)[4], const float(&r)[4]) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < TK; ++j) {
              sa[i][j] = fmaf(q[i], hk[j], sa[i][j]);
              sb[i][j] = fmaf(r[i], hk[j], sb[i][j]);
            }
        };
        load(0, ha, qa, ra);
#pragma unroll 1
        for (int n = 0; n < nf; n += 2) {
          load(n + 1 < nf ? n + 1 : n, hb, qb, rb);
          fma_frame(ha, qa, ra);
          if (n + 1 >= nf) break;
          load(n + 2 < nf ? n + 2 : n, ha, qa, ra);
          fma_frame(hb, qb, rb);
        }
        const int FP = (F + 3) & ~3;  // partial planes padded so K2 can read float4 quads
        float* outA = a.stats + size_t(blockIdx.x) * 2 * FP * KP;
        float* outB = outA + size_t(FP) * KP;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int rl = rgs + 8 * i;
          if (rl < rows) {
            const int f = c0 + rl;
#pragma unroll
            for (int j = 0; j < TK; ++j) {
              const int k = KM::k_of(kgs, j);
              outA[size_t(k) * FP + f] = sa[i][j];
              outB[size_t(k) * FP + f] = sb[i][j];
            }
          }
        }
      }
      __syncwarp();
      PROF_MARK(6);  // statistics
    }
  }

  // divergence partial of this CTA (fixed-order reduction)
  if (a.divpart) {
    double d = warp_sum_d(double(divacc));
    if (lane == 0) red[warp] = d;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s += red[w];
      a.divpart[blockIdx.x] = s;
    }
  }

  // final activations
  write_final_h(a, n0, nf, [&](int n, int k) { return Hs[n * KP + k]; });
  PROF_MARK(7);  // epilogue
}

// ---------------------------------------------------------------------------
// K2 — fold_commit_kernel: the per-CTA statistics partials of one mini-batch
// are folded into pending (online.hpp:360-361) and, at a mini-batch boundary,
// the whole dictionary_commit (online.hpp:319-336) runs in the same launch:
// A = rho A + pending, W = sqrt(A/B) (update_w, kernels.hpp:142-159), the l1
// column rescale (model.hpp:73-86), ||dW||_F, the trace point and the eta stop.
//
// Grid = K columns x kFoldCluster CTAs; one thread-block cluster per column.
// Rank r sums partial blocks [r*n/C, (r+1)*n/C) for every row of column k
// (float4 loads, fp64 sums), the cluster exchanges the C row sums through
// distributed shared memory and rank r finalises rows [r*F/C, (r+1)*F/C) —
// the column sum s_k is exchanged the same way, so no second launch and no
// global round trip is needed for the rescale.  Every sum is in a fixed order
// (bitwise reproducible).  The last CTA of the grid (ticket) folds the
// per-CTA ||dW||^2 / sum W partials in CTA order.
//
// Error bits found here go to DevState::fold_err and are merged into status by
// the last CTA: status is read at kernel entry by every CTA, so it must not
// change while a cluster is running (a CTA returning early would leave its
// cluster waiting at the barrier).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// K1C (csrc/kernels_tc.cuh) layout of one CTA's half of W^T: K-major without swizzle,
// N = k' (hi k | lo k), K = row, core matrices of 8 k' x 4 rows
constexpr int kWbRows = 256;
__host__ __device__ __forceinline__ int wb_offset(int kp, int row) {
  return (((kp >> 3) * (kWbRows / 4) + (row >> 2)) << 5) + ((kp & 7) << 2) + (row & 3);
}

struct FoldArgs {
  const float* stats;  // [nblk][2][KP][FP]
  const double* divpart;
  int nstat;  // statistics partial blocks to fold into pending (0: none)
  int ndiv;   // divergence partials to fold into pending_div
  int F, K, KP, WS;
  int nframes;
  double* W64;  // F x K column-major
  double* pa;   // pending_a
  double* pb;
  double* A;
  double* B;
  float* W32;
  float* WB;         // optional: the K1C layout of W^T (hi | lo, pc_off_wb), kp rows per half
  int wb_kp;
  double* P;         // prefix products of the column scales [commits+1][K]
  double* cta_part;  // [gridDim][2]: dW^2, sum W of this CTA
  int do_commit;
  double rho;
  DevState* st;
  unsigned int* halt;
  double eta;
  unsigned long long* tr_t;
  double* tr_obj;
  unsigned long long* tr_ns;
  long long tr_cap;
  double* scale_out;  // optional: column scales s_k of this commit (batch H compensation)
  int batch_mode;
  int stats_cap;      // planes / divergence partials allocated (debug checks; 0 = unchecked)
  int after_k1;       // this launch follows a K1 launch (the previous commit completed before that K1 started)
  int stats_tiled;    // 1: K1T's chained layout [window of 32 rows][sa|sb][KP][32], rows swizzled by k; 2: K1M's
                      // [window of 16 rows][sa|sb][K][16] (kernels_mma.cuh mm_plane_off)
  long long p_cap;    // rows of P (debug checks; 0 = unchecked)
  long long* tprof;  // ISNMF_PHASE_PROF builds: [gridDim][8] globaltimer stamps of thread 0
};

#ifdef ISNMF_PHASE_PROF
#define FOLD_T(i) \
  if (tid == 0 && a.tprof) a.tprof[blockIdx.x * 8 + (i)] = (long long)globaltimer_ns()
#else
#define FOLD_T(i)
#endif

constexpr int kFoldCluster = 4;
constexpr int kFoldThreads = 512;
constexpr int kFoldWarps = kFoldThreads / 32;

__host__ __device__ inline int fold_groups(int F) {
  const int nq = (F + 3) / 4;
  const int g = kFoldThreads / nq;
  return g < 1 ? 1 : (g > 16 ? 16 : g);
}
__host__ __device__ inline int fold_rows(int F) { return (F + kFoldCluster - 1) / kFoldCluster; }
// dynamic shared memory of fold_commit_kernel: row sums [2][F], this rank's rows of
// W, pending_a, pending_b, A, B (prefetched) and W_tmp, group partials
__host__ __device__ inline size_t fold_smem_bytes(int F) {
  const int nq = (F + 3) / 4, g = fold_groups(F);
  return sizeof(double) * (2 * size_t(F) + 6 * size_t(fold_rows(F)) + (g > 1 ? size_t(g) * nq * 8 : 0));
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// generic address of `p` (this CTA's shared memory) in the shared memory of cluster rank `r`
template <class T>
__device__ __forceinline__ const T* map_rank(const T* p, unsigned r) {
  const T* q;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(q) : "l"(p), "r"(r));
  return q;
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}

// fixed-order block sum (warp tree, then warps in order); valid in thread 0
__device__ __forceinline__ double block_sum_d(double v, double* red) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kFoldWarps; ++w) s += red[w];
  return s;
}

// two values at once (same per-value order as block_sum_d; red holds 2 * kFoldWarps doubles)
__device__ __forceinline__ void block_sum2_d(double& x, double& y, double* red) {
  x = warp_sum_d(x);
  y = warp_sum_d(y);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    red[warp] = x;
    red[kFoldWarps + warp] = y;
  }
  __syncthreads();
  double sx = 0.0, sy = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kFoldWarps; ++w) {
      sx += red[w];
      sy += red[kFoldWarps + w];
    }
  x = sx;
  y = sy;
}

#ifndef ISNMF_TEMPLATES_ONLY  // defined once, in engine.cu's translation unit
__global__ void __cluster_dims__(kFoldCluster, 1, 1) __launch_bounds__(kFoldThreads)
    fold_commit_kernel(const FoldArgs a) {
  pdl_trigger();  // the next K1 may start its launch; it waits for this grid before touching its outputs
  extern __shared__ __align__(16) double fsm[];
  __shared__ double red[2 * kFoldWarps];
  __shared__ double s_csr[kFoldCluster];
  __shared__ int s_last;
  const int F = a.F, tid = threadIdx.x;
  FOLD_T(0);
  const unsigned r = cluster_rank();
  const int k = blockIdx.x / kFoldCluster;
  ISNMF_DASSERT(a.stats_cap == 0 || (a.nstat <= a.stats_cap && a.ndiv <= 2 * a.stats_cap));
  ISNMF_DASSERT(a.p_cap == 0 || a.batch_mode || (long long)a.st->commits + 1 < a.p_cap);
  const int lo = int((long long)r * F / kFoldCluster), hi = int((long long)(r + 1) * F / kFoldCluster);
  const int R = fold_rows(F);
  double* sums = fsm;            // [2][F]: this rank's partial sums of column k (read by the whole cluster)
  double* rw = fsm + 2 * F;      // [R] W of rows lo..hi-1, then W_tmp
  double* rpa = rw + R;          // [R] pending_a, then A_new
  double* rpb = rpa + R;         // [R] pending_b, then B_new
  double* rA = rpb + R;          // [R] A
  double* rB = rA + R;           // [R] B
  double* grp = rB + R;          // [G][NQ][8]
  // the state of this rank's rows streams into shared memory behind the partial loads
  for (int f = lo + tid; f < hi; f += kFoldThreads) {
    const size_t cell = size_t(k) * F + f;
    cp_async8(rw + (f - lo), a.W64 + cell);
    cp_async8(rpa + (f - lo), a.pa + cell);
    cp_async8(rpb + (f - lo), a.pb + cell);
    if (a.do_commit) {
      cp_async8(rA + (f - lo), a.A + cell);
      cp_async8(rB + (f - lo), a.B + cell);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  // the commit count and the column's prefix product (the P row of this commit's predecessor)
  // for the warm-store table: two dependent L2 loads, taken off the rescale phase
  unsigned long long c_prev = 0;
  double p_prev = 1.0;
  const bool early_p = a.after_k1 != 0;  // (a K2 that directly follows another may still see the old count)
  if (early_p && a.do_commit && !a.batch_mode && r == 0 && tid == 0) {
    c_prev = a.st->commits;
    p_prev = a.P[size_t(c_prev) * a.K + k];
  }
  // the row state above is written only by the previous K2 (complete before the K1 that
  // precedes this grid started); the partials and the status come from that K1
  pdl_wait();
  if (a.st->status || *a.halt) {  // both fixed for the whole launch (see above)
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  // ---- 1. this rank's share of the partial blocks, all rows of column k
  const int NQ = (F + 3) / 4, G = fold_groups(F);
  const int FP = (F + 3) & ~3;
  const size_t plane = size_t(FP) * a.KP;
  const int b0 = int((long long)r * a.nstat / kFoldCluster), b1 = int((long long)(r + 1) * a.nstat / kFoldCluster);
  // plane geometry: [sa|sb][KP][FP], or K1T's chained window tiles (kernels_large_tc.cuh tc_stat_off)
  // or K1M's windows of 16 rows [window][sa|sb][K][16] (stats_tiled = 2, kernels_mma.cuh mm_plane_off)
  const size_t pstride = a.stats_tiled == 2   ? size_t((F + 15) / 16) * 2 * a.K * 16
                         : a.stats_tiled == 1 ? size_t((F + 31) / 32) * 2 * a.KP * 32
                                              : 2 * plane;
  const size_t yoff = a.stats_tiled == 2 ? size_t(a.K) * 16 : a.stats_tiled == 1 ? size_t(a.KP) * 32 : plane;
  for (int it = tid; it < NQ * G; it += kFoldThreads) {
    const int q = it % NQ, g = it / NQ;
    const float* base =
        a.stats_tiled == 2   ? a.stats + size_t(q >> 2) * 2 * a.K * 16 + size_t(k) * 16 +
                                   ((4 * (q & 3)) ^ (((k >> 1) & 1) << 3))
        : a.stats_tiled == 1 ? a.stats + size_t(q >> 3) * 2 * a.KP * 32 + size_t(k) * 32 +
                                   ((4 * (q & 7)) ^ (((k >> 1) & 3) << 3))
                             : a.stats + size_t(k) * FP + 4 * q;
    double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
    for (int b = b0 + g; b < b1; b += G) {
      const float4 x = __ldcg(reinterpret_cast<const float4*>(base + size_t(b) * pstride));
      const float4 y = __ldcg(reinterpret_cast<const float4*>(base + size_t(b) * pstride + yoff));
      s[0] += x.x;
      s[1] += x.y;
      s[2] += x.z;
      s[3] += x.w;
      s[4] += y.x;
      s[5] += y.y;
      s[6] += y.z;
      s[7] += y.w;
    }
    if (G == 1) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (4 * q + e < F) {
          sums[4 * q + e] = s[e];
          sums[F + 4 * q + e] = s[4 + e];
        }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) grp[size_t(it) * 8 + e] = s[e];
    }
  }
  FOLD_T(1);
  if (blockIdx.x == 0) {  // divergence + counters (fixed order: thread-strided, then the block tree)
    double d = 0.0;
    for (int b = tid; b < a.ndiv; b += kFoldThreads) d += a.divpart[b];
    d = block_sum_d(d, red);
    if (tid == 0) {
      a.st->pending_div += d;
      a.st->pending_count += (unsigned long long)a.nframes;
      a.st->t += (unsigned long long)a.nframes;
    }
  }
  if (G > 1) {
    __syncthreads();
    for (int f = tid; f < F; f += kFoldThreads) {
      const int q = f >> 2, e = f & 3;
      double ta = 0.0, tb = 0.0;
      for (int g = 0; g < G; ++g) {
        ta += grp[(size_t(g) * NQ + q) * 8 + e];
        tb += grp[(size_t(g) * NQ + q) * 8 + 4 + e];
      }
      sums[f] = ta;
      sums[F + f] = tb;
    }
  }
  cp_async_wait_all();
  cluster_sync_all();  // row sums of every rank (and this thread's prefetched rows) visible
  FOLD_T(2);
  // ---- 2. rows [lo, hi) of column k: cluster-wide sums in rank order, pending / commit part 1
  double cs = 0.0;
  unsigned bad = 0;
  for (int f = lo + tid; f < hi; f += kFoldThreads) {
    double ta = 0.0, tb = 0.0;
#pragma unroll
    for (int i = 0; i < kFoldCluster; ++i) {
      const double* rs = map_rank(sums, unsigned(i));
      ta += rs[f];
      tb += rs[F + f];
    }
    const int j = f - lo;
    const size_t cell = size_t(k) * F + f;
    const double w = rw[j];
    const double pa = rpa[j] + w * w * ta;
    const double pb = rpb[j] + tb;
    if (!a.do_commit) {
      a.pa[cell] = pa;
      a.pb[cell] = pb;
      continue;
    }
    const double An = a.rho * rA[j] + pa;  // rho scales the past (online.hpp:319-320)
    const double Bn = a.rho * rB[j] + pb;
    a.pa[cell] = 0.0;
    a.pb[cell] = 0.0;
    double wn = w;
    if (Bn > 0.0)
      wn = sqrt(An / Bn);
    else if (An > 0.0)
      bad |= ST_INCONSISTENT;
    if (!isfinite(wn)) bad |= ST_NONFINITE_W;
    rpa[j] = An;
    rpb[j] = Bn;
    rA[j] = wn;  // W_tmp (rw keeps the old W for ||dW||)
    cs += wn;
  }
  if (!a.do_commit) {
    cluster_sync_all();  // the other ranks may still read this CTA's sums
    return;
  }
  if (bad) atomicOr(&a.st->pad, bad);
  FOLD_T(3);
  cs = block_sum_d(cs, red);
  // ---- 3. column scale s_k, rescale of this rank's rows: every rank pushes its partial into
  // all four CTAs (DSMEM stores), one cluster barrier, then the same rank-order sum everywhere
  // (no rank touches another's shared memory after the barrier)
  if (tid == 0)
    for (int i = 0; i < kFoldCluster; ++i) *const_cast<double*>(map_rank(&s_csr[r], unsigned(i))) = cs;
  cluster_sync_all();
  FOLD_T(4);
  double sc = 0.0;
#pragma unroll
  for (int i = 0; i < kFoldCluster; ++i) sc += s_csr[i];
  const bool ok = sc > 0.0;
  double d2 = 0.0, cw = 0.0;
  for (int f = lo + tid; f < hi; f += kFoldThreads) {
    const int j = f - lo;
    const size_t cell = size_t(k) * F + f;
    if (!ok) {  // ZeroColumn: A, B committed, W unchanged (the status aborts the run)
      a.A[cell] = rpa[j];
      a.B[cell] = rpb[j];
      continue;
    }
    const double wn = rA[j] / sc;
    const double d = wn - rw[j];
    d2 += d * d;
    cw += wn;
    a.W64[cell] = wn;
    a.A[cell] = rpa[j] / sc;
    a.B[cell] = rpb[j] * sc;
    const float w32 = float(wn);
    a.W32[size_t(f) * a.WS + k] = w32;
    if (a.WB && f < 2 * kWbRows) {  // K1C's W^T halves: hi = the fp32 value, lo = its tf32 remainder
      const size_t half = size_t(f / kWbRows) * 2 * a.wb_kp * kWbRows;
      a.WB[half + wb_offset(k, f % kWbRows)] = w32;
      a.WB[half + wb_offset(a.wb_kp + k, f % kWbRows)] = w32 - __uint_as_float(__float_as_uint(w32) & 0xffffe000u);
    }
  }
  if (ok && r == 0 && tid == 0) {
    if (!a.batch_mode && !early_p) {
      c_prev = a.st->commits;
      p_prev = a.P[size_t(c_prev) * a.K + k];
    }
    if (!a.batch_mode) a.P[size_t(c_prev + 1) * a.K + k] = p_prev * sc;
    if (a.scale_out) a.scale_out[k] = sc;
  }
  if (!ok && tid == 0) atomicOr(&a.st->pad, ST_ZERO_COLUMN);
  FOLD_T(5);
  block_sum2_d(d2, cw, red);
  if (tid == 0) {
    a.cta_part[2 * blockIdx.x] = d2;
    a.cta_part[2 * blockIdx.x + 1] = cw;
    __threadfence();
    s_last = atomicAdd(&a.st->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  FOLD_T(6);
  if (!s_last) return;
  // ---- 4. last CTA: ||dW||_F, mean W, objective, trace point, stop rule
  __threadfence();
  double pd = 0.0, pw = 0.0;
  for (unsigned int b = tid; b < gridDim.x; b += kFoldThreads) {
    pd += __ldcg(a.cta_part + 2 * b);
    pw += __ldcg(a.cta_part + 2 * b + 1);
  }
  block_sum2_d(pd, pw, red);
  if (tid == 0) {
    volatile DevState* st = a.st;
    const unsigned int err = st->pad;
    const unsigned long long c = st->commits, t = st->t, pc = st->pending_count, tb = st->trace_base;
    const double pdiv = st->pending_div;
    st->ticket = 0;
    st->pad = 0;
    if (err) {
      st->status |= err;
      return;
    }
    const double delta = sqrt(pd), obj = pc ? pdiv / double(pc) : 0.0;
    if (a.batch_mode) {
      // epoch e = c + 1 of batch_train (batch.hpp:104-141): obj is the objective of
      // (W_{e-1}, H_{e-1}) from this epoch's K1; it must not exceed the previous one
      // (DivergedObjective, batch.hpp:129-131; the epoch count stays at e - 1)
      if (c > 0 && obj > st->prev_obj + 1e-6 * st->prev_obj + 1e-15) {
        st->status |= ST_DIVERGED;
        return;
      }
      st->prev_obj = obj;
      if (a.tr_obj && (long long)c < a.tr_cap) a.tr_obj[c] = obj;
      st->last_delta = delta;
      st->pending_div = 0.0;
      st->pending_count = 0;
      st->commits = c + 1;
      if (a.eta > 0.0 && delta < a.eta) *a.halt = 1u;  // stop after this epoch
      return;
    }
    st->last_delta = delta;
    st->kmeanw = double(a.K) * (pw / (double(a.F) * double(a.K)));
    st->last_obj = obj;
    const long long ti = (long long)(c - tb);
    if (a.tr_t && ti >= 0 && ti < a.tr_cap) {
      a.tr_t[ti] = t;
      a.tr_obj[ti] = obj;
      a.tr_ns[ti] = globaltimer_ns();
    }
    st->pending_div = 0.0;
    st->pending_count = 0;
    st->commits = c + 1;
    if (!a.batch_mode && a.eta > 0.0 && delta < a.eta) *a.halt = 1u;
  }
  FOLD_T(7);
}
#endif

// ---------------------------------------------------------------------------
// K0 — std::mt19937_64 (libstdc++ algorithm) per frame for fresh restarts.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

#ifndef ISNMF_TEMPLATES_ONLY  // defined once, in engine.cu's translation unit
__global__ void fresh_kernel(uint64_t seed, uint64_t t0, int n, int K, double* u01) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  constexpr int NN = 312, MM = 156;
  constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
  uint64_t mt[NN];
  // make_engine(mix_seed(seed, t)) = mt19937_64(splitmix64(mix_seed(seed, t)))  (rng.hpp:17-23)
  const uint64_t ms = splitmix64_d(splitmix64_d(seed) ^ splitmix64_d(~(t0 + uint64_t(i))));
  mt[0] = splitmix64_d(ms);
  for (int j = 1; j < NN; ++j) mt[j] = 6364136223846793005ULL * (mt[j - 1] ^ (mt[j - 1] >> 62)) + uint64_t(j);
  int p = NN;
  for (int k = 0; k < K; ++k) {
    if (p >= NN) {
      int j = 0;
      for (; j < NN - MM; ++j) {
        const uint64_t y = (mt[j] & UM) | (mt[j + 1] & LM);
        mt[j] = mt[j + MM] ^ (y >> 1) ^ ((y & 1ULL) ? MA : 0ULL);
      }
      for (; j < NN - 1; ++j) {
        const uint64_t y = (mt[j] & UM) | (mt[j + 1] & LM);
        mt[j] = mt[j + (MM - NN)] ^ (y >> 1) ^ ((y & 1ULL) ? MA : 0ULL);
      }
      const uint64_t y = (mt[NN - 1] & UM) | (mt[0] & LM);
      mt[NN - 1] = mt[MM - 1] ^ (y >> 1) ^ ((y & 1ULL) ? MA : 0ULL);
      p = 0;
    }
    uint64_t z = mt[p++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    u01[size_t(i) * K + k] = 1.0 - double(z >> 11) * 0x1.0p-53;  // uniform_open01 (rng.hpp:27-34)
  }
}
#endif

}  // namespace isnmf_dev

namespace isnmf_dev {

// ---------------------------------------------------------------------------
// K1g — generic solve for any K (used when W does not fit shared memory, e.g.
// config 4: F = 1025, K = 256).  W is streamed through shared memory in
// 32-row chunks every pass; each thread keeps num / den of its (k, n) pairs in
// registers.  Same inputs / outputs as solve_kernel (stats partials
// [CTA][2][KP][FP], divergence partials, H out / warm store).
// ---------------------------------------------------------------------------
constexpr int kGenThreads = 512;
constexpr int kGenChunk = 32;
constexpr int kGenMaxPairs = 32;  // (k, n) pairs per thread: K * NT <= 512 * 32

struct GenShape {
  int NT, KP, WS, QS;
  __host__ __device__ static int ws_for(int KP) { return ((KP / 4) % 2 == 1) ? KP : KP + 4; }
  __host__ __device__ GenShape(int nt, int K) : NT(nt), KP((K + 3) & ~3), WS(ws_for((K + 3) & ~3)), QS(2 * nt + 1) {}
  __host__ __device__ size_t smem_floats() const { return size_t(NT) * KP + size_t(kGenChunk) * WS + size_t(kGenChunk) * QS; }
};

#ifndef ISNMF_TEMPLATES_ONLY  // defined once, in engine.cu's translation unit
__global__ void __launch_bounds__(kGenThreads, 1) solve_generic_kernel(const SolveArgs a, int NT) {
  if (*a.status || (a.halt && *a.halt)) return;
  const int F = a.F, K = a.K;
  const GenShape G(NT, K);
  const int KP = G.KP, WS = G.WS, QS = G.QS;
  extern __shared__ __align__(16) float smem[];
  float* Hs = smem;                  // [NT][KP]
  float* Wc = Hs + NT * KP;          // [chunk rows][WS]
  float* QR = Wc + kGenChunk * WS;   // [chunk rows][q 0..NT-1 | r NT..2NT-1]
  __shared__ const float* fptr[64];
  __shared__ double red[kGenThreads / 32];
  __shared__ double meanv[64];
  __shared__ int s_bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.x * NT;
  const int nf = min(NT, a.nframes - n0);
  if (tid < NT) {
    const int64_t fr = tid < nf ? (a.vsel ? a.vsel[n0 + tid] : a.v0 + n0 + tid) : 0;
    fptr[tid] = a.V + fr * a.ldv;
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();
  if (a.h0_mode == 2) {
    for (int n = warp; n < nf; n += kGenThreads / 32) {
      double s = 0.0;
      for (int f = lane; f < F; f += 32) s += double(fptr[n][f]);
      s = warp_sum_d(s);
      if (lane == 0) meanv[n] = s / double(F);
    }
    __syncthreads();
  }
  for (int idx = tid; idx < NT * KP; idx += kGenThreads) {
    const int n = idx / KP, k = idx - n * KP;
    float val = 0.0f;
    if (n < nf && k < K) {
      int bad = 0;
      const int64_t col = a.h0_mode == 1 ? warm_col(a, n0 + n) : 0;
      val = solve_h0(a, n0 + n, k, col, a.h0_mode == 1 ? a.T[col] : 0u, a.h0_mode == 2 ? meanv[n] : 0.0, bad);
      if (a.check_h0 && bad) s_bad = 1;
    }
    Hs[idx] = val;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicOr(a.status, ST_NONPOS_INIT);
    return;
  }
  const float eps = a.eps;
  const int npairs = K * NT;
  float divacc = 0.0f;
  const int passes = a.iters + (a.do_stats ? 1 : 0);
  for (int pass = 0; pass < passes; ++pass) {
    const bool stats_pass = pass == a.iters;
    const bool want_div = a.div_first ? pass == 0 : stats_pass;
    float num[kGenMaxPairs], den[kGenMaxPairs];
#pragma unroll
    for (int i = 0; i < kGenMaxPairs; ++i) num[i] = den[i] = 0.0f;
    for (int c0 = 0; c0 < F; c0 += kGenChunk) {
      const int rows = min(kGenChunk, F - c0);
      __syncthreads();  // previous chunk's Wc / QR consumers are done
      for (int i = tid; i < rows * WS / 4; i += kGenThreads)
        reinterpret_cast<float4*>(Wc)[i] = __ldg(reinterpret_cast<const float4*>(a.W32 + size_t(c0) * WS) + i);
      __syncthreads();
      // phase A: lam, q, r for rows x NT cells
      for (int cell = tid; cell < rows * NT; cell += kGenThreads) {
        const int rl = cell / NT, n = cell - rl * NT;
        const float* wr = Wc + rl * WS;
        const float* hr = Hs + n * KP;
        float acc = 0.0f;
        for (int k = 0; k < KP; k += 4) {
          const float4 w4 = *reinterpret_cast<const float4*>(wr + k);
          const float4 h4 = *reinterpret_cast<const float4*>(hr + k);
          acc = fmaf(w4.x, h4.x, acc);
          acc = fmaf(w4.y, h4.y, acc);
          acc = fmaf(w4.z, h4.z, acc);
          acc = fmaf(w4.w, h4.w, acc);
        }
        const bool valid = n < nf;
        const float v = valid ? __ldg(fptr[n] + c0 + rl) : 0.0f;
        const float r = rcp_approx(acc + eps);
        const float vpe = v + eps;
        if (want_div && valid) divacc += is_term_ratio(vpe * r);
        QR[rl * QS + n] = valid ? vpe * r * r : 0.0f;
        QR[rl * QS + NT + n] = valid ? r : 0.0f;
      }
      __syncthreads();
      if (!stats_pass) {
        // phase B: num[k,n] += sum_f W[f,k] q[f,n], den with r
#pragma unroll
        for (int i = 0; i < kGenMaxPairs; ++i) {
          const int p = tid + i * kGenThreads;
          if (p < npairs) {
            const int n = p / K, k = p - n * K;
            float nu = num[i], de = den[i];
            for (int rl = 0; rl < rows; ++rl) {
              const float w = Wc[rl * WS + k];
              nu = fmaf(w, QR[rl * QS + n], nu);
              de = fmaf(w, QR[rl * QS + NT + n], de);
            }
            num[i] = nu;
            den[i] = de;
          }
        }
      } else if (a.stats) {
        // statistics of the chunk rows: sa[f,k] = sum_n q h, sb[f,k] = sum_n r h
        const int FP = (F + 3) & ~3;
        float* outA = a.stats + size_t(blockIdx.x) * 2 * FP * KP;
        float* outB = outA + size_t(FP) * KP;
        for (int cell = tid; cell < rows * KP; cell += kGenThreads) {
          const int k = cell / rows, rl = cell - k * rows;
          float sa = 0.0f, sb = 0.0f;
          for (int n = 0; n < nf; ++n) {
            const float h = Hs[n * KP + k];
            sa = fmaf(QR[rl * QS + n], h, sa);
            sb = fmaf(QR[rl * QS + NT + n], h, sb);
          }
          outA[size_t(k) * FP + c0 + rl] = sa;
          outB[size_t(k) * FP + c0 + rl] = sb;
        }
      }
    }
    if (!stats_pass) {
      __syncthreads();  // all phase-A reads of Hs done
#pragma unroll
      for (int i = 0; i < kGenMaxPairs; ++i) {
        const int p = tid + i * kGenThreads;
        if (p < npairs) {
          const int n = p / K, k = p - n * K;
          if (n < nf) Hs[n * KP + k] *= sqrtf(num[i] / den[i]);
        }
      }
      __syncthreads();
    }
  }
  if (a.divpart) {
    double d = warp_sum_d(double(divacc));
    if (lane == 0) red[warp] = d;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kGenThreads / 32; ++w) s += red[w];
      a.divpart[blockIdx.x] = s;
    }
  }
  __syncthreads();
  write_final_h(a, n0, nf, [&](int n, int k) { return Hs[n * KP + k]; });
}
#endif

}  // namespace isnmf_dev

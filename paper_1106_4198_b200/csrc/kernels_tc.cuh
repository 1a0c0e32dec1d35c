// K1C — the K <= 56 mini-batch solve (config 3: F = 513, K = 50, beta = 4096) on the
// 5th-generation tensor cores.  Same contract as the other K1 kernels (SolveArgs;
// solve_h kernels.hpp:62-80, accumulate_sample_stats kernels.hpp:95-108, the
// divergence online.hpp:303-309), online mode (do_stats, !div_first).
//
// A 2-CTA cluster owns up to 64 frames of the mini-batch; CTA rank r owns dictionary
// rows [256 r, 256 r + 256) for all of them (rows >= 512, at most kPcMaxTail, are
// done on the FP32 pipe by the tail warp).  3xTF32 everywhere (hi = the raw fp32
// value, which the tensor core truncates to tf32; lo = the remainder).
//
// Per MM iteration (one "pass"):
//   phase A   D_A[t][row][n] = W[row][:] h[:][n]        tcgen05.mma kind::tf32, A = the
//             CTA's dictionary rows hi | lo resident in TMEM for the whole launch
//             (tile t = rows 128t..), B = h (K-major, smem), M = 128, N = 64:
//             W_hi h_hi + W_hi h_lo + W_lo h_hi
//   epilogue  8 warps, warp (q, hh) = TMEM lane quarter q, frames 32hh..: Lam from TMEM,
//             q = (v+eps)/Lam^2, r = 1/Lam -> the phase-B A operands of the 32-row chunk
//             (q, t): [q_hi; r_hi] and [q_lo; r_lo] (M = 128 = 64 q frames + 64 r frames,
//             MN-major 128B_BASE32B swizzle), two chunk slots in flight
//   phase B   D_B[m][k'] += [q|r]_hi [W_hi | W_lo] + [q|r]_lo W_hi (M = 128, K = the chunk's
//             rows; B = W^T pre-split and laid out K-major by K2: WB)
//   update    D_B -> num / den partials of this CTA's rows, exchanged with the peer CTA
//             through distributed shared memory; both CTAs sum (own + peer + tail rows) in
//             the same fixed order and apply h *= sqrt(num/den) to all frames
// Statistics pass (final h): phase A, then per tile [q|r]_{hi,lo} written to TMEM as A
//   operands and sa[row][k] = sum_n q h, sb = sum_n r h (B = h^T, K-major, smem), 3xTF32,
//   drained into the pair's statistics plane (rows of this CTA).
//
// TMEM (512 columns): W_A [0, 4KP) | D_B [4KP, 6KP) | D_A[0] [384, 448) | D_A[1] [448, 512);
// statistics pass: A_S q_hi q_lo r_hi r_lo [0, 256) | D_S sa [256, 320) sb [320, 384).
// Shared memory: two 32 KB chunk slots (also the num/den exchange and h^T of the
// statistics pass) | WB (this CTA's half, 2KP x 256 floats, TMA) | h hi | h lo | tail rows.
#pragma once

#include "kernels_large_tc.cuh"
#include "kernels_mma.cuh"  // is_term_fast, sqrt_approx

namespace isnmf_dev {

constexpr int kPcRows = 256;    // dictionary rows per CTA
constexpr int kPcFrames = 64;   // frames of a pair (phase-A N, half of phase-B M)
constexpr int kPcEpiWarps = 8;  // epilogue warps: (quarter q = warp & 3, frame half hh = warp >> 2)
constexpr int kPcIssueWarp = 0; // its lane 0 issues phase A, tile 0's chunks and the statistics MMAs
constexpr int kPcTailWarp = 7;  // also the FP32 tail rows (quarter 3 waits for a slot first)
// lane 0 of this warp issues phase A of tile 1 once tile 0's is done (quarter 2 waits for its
// slot then; D_A[1] is its own accumulator, so the MMA issue order stays deterministic)
constexpr int kPcA1Warp = 6;
constexpr int kPcThreads = 256; // two warps per SM sub-partition: 255 registers, v + eps resident
// chunk issue order within tile t: quarters t, t + 1, t + 2, t + 3 (mod 4).  Tile t's chunks
// are issued by lane 0 of warp t (quarter t, frames 0..31), right after it has staged the
// tile's first chunk; warp 1 takes over from warp 0 at the tile boundary (mbarrier handoff +
// tcgen05 fences keep the issue order), so warp 0 stages its tile-1 chunk while warp 1 issues
__host__ __device__ constexpr int pc_chunk_quarter(int t, int i) { return (i + t) & 3; }
__host__ __device__ constexpr int pc_quarter_chunk(int t, int q) { return (q - t) & 3; }
constexpr int kPcMaxTail = 8;   // rows >= 512 on the FP32 pipe
constexpr int kPcSlotFloats = 2 * 128 * 32;

template <int KB>
struct PcShape {
  static constexpr int KP = 8 * KB;
  static constexpr int KP2 = 2 * KP;            // [hi | lo] rows of WB, columns of W_A per tile
  static constexpr int NHI = (KP + 15) & ~15;   // N of the hi-only MMAs
  static constexpr int XS = KP + 4;             // exchange row stride (conflict-free float4 rows)
  static constexpr int WB_FLOATS = KP2 * kPcRows;
  static constexpr int HA_FLOATS = kPcFrames * KP;
  static constexpr int HT_ROWS = KP2 + 8;       // h^T rows (+8: the hi-only B of the lo half reads past)
  static constexpr int TAIL_FLOATS = kPcMaxTail * KP + 2 * kPcMaxTail * kPcFrames;
  static constexpr uint32_t C_DB = 4 * KP, C_DA = 384, C_AS = 0, C_DS = 256;
  static_assert(6 * KP <= 384, "TMEM budget");
  static_assert(4 * kPcFrames * XS <= 2 * kPcSlotFloats, "exchange buffer fits the chunk slots");
  static_assert(HT_ROWS * kPcFrames <= 2 * kPcSlotFloats, "h^T fits the chunk slots");
  static constexpr size_t smem_bytes() {
    return sizeof(float) * (2 * kPcSlotFloats + WB_FLOATS + 2 * HA_FLOATS + TAIL_FLOATS) + 1024;
  }
};

// offsets (floats) in the layouts above (WB: wb_offset, csrc/kernels.cuh)
static_assert(kPcRows == kWbRows, "K1C rows per CTA = the WB half");
// h (phase-A B operand): K-major, N = frame, K = k
template <int KP>
__device__ __forceinline__ int pc_off_h(int n, int k) {
  return (((n >> 3) * (KP / 4) + (k >> 2)) << 5) + ((n & 7) << 2) + (k & 3);
}
// h^T (statistics B operand): K-major, N = k' (hi | lo), K = frame
__device__ __forceinline__ int pc_off_ht(int kp, int n) {
  return (((kp >> 3) * (kPcFrames / 4) + (n >> 2)) << 5) + ((kp & 7) << 2) + (n & 3);
}
// chunk A operand (phase B): MN-major 128B_BASE32B, MN = m (64 q frames + 64 r frames),
// K = row of the 32-row chunk: atoms of 32 m x 4 rows, [row atom][m atom], the four
// 32-byte chunks of a 128-byte atom row XOR-ed with row % 4 (csrc/kernels_large_tc.cuh)
__device__ __forceinline__ int pc_off_st(int m, int row) {
  const int r4 = row & 3;
  return ((((row >> 2) << 2) + (m >> 5)) << 7) + (r4 << 5) + ((((m & 31) >> 3) ^ r4) << 3) + (m & 7);
}

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(
          d),
      "r"(a), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
// arrive on the mbarrier at the same offset in the peer CTA (release, cluster scope)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(dsmem_addr(bar, rank))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, "
        "0, P;\n\t}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void dsmem_st4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// tcgen05.ld / st of N consecutive columns of this warp's 32 lanes (32x32b shape)
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float* v);
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t ta, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(ta));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t ta, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(ta));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t ta, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<32>(uint32_t ta, float* v) {
  tmem_ld<16>(ta, v);
  tmem_ld<16>(ta + 16, v + 16);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const float* v);
template <>
__device__ __forceinline__ void tmem_st<8>(uint32_t ta, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
template <>
__device__ __forceinline__ void tmem_st<16>(uint32_t ta, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          ta),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
// N (a multiple of 8, <= 64) columns as 16- and 8-column pieces
template <int N>
__device__ __forceinline__ void tmem_st_n(uint32_t ta, const float* v) {
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16) tmem_st<16>(ta + c, v + c);
  if constexpr (N % 16 != 0) tmem_st<8>(ta + (N & ~15), v + (N & ~15));
}
template <int N>
__device__ __forceinline__ void tmem_ld_n(uint32_t ta, float* v) {
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16) tmem_ld<16>(ta + c, v + c);
  if constexpr (N % 16 >= 8) tmem_ld<8>(ta + (N & ~15), v + (N & ~15));
  if constexpr (N % 8 != 0) tmem_ld<4>(ta + (N & ~7), v + (N & ~7));
}

__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// ISNMF_PC_TRACE builds (make trace): the last site each warp reached, written to mapped
// host memory (readable while the kernel runs): [CTA][warp] = pass << 24 | site << 16 | arg
#ifdef ISNMF_PC_TRACE
static __device__ unsigned long long* g_pc_trace = nullptr;  // (tc_table.cu's copy is set)
// per-warp timeline of CTAs 0 and 1 in shared memory (a store to sysmem before a
// barrier.cluster.arrive.release would be waited for), dumped at the end of the launch to
// g_pc_trace[4096 + (cta * 10 + warp) * 512 ..]: clock64 << 16 | site << 8 | (arg & 0xff)
constexpr int kPcLog = 128;
#ifndef ISNMF_PC_TRACE_MIN
#define ISNMF_PC_TRACE_MIN 0  // 7: pass-level sites only (the whole launch fits the log)
#endif
#define PC_MARK(site, arg)                                                                            \
  do {                                                                                                \
    if ((threadIdx.x & 31) == 0 && pc_n < kPcLog &&                                                   \
        ((site) >= ISNMF_PC_TRACE_MIN && !((site) >= 21 && (site) <= 25) || ISNMF_PC_TRACE_MIN == 0))   \
      pc_log[(threadIdx.x >> 5) * kPcLog + pc_n++] =                                                  \
          (unsigned long long)clock64() << 16 | (unsigned long long)(site) << 8 | ((arg) & 0xff);     \
  } while (0)
#else
#define PC_MARK(site, arg)
#endif

template <int KB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPcThreads, 1) solve_pair_kernel(const SolveArgs a) {
  using S = PcShape<KB>;
  constexpr int KP = S::KP, KP2 = S::KP2, NHI = S::NHI, XS = S::XS, KH = KP / 2;
  extern __shared__ __align__(16) float smem_raw[];
  const uint32_t sbase = smem_addr(smem_raw);
  float* smem = smem_raw + ((((sbase + 1023u) & ~1023u) - sbase) >> 2);
  float* slot = smem;                    // [2][2][128 x 32] chunk A operands | exchange | h^T
  float* WB = slot + 2 * kPcSlotFloats;  // this CTA's rows of W^T (hi | lo), from a.WB by TMA
  float* Hh = WB + S::WB_FLOATS;         // h (raw fp32 = hi), phase-A B operand
  float* Hl = Hh + S::HA_FLOATS;         // h lo
  float* Wt = Hl + S::HA_FLOATS;         // [kPcMaxTail][KP] tail rows of W
  float* Qt = Wt + kPcMaxTail * KP;      // [kPcMaxTail][64] q of the tail rows
  float* Rt = Qt + kPcMaxTail * kPcFrames;
  float* XB = slot;                      // [src][num|den][64][XS] num / den partials
  float* HT = slot;                      // [HT_ROWS] h^T (statistics pass)
  __shared__ const float* fptr[kPcFrames];
  __shared__ double meanv[kPcFrames];
  __shared__ int64_t colv[kPcFrames];
  __shared__ uint32_t tagv[kPcFrames];
  __shared__ double red[kPcThreads / 32];
  __shared__ int s_bad, s_go, s_go_peer;
  __shared__ uint32_t s_tmem;
  // bar_full / bar_empty per chunk (each completes once a pass, so a parity wait is exact)
  __shared__ __align__(8) uint64_t bar_w, bar_a[2], bar_full[8], bar_empty[8], bar_b, bar_sa, bar_s;
  // exchange: bar_pfree = the peer's phase B is done (its slots take our partials), bar_xfull =
  // the peer's partials have landed in our slots (bulk copy, complete_tx)
  __shared__ __align__(8) uint64_t bar_pfree, bar_xfull;
  __shared__ __align__(8) uint64_t bar_h;  // the peer's updated h (its frames) has landed in our Hh
  __shared__ __align__(8) uint64_t bar_hand;  // tile 0's chunks are issued (warp 0 -> warp 1)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_ctarank(), peer = rank ^ 1u;
  const int pair = blockIdx.x >> 1;
  const int F = a.F, K = a.K;
  const int n0 = pair * a.cta_frames;
  const int nf = min(a.cta_frames, a.nframes - n0);
  const int rowF = min(F, 2 * kPcRows);          // rows on the tensor cores: [0, rowF)
  const int ntail = F > 2 * kPcRows ? F - 2 * kPcRows : 0;
  const float eps = a.eps;
  int pass_no = 0, pc_n = 0;
  (void)pass_no;
  (void)pc_n;
#ifdef ISNMF_PC_TRACE
  __shared__ unsigned long long pc_log[(kPcThreads / 32) * kPcLog];
#endif

  PC_MARK(19, 0);
  // ---- before the PDL wait (overlaps the previous mini-batch's K2): nothing K2 writes
  if (warp == kPcIssueWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&s_tmem)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  cluster_arrive();  // (waited before the first access to the peer's shared memory)
  if (tid == 0) {
    s_bad = 0;
    mbar_init(&bar_w, 1);
    for (int i = 0; i < 2; ++i) mbar_init(&bar_a[i], 1);
    for (int i = 0; i < 8; ++i) {
      mbar_init(&bar_full[i], 64);
      mbar_init(&bar_empty[i], 1);
    }
    mbar_init(&bar_b, 1);
    mbar_init(&bar_sa, 32 * kPcEpiWarps);
    mbar_init(&bar_s, 1);
    mbar_init(&bar_pfree, 1);
    mbar_init(&bar_xfull, 1);  // thread 0's arrive.expect_tx + the peer's bulk copy
    mbar_init(&bar_h, 1);      // the same for the h block
    mbar_init(&bar_hand, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < kPcFrames) {
    const int64_t fr = tid < nf ? (a.vsel ? a.vsel[n0 + tid] : a.v0 + n0 + tid) : 0;
    fptr[tid] = a.V + fr * a.ldv;
  }
  __syncthreads();
  const int q = warp & 3, hh = (warp >> 2) & 1;
  // v + eps of this thread's cells (rows 128t + 32q + lane, frames 32hh ..), resident for every pass
  float vr[2][32];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int row = int(rank) * kPcRows + 128 * t + 32 * q + lane;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = 32 * hh + j;
      vr[t][j] = (row < rowF && n < nf ? __ldg(fptr[n] + row) : 0.0f) + eps;
    }
  }
  if (a.h0_mode == 1 && tid < nf) warm_prefetch(a, n0 + tid);
  pdl_wait();
  PC_MARK(20, 0);
  if (tid == 0) {
    s_go = !(*a.status || (a.halt && *a.halt));
    if (s_go) {  // this CTA's half of W^T by TMA bulk copies
      const uint32_t bytes = uint32_t(S::WB_FLOATS) * 4u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar_w)), "r"(bytes));
      const char* src = reinterpret_cast<const char*>(a.WB + size_t(rank) * S::WB_FLOATS);
      constexpr uint32_t kPiece = 32768;
      for (uint32_t off = 0; off < bytes; off += kPiece) {
        const uint32_t nb = bytes - off < kPiece ? bytes - off : kPiece;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(WB) + off),
            "l"(src + off), "r"(nb), "r"(smem_addr(&bar_w))
            : "memory");
      }
    }
  }
  // the dictionary rows for TMEM (W_A: warp (q, t = hh) holds rows 128t + 32q + lane), loaded
  // now, stored after the warm-store reads below are in flight
  const int wa_row = int(rank) * kPcRows + 128 * hh + 32 * q + lane;
  float4 wa[KP / 4];
#pragma unroll
  for (int k4 = 0; k4 < KP / 4; ++k4)
    wa[k4] = wa_row < rowF ? __ldg(reinterpret_cast<const float4*>(a.W32 + size_t(wa_row) * a.ws + 4 * k4))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
  PC_MARK(26, 0);
  if (a.h0_mode == 1 && tid < nf) {  // warm-store column and tag of every frame
    const int64_t col = warm_col(a, n0 + tid);
    colv[tid] = col;
    tagv[tid] = a.T[col];
  }
  __syncthreads();
  if (a.h0_mode == 2) {  // fresh: mean of each frame (fresh_h_init's v.mean())
    for (int n = warp; n < nf; n += kPcThreads / 32) {
      double s = 0.0;
      for (int f = lane; f < F; f += 32) s += double(fptr[n][f]);
      s = warp_sum_d(s);
      if (lane == 0) meanv[n] = s / double(F);
    }
    __syncthreads();
  }
  PC_MARK(27, 0);
  // h0 of every frame of the pair (both CTAs hold all of h), zero outside n < nf, k < K
  if (a.h0_mode == 1 && kPcThreads == 4 * kPcFrames) {
    // warm store (kernels.cuh warm_value / solve_h0): thread (frame n, k phase kq) issues all its
    // U and P loads before using any (the store is cold in HBM: one latency, not KP / 4)
    constexpr int NKQ = (KP + 3) / 4;
    const int n = tid >> 2, kq = tid & 3;
    const bool fr = n < nf;
    const int64_t col = fr ? colv[n] : 0;
    const uint32_t tag = fr ? tagv[n] : 0u;
    const double* urow = a.U + size_t(col) * K;
    const double* prow = a.P + size_t(tag) * K;
    const double* pnow = a.P + size_t(a.c_now) * K;
    double u[NKQ], pt[NKQ], pn[NKQ];
#pragma unroll
    for (int j = 0; j < NKQ; ++j) {
      const int k = 4 * j + kq;
      const bool ok = fr && k < K;
      u[j] = ok ? urow[k] : 0.0;
      pt[j] = ok ? prow[k] : 1.0;
      pn[j] = ok ? pnow[k] : 1.0;
    }
    int bad = 0;
#pragma unroll
    for (int j = 0; j < NKQ; ++j) {
      const int k = 4 * j + kq;
      if (k >= KP) continue;
      float val = 0.0f;
      if (fr && k < K) {
        const double h0 = u[j] * (pn[j] / pt[j]);
        if (!(h0 > 0.0)) bad = 1;
        val = h0 < double(kWarmFloor) && h0 > 0.0 ? kWarmFloor : float(h0);
      }
      Hh[pc_off_h<KP>(n, k)] = val;
      Hl[pc_off_h<KP>(n, k)] = tf32_lo(val);
    }
    if (a.check_h0 && bad) s_bad = 1;
  } else {
    for (int idx = tid; idx < kPcFrames * KP; idx += kPcThreads) {
      const int n = idx / KP, k = idx - n * KP;
      float val = 0.0f;
      if (n < nf && k < K) {
        int bad = 0;
        val = solve_h0(a, n0 + n, k, a.h0_mode == 1 ? colv[n] : 0, a.h0_mode == 1 ? tagv[n] : 0u,
                       a.h0_mode == 2 ? meanv[n] : 0.0, bad);
        if (a.check_h0 && bad) s_bad = 1;
      }
      Hh[pc_off_h<KP>(n, k)] = val;
      Hl[pc_off_h<KP>(n, k)] = tf32_lo(val);
    }
  }
  PC_MARK(28, 0);
  // tail rows of W (rows >= 512) for the FP32 tail warp
  for (int idx = tid; idx < ntail * KP; idx += kPcThreads) {
    const int i = idx / KP, k = idx - i * KP;
    Wt[idx] = k < K ? a.W32[size_t(2 * kPcRows + i) * a.ws + k] : 0.0f;
  }
  const uint32_t tmem = s_tmem;
  {  // W_A: hi = the fp32 value (the tensor core reads its tf32 part), lo = the remainder
    float hi[KP], lo[KP];
#pragma unroll
    for (int k4 = 0; k4 < KP / 4; ++k4) {
      hi[4 * k4] = wa[k4].x;
      hi[4 * k4 + 1] = wa[k4].y;
      hi[4 * k4 + 2] = wa[k4].z;
      hi[4 * k4 + 3] = wa[k4].w;
    }
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      if (k >= K) hi[k] = 0.0f;
      lo[k] = tf32_lo(hi[k]);
    }
    const uint32_t ta = tmem + (uint32_t(32 * q) << 16) + uint32_t(hh * KP2);
    tmem_st_n<KP>(ta, hi);
    tmem_st_n<KP>(ta + KP, lo);
    tmem_st_wait();
  }
  PC_MARK(29, 0);
  proxy_fence();
  tc_fence_before();
  // the go decision of both CTAs (a status bit set by another cluster of this launch could
  // otherwise split the pair); also orders every prologue read of the warm store before the
  // owners' final writes
  cluster_wait();  // the peer has started: its shared memory may be accessed
  PC_MARK(30, 0);
  if (tid == 0) {
    const uint32_t ra = dsmem_addr(&s_go_peer, peer);
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(s_go) : "memory");
  }
  cluster_arrive();
  cluster_wait();
  tc_fence_after();
  const bool go = s_go && s_go_peer;
  const bool bad = s_bad != 0;
  if (!go || bad) {
    if (bad && go && tid == 0) atomicOr(a.status, ST_NONPOS_INIT);
    if (s_go) mbar_wait(&bar_w, 0);  // the TMA must land before the CTA exits
    tc_fence_before();
    __syncthreads();
    if (warp == kPcIssueWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    return;
  }
  mbar_wait(&bar_w, 0);
  PC_MARK(1, 0);

  const uint32_t tlane = tmem + (uint32_t(32 * q) << 16);
  float divacc = 0.0f;
  // ---- MMA issue (lane 0 of warp kPcIssueWarp, in program order between its epilogue steps)
  auto issue_phase_a = [&](int t) {  // tile t: D_A[t] = W_hi h_hi + W_hi h_lo + W_lo h_hi
    tc_fence_after();
    constexpr uint32_t idA = umma_idesc_tf32(128, kPcFrames, 0, 0);
    const uint32_t d = tmem + S::C_DA + uint32_t(64 * t);
#pragma unroll
    for (int s = 0; s < KB; ++s) {
      const uint32_t ahi = tmem + uint32_t(t * KP2 + 8 * s), alo = ahi + KP;
      const uint64_t bh = umma_desc(smem_addr(Hh + 64 * s), 128, (KP / 4) * 128, 0);
      const uint64_t bl = umma_desc(smem_addr(Hl + 64 * s), 128, (KP / 4) * 128, 0);
      umma_ts(d, ahi, bh, idA, s > 0 ? 1u : 0u);
      umma_ts(d, ahi, bl, idA, 1u);
      umma_ts(d, alo, bh, idA, 1u);
    }
    umma_commit(&bar_a[t]);
  };
  // phase B of chunks c0 .. c0 + n - 1 (issue order: tile c / 4, quarter pc_chunk_quarter(c % 4)),
  // each once its slot is staged
  auto issue_chunks = [&](int c0, int n, int pass) {
    constexpr uint32_t id1 = umma_idesc_tf32(128, KP2, 1, 0), id2 = umma_idesc_tf32(128, NHI, 1, 0);
#pragma unroll 1
    for (int c = c0; c < c0 + n; ++c) {
      const int sl = c & 1, t = c >> 2, qq = pc_chunk_quarter(t, c & 3);
      if (c == 4) {  // tile 0's MMAs were issued by warp 0
        mbar_wait(&bar_hand, pass & 1);
        tc_fence_after();
      }
      PC_MARK(21, c);
      mbar_wait(&bar_full[c], pass & 1);
      PC_MARK(22, c);
      tc_fence_after();
      const float* op0 = slot + sl * kPcSlotFloats;
      const float* op1 = op0 + kPcSlotFloats / 2;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int row0 = 128 * t + 32 * qq + 8 * s;
        const uint64_t a0 = umma_desc(smem_addr(op0 + 2 * s * 4 * 128), 512, 4 * 512, 1);
        const uint64_t a1 = umma_desc(smem_addr(op1 + 2 * s * 4 * 128), 512, 4 * 512, 1);
        const uint64_t bw = umma_desc(smem_addr(WB + (row0 >> 2) * 32), 128, (kPcRows / 4) * 128, 0);
        umma_tf32(tmem + S::C_DB, a0, bw, id1, (c > 0 || s > 0) ? 1u : 0u);
        umma_tf32(tmem + S::C_DB, a1, bw, id2, 1u);
      }
      umma_commit(&bar_empty[c]);
      if (c == 3) {
        tc_fence_before();
        mbar_arrive(&bar_hand);
      }
    }
    if (c0 + n == 8) {
      umma_commit(&bar_b);
      PC_MARK(23, 0);
    }
  };
  // statistics MMAs of tile t once every thread has written its A_S columns
  auto issue_stats = [&](int t) {
    constexpr uint32_t idS = umma_idesc_tf32(128, NHI, 0, 0);
    PC_MARK(24, t);
    mbar_wait(&bar_sa, t & 1);
    PC_MARK(25, t);
    tc_fence_after();
#pragma unroll
    for (int s = 0; s < kPcFrames / 8; ++s) {
      const uint64_t bh = umma_desc(smem_addr(HT + 64 * s), 128, (kPcFrames / 4) * 128, 0);
      const uint64_t bl =
          umma_desc(smem_addr(HT + (KP / 8) * (kPcFrames / 4) * 32 + 64 * s), 128, (kPcFrames / 4) * 128, 0);
      const uint32_t qh = tmem + S::C_AS + 8 * s, ql = qh + 64, rh = qh + 128, rl = qh + 192;
      const uint32_t da = tmem + S::C_DS, db = da + 64;
      umma_ts(da, qh, bh, idS, s > 0 ? 1u : 0u);
      umma_ts(da, qh, bl, idS, 1u);
      umma_ts(da, ql, bh, idS, 1u);
      umma_ts(db, rh, bh, idS, s > 0 ? 1u : 0u);
      umma_ts(db, rh, bl, idS, 1u);
      umma_ts(db, rl, bh, idS, 1u);
    }
    umma_commit(&bar_s);
  };

  // rows >= 512 on the FP32 pipe (lanes 1..31 of the issuer warp, beside the MMA issue):
  // q / r of every frame for the update, and in the statistics pass their plane rows
  auto tail_rows = [&](int l, int nl, bool stats_pass) {
    for (int i = 0; i < ntail; ++i) {
      const int row = 2 * kPcRows + i;
      for (int n = l; n < kPcFrames; n += nl) {
        float lam = 0.0f;
#pragma unroll
        for (int k = 0; k < KP; ++k) lam = fmaf(Wt[i * KP + k], Hh[pc_off_h<KP>(n, k)], lam);
        const bool valid = n < nf;
        const float rr = rcp_approx(lam + eps);
        const float ve = (valid ? __ldg(fptr[n] + row) : 0.0f) + eps;
        Qt[i * kPcFrames + n] = valid ? ve * rr * rr : 0.0f;
        Rt[i * kPcFrames + n] = valid ? rr : 0.0f;
        if (stats_pass && rank == 1 && valid) divacc += is_term_fast(ve * rr);
      }
    }
  };
  auto tail_stats = [&](int l, int nl) {  // rank 1: the tail rows of the pair's statistics plane
    const int FP = (F + 3) & ~3;
    float* outA = a.stats + size_t(pair) * 2 * FP * KP;
    float* outB = outA + size_t(FP) * KP;
    for (int idx = l; idx < ntail * K; idx += nl) {
      const int i = idx / K, k = idx - i * K;
      float sa = 0.0f, sb = 0.0f;
      for (int n = 0; n < kPcFrames; ++n) {
        const float h = Hh[pc_off_h<KP>(n, k)];
        sa = fmaf(Qt[i * kPcFrames + n], h, sa);
        sb = fmaf(Rt[i * kPcFrames + n], h, sb);
      }
      outA[size_t(k) * FP + 2 * kPcRows + i] = sa;
      outB[size_t(k) * FP + 2 * kPcRows + i] = sb;
    }
  };

  const int passes = a.iters + 1;
  for (int pass = 0; pass < passes; ++pass) {
    const bool stats_pass = pass == a.iters;
    pass_no = pass;
    if (stats_pass) pdl_trigger();
    // ------------------------------------------------------------------ issuer (+ tail rows)
    if (warp == kPcIssueWarp) {  // tile 0 now; tile 1 by warp kPcA1Warp once it is done
      if (lane == 0) issue_phase_a(0);
      __syncwarp();
    }
    if (warp == kPcTailWarp && ntail > 0) {
      tail_rows(lane, 32, stats_pass);
      if (stats_pass && rank == 1 && a.stats) {
        __syncwarp();
        tail_stats(lane, 32);
      }
      __syncwarp();
    }
    if (stats_pass) {
      // h^T (hi | lo rows) for the statistics B operand, built while phase A runs; the slots are
      // free (the last update read the exchange buffer before the end-of-pass barrier)
      // item = (atom k = 8a + it % 8, frames 4jj ..): a quarter warp writes the 8 rows of one
      // core-matrix group (conflict-free float4 stores), its h reads are 4-way conflicted scalar
      // loads (the earlier row-major walk was 8- to 16-way conflicted on both sides, ~4k cycles)
      static_assert(S::HT_ROWS == KP2 + 8 && kPcFrames == 64, "h^T item map");
      for (int it = tid; it < (KP + 8) * (kPcFrames / 4); it += kPcThreads) {
        const int t8 = it & 7, jj = (it >> 3) & 15, k = ((it >> 7) << 3) + t8;
        if (k < KP) {
          float x[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) x[e] = Hh[pc_off_h<KP>(4 * jj + e, k)];
          *reinterpret_cast<float4*>(HT + pc_off_ht(k, 4 * jj)) = make_float4(x[0], x[1], x[2], x[3]);
          *reinterpret_cast<float4*>(HT + pc_off_ht(KP + k, 4 * jj)) =
              make_float4(tf32_lo(x[0]), tf32_lo(x[1]), tf32_lo(x[2]), tf32_lo(x[3]));
        } else {  // the 8 zero rows behind the lo half
          *reinterpret_cast<float4*>(HT + pc_off_ht(KP2 + t8, 4 * jj)) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      proxy_fence();
      __syncthreads();
      PC_MARK(31, 0);
    }
    // ------------------------------------------------------------------ epilogue warps
    if (warp < kPcEpiWarps) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int row = int(rank) * kPcRows + 128 * t + 32 * q + lane;
        const bool rowok = row < rowF;
        const float rowmask = rowok ? 1.0f : 0.0f;
        const float* v = vr[t];
        PC_MARK(2, t);
        mbar_wait(&bar_a[t], pass & 1);
        PC_MARK(3, t);
        tc_fence_after();
        if (t == 0 && warp == kPcA1Warp) {
          if (lane == 0) issue_phase_a(1);
          __syncwarp();
        }
        const uint32_t cA = tlane + S::C_DA + uint32_t(64 * t + 32 * hh);
        if (!stats_pass) {
          // slot sl = c & 1 last held chunk c - 2 (or chunk c + 6 of the previous pass)
          const int c = 4 * t + pc_quarter_chunk(t, q), sl = c & 1;
          PC_MARK(4, c);
          if (c >= 2)
            mbar_wait(&bar_empty[c - 2], pass & 1);
          else if (pass > 0)
            mbar_wait(&bar_empty[c + 6], (pass - 1) & 1);
          PC_MARK(5, c);
          float* op0 = slot + sl * kPcSlotFloats;
          float* op1 = op0 + kPcSlotFloats / 2;
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {  // 16 frames at a time (register budget: 3 warps / SMSP)
            float lam[16];
            tmem_ld<16>(cA + 16 * hf, lam);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float qv[4], rv[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                // rows past F must add nothing (rowmask 0); frames past nf only feed D_B rows
                // that are never read (v = 0 there: finite values)
                const int j = 16 * hf + 4 * i + e;
                const float rr = rcp_approx(lam[4 * i + e] + eps);
                rv[e] = rr * rowmask;
                qv[e] = (v[j] * rv[e]) * rr;
              }
              const int mq = 32 * hh + 16 * hf + 4 * i;
              const int oq = pc_off_st(mq, lane), orr = pc_off_st(64 + mq, lane);
              *reinterpret_cast<float4*>(op0 + oq) = make_float4(qv[0], qv[1], qv[2], qv[3]);
              *reinterpret_cast<float4*>(op0 + orr) = make_float4(rv[0], rv[1], rv[2], rv[3]);
              *reinterpret_cast<float4*>(op1 + oq) =
                  make_float4(tf32_lo(qv[0]), tf32_lo(qv[1]), tf32_lo(qv[2]), tf32_lo(qv[3]));
              *reinterpret_cast<float4*>(op1 + orr) =
                  make_float4(tf32_lo(rv[0]), tf32_lo(rv[1]), tf32_lo(rv[2]), tf32_lo(rv[3]));
            }
          }
          proxy_fence();
          mbar_arrive(&bar_full[c]);
          PC_MARK(6, c);
          if (warp == t) {  // this tile's chunks, in order (ours first)
            if (lane == 0) issue_chunks(4 * t, 4, pass);
            __syncwarp();
          }

        } else {
          // statistics pass: q / r (hi | lo) of this tile into TMEM as the A operands (A_S
          // overlays W_A: both tiles' phase-A MMAs must be done; for tile 1 the tile-0
          // statistics MMAs are, since their D_S was drained below first)
          PC_MARK(32, t);
          if (t == 0) {
            mbar_wait(&bar_a[1], pass & 1);
            tc_fence_after();
          }
          PC_MARK(33, t);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            float lam[16], x[16];
            tmem_ld<16>(cA + 16 * hf, lam);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = 32 * hh + 16 * hf + j;
              const bool valid = rowok && n < nf;
              const float rr = rcp_approx(lam[j] + eps);
              const float ve = v[16 * hf + j];
              if (valid) divacc += is_term_fast(ve * rr);
              x[j] = valid ? ve * rr * rr : 0.0f;  // q
              lam[j] = valid ? rr : 0.0f;          // r
            }
            const uint32_t ca = tlane + S::C_AS + uint32_t(32 * hh + 16 * hf);
            tmem_st<16>(ca, x);
            tmem_st<16>(ca + 128, lam);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              x[j] = tf32_lo(x[j]);
              lam[j] = tf32_lo(lam[j]);
            }
            tmem_st<16>(ca + 64, x);
            tmem_st<16>(ca + 192, lam);
          }
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bar_sa);
          PC_MARK(10, t);
          if (warp == kPcIssueWarp) {
            if (lane == 0) issue_stats(t);
            __syncwarp();
          }

          // statistics of this tile -> the pair's plane (rows of this CTA)
          mbar_wait(&bar_s, t & 1);
          PC_MARK(11, t);
          tc_fence_after();
          const int FP = (F + 3) & ~3;
          float* out = a.stats ? a.stats + size_t(pair) * 2 * FP * KP : nullptr;
#pragma unroll
          for (int ab = 0; ab < 2; ++ab) {  // sa, then sb
            float sv[KH];
            tmem_ld_n<KH>(tlane + S::C_DS + uint32_t(64 * ab + KH * hh), sv);
            tmem_ld_wait();
            if (out && rowok) {
              float* o = out + size_t(ab) * FP * KP + size_t(KH * hh) * FP + row;
              const int kend = min(KH, K - KH * hh);
#pragma unroll
              for (int j = 0; j < KH; ++j, o += FP)
                if (j < kend) *o = sv[j];
            }
          }
          tc_fence_before();
        }
      }
    }
    if (stats_pass) break;
    // ------------------------------------------------------------------ h update
    // all warps: D_B -> this CTA's num / den partials -> exchange -> h *= sqrt(num / den)
    PC_MARK(7, 0);
    mbar_wait(&bar_b, pass & 1);  // (every warp is an epilogue warp)
    tc_fence_after();
    PC_MARK(8, 0);
    // Frame ownership: rank r updates frames [32 r, 32 r + 32) only.  It needs the peer's num / den
    // partials of those frames (half of the old exchange volume each way), and afterwards sends
    // its block of h (hi copy, one contiguous 7 KB piece of the K-major layout) to the peer, which
    // rebuilds the lo copy: two short DSMEM hops instead of one long one, and half the update.
    const int own0 = 32 * int(rank), ownc = max(0, min(32, nf - own0));
    const int peer0 = 32 * int(peer), peerc = max(0, min(32, nf - peer0));
    if (tid == 0) {
      mbar_expect_tx(&bar_xfull, uint32_t(2 * ownc * XS * sizeof(float)));  // the peer's partials of our frames
      mbar_expect_tx(&bar_h, uint32_t(4 * (KP / 4) * 32 * sizeof(float)));  // and, later, its h block
      mbar_arrive_remote(&bar_pfree, peer);  // our phase B is done: our slots may take them
    }
    {
      // lane m = 32q + lane of D_B: m < 64 -> num of frame m, else den of frame m - 64;
      // num (or den) partial = [q|r]_hi W_hi + [q|r]_lo W_hi (columns k) + [q|r]_hi W_lo (KP + k)
      const int m = 32 * q + lane, nd = m >> 6, n = m & 63;
      float part[KH];
      const uint32_t cb = tlane + S::C_DB + uint32_t(KH * hh);
      tmem_ld_n<KH>(cb, part);
      tmem_ld_wait();
#pragma unroll
      for (int j0 = 0; j0 < KH; j0 += 8) {  // the W_lo columns, 8 at a time (register budget)
        float y[8];
        if (j0 + 8 <= KH) tmem_ld<8>(cb + KP + j0, y);
        else tmem_ld<4>(cb + KP + j0, y);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < KH) part[j0 + j] += y[j];
      }
      tc_fence_before();
      float* dst = XB + ((int(rank) * 2 + nd) * kPcFrames + n) * XS + KH * hh;
#pragma unroll
      for (int j = 0; j < KH; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(part[j], part[j + 1], part[j + 2], part[j + 3]);
    }
    proxy_fence();  // the partials, for the bulk copy (async proxy)
    __syncthreads();
    PC_MARK(16, 0);
    if (tid == 0) {  // our partials of the peer's frames -> the same place in the peer's slots
      const uint32_t xrow_bytes = uint32_t(peerc * XS * sizeof(float));
      mbar_wait_cluster(&bar_pfree, pass & 1);  // the peer's phase B is done: its slots are free
      PC_MARK(9, 0);
      const uint32_t rbar = dsmem_addr(&bar_xfull, peer);
      if (peerc > 0) {
#pragma unroll
        for (int nd = 0; nd < 2; ++nd) {
          const float* src = XB + ((int(rank) * 2 + nd) * kPcFrames + peer0) * XS;
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  dsmem_addr(src, peer)),
              "r"(smem_addr(src)), "r"(xrow_bytes), "r"(rbar)
              : "memory");
        }
      }
    }
    mbar_wait_cluster(&bar_xfull, pass & 1);  // the peer's partials of our frames have landed
    PC_MARK(12, 0);
    {
      // our frames' h, fixed order (rank 0 + rank 1 + tail); thread (frame own0 + tid % 32, k
      // quads g8, g8 + 8, ...) loads all its operands first.  A quarter warp touches 8 consecutive
      // frames: conflict-free in the exchange rows (stride XS) and in the h core matrices.
      // Frames >= nf and atoms >= K keep h = 0.
      constexpr int NQ = KP / 4, NI = (NQ + 7) / 8;
      const int n = own0 + (tid & 31), g8 = tid >> 5, nk4 = (K + 3) >> 2;
#pragma unroll
      for (int i0 = 0; i0 < NI; i0 += 2) {
        if (n >= nf) break;
        float4 a0[2], a1[2], b0[2], b1[2], hq[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int kq = g8 + 8 * (i0 + i), k4 = 4 * kq;
          if (i0 + i < NI && kq < nk4) {
            a0[i] = *reinterpret_cast<const float4*>(XB + (0 * kPcFrames + n) * XS + k4);
            a1[i] = *reinterpret_cast<const float4*>(XB + (2 * kPcFrames + n) * XS + k4);
            b0[i] = *reinterpret_cast<const float4*>(XB + (1 * kPcFrames + n) * XS + k4);
            b1[i] = *reinterpret_cast<const float4*>(XB + (3 * kPcFrames + n) * XS + k4);
            hq[i] = *reinterpret_cast<const float4*>(Hh + pc_off_h<KP>(n, k4));
          }
        }
        PC_MARK(34, i0);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int kq = g8 + 8 * (i0 + i), k4 = 4 * kq;
          if (i0 + i >= NI || kq >= nk4) continue;
          float num[4] = {a0[i].x + a1[i].x, a0[i].y + a1[i].y, a0[i].z + a1[i].z, a0[i].w + a1[i].w};
          float den[4] = {b0[i].x + b1[i].x, b0[i].y + b1[i].y, b0[i].z + b1[i].z, b0[i].w + b1[i].w};
#pragma unroll
          for (int r = 0; r < kPcMaxTail; ++r) {  // (unrolled: no runtime-trip loop in the update)
            if (r >= ntail) break;
            const float qt = Qt[r * kPcFrames + n], rt = Rt[r * kPcFrames + n];
            const float4 wt = *reinterpret_cast<const float4*>(Wt + r * KP + k4);
            const float w4[4] = {wt.x, wt.y, wt.z, wt.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              num[e] = fmaf(w4[e], qt, num[e]);
              den[e] = fmaf(w4[e], rt, den[e]);
            }
          }
          float hv[4] = {hq[i].x, hq[i].y, hq[i].z, hq[i].w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (k4 + e < K) hv[e] = hv[e] * sqrt_approx(num[e] * rcp_approx(den[e]));
          const int o = pc_off_h<KP>(n, k4);
          *reinterpret_cast<float4*>(Hh + o) = make_float4(hv[0], hv[1], hv[2], hv[3]);
          *reinterpret_cast<float4*>(Hl + o) =
              make_float4(tf32_lo(hv[0]), tf32_lo(hv[1]), tf32_lo(hv[2]), tf32_lo(hv[3]));
        }
      }
    }
    PC_MARK(17, 0);
    {
      // our h block (hi copy) -> the peer; its block -> our Hh, lo copy rebuilt here
      constexpr int kBlk = 4 * (KP / 4) * 32;  // floats of 32 frames of the K-major h layout
      proxy_fence();  // the updated block, for the bulk copy (async proxy)
      __syncthreads();
      if (tid == 0) {
        const float* src = Hh + int(rank) * kBlk;
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                dsmem_addr(src, peer)),
            "r"(smem_addr(src)), "r"(uint32_t(kBlk * sizeof(float))), "r"(dsmem_addr(&bar_h, peer))
            : "memory");
      }
      mbar_wait_cluster(&bar_h, pass & 1);
      for (int i = tid; i < kBlk; i += kPcThreads) Hl[int(peer) * kBlk + i] = tf32_lo(Hh[int(peer) * kBlk + i]);
    }
    PC_MARK(17, 0);
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    PC_MARK(18, 0);
  }

  PC_MARK(13, 0);
  // divergence partial of this CTA (fixed order)
  if (a.divpart) {
    const double d = warp_sum_d(double(divacc));
    if (lane == 0) red[warp] = d;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kPcThreads / 32; ++w) s += red[w];
      a.divpart[2 * pair + int(rank)] = s;
    }
  }
  // final h of the frames this CTA owns (rank r: frames 32r ..)
  const int own0 = 32 * int(rank), nown = max(0, min(32, nf - own0));
  if (a.h0_mode == 1 && a.write_store) {
    // warm store (kernels.cuh warm_put): thread (frame own0 + tid / 8, k = tid % 8 + 8 j) issues every
    // U / P load of its cells before any store (one HBM latency instead of one per cell)
    constexpr int NJ = KP / 8;
    const int nl = tid >> 3, k0 = tid & 7, n = own0 + nl;
    const bool fr = nl < nown;
    const int64_t col = fr ? colv[n] : 0;
    const uint32_t tag = fr ? tagv[n] : 0u;
    const double* urow = a.U + size_t(col) * K;
    const double* prow = a.P + size_t(tag) * K;
    const double* pnow = a.P + size_t(a.c_now) * K;
    double u[NJ], pt[NJ], pn[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = k0 + 8 * j;
      const bool ok = fr && k < K;
      u[j] = ok ? urow[k] : 0.0;
      pt[j] = ok ? prow[k] : 1.0;
      pn[j] = ok ? pnow[k] : 1.0;
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int k = k0 + 8 * j;
      if (!fr || k >= K) continue;
      const float h = Hh[pc_off_h<KP>(n, k)];
      const double h0 = u[j] * (pn[j] / pt[j]);
      a.U[size_t(col) * K + k] = h0 < double(kWarmFloor) ? h0 * (double(h) / double(kWarmFloor)) : double(h);
      if (a.Hout) a.Hout[size_t(n0 + n) * K + k] = h;
    }
    __syncthreads();  // every U write of this CTA has used its column's old tag
    if (tid < nown) a.T[colv[own0 + tid]] = a.c_now;
  } else {
    write_final_h(a, n0 + own0, nown, [&](int n, int k) { return Hh[pc_off_h<KP>(own0 + n, k)]; });
  }
  tc_fence_before();
  __syncthreads();
  PC_MARK(14, 0);
  cluster_arrive();  // no DSMEM access reaches an exited CTA
  cluster_wait();
  PC_MARK(15, 0);
#ifdef ISNMF_PC_TRACE
  if (g_pc_trace && blockIdx.x < 2 && (threadIdx.x & 31) == 0)
    for (int i = 0; i < pc_n; ++i)
      g_pc_trace[4096 + (blockIdx.x * 10 + (threadIdx.x >> 5)) * 512 + i] = pc_log[(threadIdx.x >> 5) * kPcLog + i];
#endif
  if (warp == kPcIssueWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace isnmf_dev

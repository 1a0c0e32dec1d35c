// Host side of the B200 IS-NMF engine: device contexts, launch orchestration,
// H2D streaming and the extern "C" boundary declared in include/isnmf_b200.h.
//
// The online path follows online_resume / online_step / dictionary_commit
// (reference proj/include/isnmf/online.hpp:318-407): frames are processed in
// blocks that never cross a mini-batch boundary; a block is one K1 launch
// (all frames of the block solved and their statistics formed in parallel —
// W is frozen inside a mini-batch, so this equals the sequential per-sample
// loop up to fp rounding), one K2 launch (fixed-order reduction into pending,
// plus the elementwise commit on the beta-th sample) and, on a commit, one K3
// launch (column renormalisation, trace point, eta stop rule).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/isnmf_b200.h"
#include "kernels.cuh"
#include "kernels_large.cuh"
#include "kernels_large_tc.cuh"
#include "kernels_mma.cuh"
#include "kernels_tc.cuh"
#include "stft.cuh"

namespace isnmf_dev {
// kernel instantiations in separate translation units (compiled in parallel):
// K1M csrc/mma_table.cu, FFMA K1 csrc/ffma_table.cu, K1L / K1T csrc/large_table.cu
void (*mma_kernel(int nw, int fg, int kb, bool multi))(const SolveArgs);
void (*ffma_kernel(int tk, int tn))(const SolveArgs);
void (*large_kernel(int mbw, int nb))(const SolveArgs);
void (*large_tc_kernel(int nb))(const SolveArgs);
void (*pair_kernel(int kb))(const SolveArgs);
size_t pair_smem(int kb);
int pc_trace_set(unsigned long long* dev_ptr);
}  // namespace isnmf_dev
using namespace isnmf_dev;

namespace {
#ifdef ISNMF_PHASE_PROF
long long* g_work_prof = nullptr;  // K1M timeline of the batch / stateless passes (CTA 0, last tile)
#endif


thread_local std::string g_err;
unsigned long long* g_trace_host = nullptr;  // isnmf_debug_pc_trace (ISNMF_PC_TRACE builds)

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return fail(ISNMF_E_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                      \
  } while (0)

#define TRY(x)             \
  do {                     \
    int rc_ = (x);         \
    if (rc_) return rc_;   \
  } while (0)

// ---------------------------------------------------------------------------
// Kernel family: solve_kernel<TK, TN> handles K <= 4*TK atoms and 4*TN frames
// per CTA.  The variant is picked per context so that one mini-batch fills the
// 148 SMs in a single wave.
// ---------------------------------------------------------------------------
using SolveFn = void (*)(const SolveArgs);
struct Variant {
  int TK, TN;
  SolveFn fn;
  size_t (*smem)(int);
  size_t static_smem;
  bool configured;
};

#define VAR(tk, tn) {tk, tn, ffma_kernel(tk, tn), &SolveShape<tk, tn>::smem_bytes, 0, false}
#ifdef ISNMF_MIN_VARIANTS  // fast experimental builds: the headline shape only
Variant g_variants[] = {VAR(13, 7), VAR(5, 2), VAR(3, 1)};
#else
Variant g_variants[] = {
    VAR(1, 1), VAR(1, 2), VAR(1, 4), VAR(1, 7), VAR(1, 8),       //
    VAR(2, 1), VAR(2, 2), VAR(2, 4), VAR(2, 7), VAR(2, 8),       //
    VAR(3, 1), VAR(3, 2), VAR(3, 4), VAR(3, 7), VAR(3, 8),       //
    VAR(5, 1), VAR(5, 2), VAR(5, 4), VAR(5, 7), VAR(5, 8),       //
    VAR(8, 1), VAR(8, 2), VAR(8, 4), VAR(8, 7), VAR(8, 8),       //
    VAR(13, 1), VAR(13, 2), VAR(13, 4), VAR(13, 7), VAR(13, 8),  //
    VAR(16, 1), VAR(16, 2), VAR(16, 4), VAR(16, 7),              //
};
#endif
#undef VAR
constexpr int kNumVariants = sizeof(g_variants) / sizeof(g_variants[0]);

int device_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                  cudaSuccess)
      sms = 148;
  }
  return sms;
}

int smem_optin() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) v = 232448;
  }
  return v;
}

int ws_for(int KP) { return ((KP / 4) % 2 == 1) ? KP : KP + 4; }
bool fold_configured = false;

// K2: one cluster of kFoldCluster CTAs per column of W.
// Programmatic dependent launch: the online engine chains K1 -> K2 -> K1 with
// programmatic stream serialization so each launch overlaps the previous grid's
// tail (the kernels call griddepcontrol.wait before touching its outputs).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("ISNMF_PDL");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}
template <class... P, class... A>
cudaError_t launch_pdl(void (*fn)(P...), int grid, int block, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, std::forward<A>(args)...);
}

// launch on 2-CTA clusters (K1P), with programmatic dependent launch when pdl
template <class... P, class... A>
cudaError_t launch_cluster2(void (*fn)(P...), int grid, int block, size_t smem, cudaStream_t s, bool pdl,
                            A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fn, std::forward<A>(args)...);
}

// Growth factor of the host-frame chunk ramp.  A chunk of r*s frames must copy in
// about the compute time of the previous s frames: copy/compute per frame is
// ~ (4F B / 50 GB/s) / (6FK(I+1) flop / 45 TFLOP/s) = 600 / (K (I+1)), so r =
// 0.95 (K (I+1)) / 600, clamped to [1.125, 4] (config 3: 1.125; config 4: 3.6 —
// each chunk boundary also costs time, so compute-heavy shapes grow fast).
// ISNMF_RAMP overrides it (A/B measurement only).
double ramp_factor(int K, int iters) {
  static const double env = [] {
    const char* e = getenv("ISNMF_RAMP");
    return e ? atof(e) : 0.0;
  }();
  if (env > 1.0) return env;
  const double r = 0.95 * double(K) * double(iters + 1) / 600.0;
  return r < 1.125 ? 1.125 : (r > 4.0 ? 4.0 : r);
}

int launch_fold(const FoldArgs& f, cudaStream_t s, bool pdl = false) {
  const size_t smem = fold_smem_bytes(f.F);
  if (smem + 1024 > size_t(smem_optin()))
    return fail(ISNMF_E_UNSUPPORTED, "F=%d too large for the commit kernel", f.F);
  if (!fold_configured) {
    CU(cudaFuncSetAttribute(fold_commit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin() - 1024));
    fold_configured = true;
  }
  if (pdl && pdl_enabled())
    CU(launch_pdl(fold_commit_kernel, f.K * kFoldCluster, kFoldThreads, smem, s, f));
  else
    fold_commit_kernel<<<f.K * kFoldCluster, kFoldThreads, smem, s>>>(f);
  return 0;
}
int fold_parts(int K) { return 2 * K * kFoldCluster; }
// Divisor of the shrinking tail of the host-frame chunk schedule (online_enqueue): 8 for
// shapes whose copy and compute are balanced, 4 for compute-bound ones.  ISNMF_TAIL overrides.
int tail_div(int K, int iters) {
  static const int env = [] {
    const char* e = getenv("ISNMF_TAIL");
    return e ? atoi(e) : 0;
  }();
  if (env > 1) return env;
  return ramp_factor(K, iters) <= 1.5 ? 8 : 4;
}

int padded_f(int F) { return (F + 3) & ~3; }

// Picks the variant for (F, K, frames per mini-batch).
int pick_variant(int64_t F, int64_t K, int64_t frames, Variant** out, int* WS, size_t* smem) {
  const int tk_need = int((K + 3) / 4);
  const int64_t per_cta = (frames + device_sms() - 1) / device_sms();
  const int tn_need = int(std::min<int64_t>(8, std::max<int64_t>(1, (per_cta + 3) / 4)));
  Variant* best = nullptr;
  for (auto& v : g_variants) {
    if (v.TK < tk_need || v.TN < tn_need) continue;
    if (!best || v.TK < best->TK || (v.TK == best->TK && v.TN < best->TN)) best = &v;
  }
  if (!best) {  // TN capped by the table: take the largest TN for the smallest TK
    for (auto& v : g_variants) {
      if (v.TK < tk_need) continue;
      if (!best || v.TK < best->TK || (v.TK == best->TK && v.TN > best->TN)) best = &v;
    }
  }
  if (!best) return 1;  // no register-tiled variant: caller uses the generic kernel
  const int w = ws_for(4 * best->TK);
  if (!best->configured) {
    cudaFuncAttributes at;
    CU(cudaFuncGetAttributes(&at, best->fn));
    best->static_smem = at.sharedSizeBytes;
    CU(cudaFuncSetAttribute(best->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            smem_optin() - int(best->static_smem)));
    best->configured = true;
  }
  const size_t sm = best->smem(int(F));
  if (sm + best->static_smem > size_t(smem_optin())) return 1;  // W does not fit: generic kernel
  *out = best;
  *WS = w;
  *smem = sm;
  return 0;
}

// Solve-kernel choice for (F, K, frames per batch): a register-tiled variant when
// W fits shared memory, else the generic streaming kernel.
// Tensor-pipe kernel for 64 < K <= 256 (config 4): [MBW - 1][NB - 1]
using LargeFn = void (*)(const SolveArgs);
size_t large_smem(int mbw, int nb) {  // = LargeShape<mbw, nb>::smem_bytes()
  const int KP = 128 * mbw, NT = 8 * nb, FMB = (NT + 15) / 16;
  return sizeof(float) * (size_t(16 * FMB) * (KP + 4) + 3 * size_t(kLgChunk) * (KP + 4) + 2 * size_t(kLgChunk) * 136);
}
static_assert(LargeShape<2, 7>::smem_bytes() == sizeof(float) * (64 * 260 + 3 * 32 * 260 + 2 * 32 * 136),
              "large_smem() mirrors LargeShape::smem_bytes()");
bool large_configured[2][8] = {};
// tcgen05 variant (128 < K <= 256): large_tc_kernel(nb)
size_t large_tc_smem(int nb) {
  switch (nb) {
    case 1: return LargeTcShape<1>::smem_bytes();
    case 2: return LargeTcShape<2>::smem_bytes();
    case 3: return LargeTcShape<3>::smem_bytes();
    case 4: return LargeTcShape<4>::smem_bytes();
    case 5: return LargeTcShape<5>::smem_bytes();
    case 6: return LargeTcShape<6>::smem_bytes();
    default: return LargeTcShape<7>::smem_bytes();
  }
}
bool large_tc_configured[7] = {};
bool tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("ISNMF_TC");
    return e ? atoi(e) != 0 : true;
  }();
  return on;
}

// K1M: all-tensor-pipe solve for K <= 56 (instantiated in csrc/mma_table.cu)
size_t mma_smem(int kb, int fg, int nw, int F, bool pair2 = false) {
  const int KP = 8 * kb, NT = 16 * fg, WS = mm_stride(KP), HT = mm_stride(NT);
  const size_t F16 = size_t((F + 15) & ~15), red = size_t(nw) * 8 * kb * 32, ht = size_t(KP) * HT;
  const size_t xr = pair2 ? size_t(2 * 2 * 32 * kb * 8) : 0;  // K1P exchange (MmShape::XR_FLOATS)
  return sizeof(float) * (F16 * WS + size_t(fg) * kb * 256 + (red > ht ? red : ht) + xr);
}
static_assert(MmShape<7, 2, 12>::WS == 56 && MmShape<7, 2, 12>::HT == 40, "K1M strides");
static_assert(MmShape<7, 2, 12>::HF == 2 * 7 * 256, "K1M fragment copy = mma_smem()");
bool mma_configured[2][2][7] = {};
// ISNMF_MMA=0 keeps K <= 56 on the FFMA register-tile kernels; otherwise K1M is
// used when a CTA gets at least ISNMF_MMA_MIN frames (default 1)
int mma_warps() {  // ISNMF_MMA_WARPS = 8 or 12 (default 12 when the CTA fits; 16 measured slower at config 1)
  static const int v = [] {
    const char* e = getenv("ISNMF_MMA_WARPS");
    return (e && atoi(e) == 8) ? 8 : 12;
  }();
  return v;
}
int mma_min_frames() {
  static const int v = [] {
    const char* e = getenv("ISNMF_MMA");
    if (e && atoi(e) == 0) return 1 << 30;
    const char* m = getenv("ISNMF_MMA_MIN");
    return m ? atoi(m) : 1;
  }();
  return v;
}

struct SolvePlan {
  bool tiled = false;       // the kernel loops over frame tiles (K1M): any grid <= tiles works
  bool pair = false;        // K1C: one 2-CTA cluster per NT frames (grid = 2 x blocks, two divergence partials each)
  bool mpair = false;       // K1P: K1M on 2-CTA clusters (rows split), same grid / partial counts as K1C
  LargeFn large = nullptr;  // tensor-pipe kernels (large K, or the resident-dictionary variant)
  LargeFn multi = nullptr;  // K1M's multi-tile instantiation (grid < tiles)
  int threads = 0;          // block size of `large`
  Variant* var = nullptr;  // nullptr: generic
  int NT = 0, KP = 0, WS = 0;
  size_t smem = 0;
  int chain = 0;            // K1T: CTAs per statistics plane (kernels_large_tc.cuh, statistics chain)
};

bool generic_configured = false;

// K1T statistics chain: ISNMF_CHAIN = CTAs per plane (default 8; 0 or 1: one plane per CTA)
int chain_len() {
  static const int v = [] {
    const char* e = getenv("ISNMF_CHAIN");
    return e ? atoi(e) : 8;
  }();
  return v;
}

// K1C (csrc/kernels_tc.cuh): ISNMF_K1C = 0 off, 1 (default) for mini-batches that give a
// pair of SMs >= 40 frames, 2 at any size (tests)
int pair_mode(int flags = 0) {
  static const int v = [] {
    const char* e = getenv("ISNMF_K1C");
    return e ? atoi(e) : 1;
  }();
  if (flags & ISNMF_FLAG_NO_PAIR) return 0;
  if (flags & ISNMF_FLAG_PAIR) return 2;
  return v;
}
bool pair_configured[8] = {};
// K1P (K1M rows split over a 2-CTA cluster): ISNMF_K1P = 0 off, 1 (default) for online
// mini-batches whose K1M CTAs would hold one frame group (<= 16 frames per CTA)
int mpair_mode(int flags = 0) {
  static const int v = [] {
    const char* e = getenv("ISNMF_K1P");
    return e ? atoi(e) : 1;
  }();
  if (flags & ISNMF_FLAG_NO_PAIR) return 0;
  return v;
}

int plan_solve(int64_t F, int64_t K, int64_t frames, SolvePlan* plan, bool force_generic = false,
               bool allow_pair = false, int flags = 0) {
  Variant* v = nullptr;
  int WS = 0;
  size_t sm = 0;
  const int pmode = pair_mode(flags);
  if (allow_pair && !force_generic && pmode != 0 && K >= 17 && K <= 56 && F > 384 &&
      F <= 2 * kPcRows + kPcMaxTail) {
    const int pairs = device_sms() / 2;
    const int64_t per = (frames + pairs - 1) / pairs;
    const int np = int(std::min<int64_t>(kPcFrames, std::max<int64_t>(8, (per + 7) & ~int64_t(7))));
    const int kb = int((K + 7) / 8);
    const size_t smem = pair_smem(kb);
    if ((per >= 40 || pmode == 2) && smem + 2048 <= size_t(smem_optin())) {
      if (!pair_configured[kb]) {
        CU(cudaFuncSetAttribute(pair_kernel(kb), cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        pair_configured[kb] = true;
      }
      plan->large = pair_kernel(kb);
      plan->pair = true;
      plan->threads = kPcThreads;
      plan->var = nullptr;
      plan->NT = np;
      plan->KP = 8 * kb;
      plan->WS = 8 * kb;
      plan->smem = smem;
      return 0;
    }
  }
  if (!force_generic && K >= 1 && K <= 56) {
    const int64_t per_cta = (frames + device_sms() - 1) / device_sms();
    // one frame group (<= 16 frames per CTA): fill it.  A K1M pass over one frame group costs
    // the same at 1 and 16 frames (the MMA tile is 16 frames either way), and fewer CTAs mean
    // fewer statistics planes for K2 to fold (config 1: 143 -> 63 planes, 17.8 -> 15.9 us).
    // ISNMF_MMA_NT overrides the floor (A/B measurement only).
    static const int nt_min = [] {
      const char* e = getenv("ISNMF_MMA_NT");
      return e ? atoi(e) : 16;
    }();
    const int nt = int(std::min<int64_t>(32, std::max<int64_t>(std::max(1, per_cta <= 16 ? nt_min : 1), per_cta)));
    const int kb = int((K + 7) / 8), fg = nt > 16 ? 2 : 1;
    int nw = mma_warps();
    // K1P: one frame group per pair of SMs (online, enough SMs for every pair)
    const int pairs = int((frames + nt - 1) / nt);
    const bool mp = allow_pair && !force_generic && fg == 1 && nw == 12 && mpair_mode(flags) != 0 &&
                    2 * pairs <= device_sms();
    if (nw == 12 && mma_smem(kb, fg, 12, int(F), mp) + 2048 > size_t(smem_optin())) nw = 8;
    const size_t smem = mma_smem(kb, fg, nw, int(F), mp && nw == 12);
    const int wi = nw == 12 ? 1 : 0;
    if (nt >= mma_min_frames() && smem + 2048 <= size_t(smem_optin())) {
      if (!mma_configured[wi][fg - 1][kb - 1]) {
        for (bool multi : {false, true})
          CU(cudaFuncSetAttribute(mma_kernel(nw, fg, kb, multi), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_optin() - 2048));
        mma_configured[wi][fg - 1][kb - 1] = true;
      }
      plan->large = mma_kernel(nw, fg, kb, false);
      plan->multi = mma_kernel(nw, fg, kb, true);
      plan->tiled = true;
      plan->mpair = mp && nw == 12;
      plan->threads = 32 * nw;
      plan->var = nullptr;
      plan->NT = nt;
      plan->KP = 8 * kb;
      plan->WS = mm_stride(8 * kb);
      plan->smem = smem;
      return 0;
    }
  }
  const int rc = force_generic ? 1 : pick_variant(F, K, frames, &v, &WS, &sm);
  if (rc == 0) {
    plan->var = v;
    plan->NT = 4 * v->TN;
    plan->KP = 4 * v->TK;
    plan->WS = WS;
    plan->smem = sm;
    return 0;
  }
  if (rc != 1) return rc;
  const int64_t per_cta = (frames + device_sms() - 1) / device_sms();
  if (!force_generic && K > 64 && K <= 256) {
    const int nb = int(std::min<int64_t>(8, std::max<int64_t>(1, (per_cta + 7) / 8)));
    const int mbw = K <= 128 ? 1 : 2;
    if (mbw == 2 && nb <= 7 && tc_enabled()) {  // phase B on tcgen05
      const size_t smem = large_tc_smem(nb);
      if (smem + 2048 <= size_t(smem_optin())) {
        if (!large_tc_configured[nb - 1]) {
          CU(cudaFuncSetAttribute(large_tc_kernel(nb), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem_optin() - 2048));
          large_tc_configured[nb - 1] = true;
        }
        plan->large = large_tc_kernel(nb);
        plan->threads = kTcThreads;
        plan->chain = (F + kTcRows - 1) / kTcRows + 2 < int64_t(kTcChainSpan) ? chain_len() : 0;
        plan->var = nullptr;
        plan->NT = 8 * nb;
        plan->KP = 256;
        plan->WS = ws_for(256);
        plan->smem = smem;
        return 0;
      }
    }
    const size_t smem = large_smem(mbw, nb);
    if (smem + 2048 <= size_t(smem_optin())) {
      if (!large_configured[mbw - 1][nb - 1]) {
        CU(cudaFuncSetAttribute(large_kernel(mbw, nb), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin() - 2048));
        large_configured[mbw - 1][nb - 1] = true;
      }
      plan->large = large_kernel(mbw, nb);
      plan->threads = kLgThreads;
      plan->var = nullptr;
      plan->NT = 8 * nb;
      plan->KP = 128 * mbw;
      plan->WS = ws_for(128 * mbw);
      plan->smem = smem;
      return 0;
    }
  }
  int nt = int(std::min<int64_t>(64, std::max<int64_t>(1, per_cta)));
  while (nt > 1 && K * nt > int64_t(kGenThreads) * kGenMaxPairs) --nt;
  if (K * nt > int64_t(kGenThreads) * kGenMaxPairs)
    return fail(ISNMF_E_UNSUPPORTED, "K=%lld too large for the generic kernel", (long long)K);
  const GenShape G(nt, int(K));
  const size_t smem = G.smem_floats() * sizeof(float);
  if (!generic_configured) {
    CU(cudaFuncSetAttribute(solve_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin() - 2048));
    generic_configured = true;
  }
  if (smem + 2048 > size_t(smem_optin()))
    return fail(ISNMF_E_UNSUPPORTED, "K=%lld: generic kernel needs %zu B of shared memory", (long long)K, smem);
  plan->var = nullptr;
  plan->NT = nt;
  plan->KP = G.KP;
  plan->WS = G.WS;
  plan->smem = smem;
  return 0;
}

void launch_solve(const SolvePlan& p, int nblk, const SolveArgs& args, cudaStream_t s, bool pdl = false) {
  SolveArgs a = args;
  a.cta_frames = p.NT;
  const LargeFn large = (p.multi && int64_t(nblk) * p.NT < a.nframes) ? p.multi : p.large;
  if (p.pair || p.mpair) nblk *= 2;  // one 2-CTA cluster per block of NT frames
  a.pair2 = p.mpair ? 1 : 0;
  if (p.mpair)
    launch_cluster2(p.large, nblk, p.threads, p.smem, s, pdl && pdl_enabled(), a);
  else if (large && pdl && pdl_enabled())
    launch_pdl(large, nblk, p.threads, p.smem, s, a);
  else if (large)
    large<<<nblk, p.threads, p.smem, s>>>(a);
  else if (p.var && pdl && pdl_enabled())
    launch_pdl(p.var->fn, nblk, kThreads, p.smem, s, a);
  else if (p.var)
    p.var->fn<<<nblk, kThreads, p.smem, s>>>(a);
  else
    solve_generic_kernel<<<nblk, kGenThreads, p.smem, s>>>(a, p.NT);
}

template <class T>
int dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  CU(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
  return 0;
}

void dfree(void* p) {
  if (p) cudaFree(p);
}

// Set-up copies/memsets go through the legacy default stream: cudaMemset is
// asynchronous and a pageable cudaMemcpy H2D may return before its DMA lands,
// while the engine's streams are non-blocking (no implicit ordering).  Every
// entry point that stages state that way settles the legacy stream before
// device work on its own streams may read it.
int settle() {
  CU(cudaStreamSynchronize(cudaStreamLegacy));
  return 0;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

__global__ void fill_u32(uint32_t* p, int64_t n, uint32_t v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}
__global__ void fill_f64(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}
// batch_train's H: fp64 (host layout) <-> the solver's fp32, on the device; *bad is set when
// an entry is not strictly positive (NonPositiveInit)
__global__ void h_to_f32(const double* src, float* dst, int64_t n, unsigned int* bad) {
  unsigned int b = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double x = src[i];
    if (!(x > 0.0)) b = 1;
    dst[i] = float(x);
  }
  if (b) atomicOr(bad, 1u);
}
__global__ void h_to_f64(const float* src, double* dst, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = double(src[i]);
}
// U[col] <- current value (U * P[c]/P[T]), T <- c_new.
__global__ void warm_rebase(double* U, uint32_t* T, const double* P, int64_t n, int K, uint32_t c_old,
                            uint32_t c_new) {
  for (int64_t col = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; col < n; col += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t tag = T[col];
    for (int k = 0; k < K; ++k) U[col * K + k] *= P[size_t(c_old) * K + k] / P[size_t(tag) * K + k];
    T[col] = c_new;
  }
}
__global__ void warm_read(const double* U, const uint32_t* T, const double* P, int64_t n, int K, uint32_t c,
                          double* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n * K; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t col = i / K;
    const int k = int(i - col * K);
    out[i] = U[i] * (P[size_t(c) * K + k] / P[size_t(T[col]) * K + k]);
  }
}
__global__ void mark_origin(DevState* st) { st->origin_ns = globaltimer_ns(); }

int status_to_code(unsigned int s, const char* where, unsigned long long t) {
  if (s & ST_NONPOS_INIT) return fail(ISNMF_E_NON_POSITIVE_INIT, "%s: h0 must be positive (t = %llu)", where, t);
  if (s & ST_INCONSISTENT) return fail(ISNMF_E_INCONSISTENT_STATS, "update_w: a > 0 with b = 0 (t = %llu)", t);
  if (s & ST_NONFINITE_W)
    return fail(ISNMF_E_NUMERICAL_FAILURE, "%s: non-finite dictionary update at t = %llu", where, t);
  if (s & ST_ZERO_COLUMN) return fail(ISNMF_E_ZERO_COLUMN, "rescale_dictionary: dead atom (t = %llu)", t);
  if (s & ST_DIVERGED) return fail(ISNMF_E_DIVERGED_OBJECTIVE, "%s: objective increased", where);
  if (s & ST_CHAIN_TIMEOUT)
    return fail(ISNMF_E_CUDA, "%s: statistics chain timed out (t = %llu)", where, t);
  return fail(ISNMF_E_CUDA, "%s: unknown device status %u", where, s);
}

}  // namespace

// ===========================================================================
// Online context
// ===========================================================================
struct isnmf_online {
  isnmf_online_config cfg{};
  int F = 0, K = 0, beta = 0, iters = 0, restart = 0;
  double eps = 0.0;
  SolvePlan plan;
  int WS = 0, KP = 0, NT = 0;
  cudaStream_t cs = nullptr, xs = nullptr;
  DevState* st = nullptr;
  double *W64 = nullptr, *A = nullptr, *B = nullptr, *pa = nullptr, *pb = nullptr;
  double* cta_part = nullptr;
  double* P = nullptr;
  int64_t Pcap = 0;
  float* W32 = nullptr;
  float* WB = nullptr;  // K1C layout of W^T (plan.pair only)
  float* stats = nullptr;
  double* divpart = nullptr;
  int maxblk = 0;
  uint32_t* chain_flags = nullptr;  // K1T statistics chain: one progress word per CTA
  uint32_t chain_epoch = 0;
  double* U = nullptr;  // warm activation store (fp64, see kernels.cuh warm_value)
  uint32_t* T = nullptr;
  int64_t nstore = 0;
  double* u01 = nullptr;
  float* Hlast = nullptr;
  unsigned long long* tr_t = nullptr;
  double* tr_obj = nullptr;
  unsigned long long* tr_ns = nullptr;
  int64_t tr_cap = 0;
  float* vbuf[2] = {nullptr, nullptr};
  uint64_t* ibuf[2] = {nullptr, nullptr};
  int64_t chunk = 0;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  uint64_t t_host = 0, commits_host = 0, trace_base = 0;
  double rho = 1.0;
  double eta = 0.0;
  int64_t launches = 0;
  // profiling (isnmf_online_profile_begin/end)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  bool span_open = false;           // between profile_begin and profile_end
  std::vector<cudaEvent_t> ev_tail;  // K2 start, K3 end per mini-batch (profiling)
  size_t tail_used = 0;
  int64_t prof_frames = 0;
  cudaEvent_t ev_span[2] = {nullptr, nullptr};
  long long* phase_prof = nullptr;  // ISNMF_PHASE_PROF builds only
  long long* fold_prof = nullptr;   // ISNMF_PHASE_PROF builds only
};

namespace {

int online_free(isnmf_online* c) {
  if (!c) return 0;
  if (c->cs) cudaStreamSynchronize(c->cs);
  if (c->xs) cudaStreamSynchronize(c->xs);
  void* ptrs[] = {c->st, c->W64, c->A, c->B, c->pa, c->pb, c->cta_part, c->P, c->W32, c->WB, c->stats,
                  c->chain_flags, c->divpart, c->U, c->T, c->u01, c->Hlast, c->tr_t, c->tr_obj, c->tr_ns, c->vbuf[0],
                  c->vbuf[1], c->ibuf[0], c->ibuf[1]};
  for (void* p : ptrs) dfree(p);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    if (c->ev_free[i]) cudaEventDestroy(c->ev_free[i]);
    if (c->ev_span[i]) cudaEventDestroy(c->ev_span[i]);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto e : c->ev_tail) cudaEventDestroy(e);
  if (c->cs) cudaStreamDestroy(c->cs);
  if (c->xs) cudaStreamDestroy(c->xs);
  delete c;
  return 0;
}

int read_state(isnmf_online* c, DevState* h) {
  CU(cudaStreamSynchronize(c->cs));
  CU(cudaMemcpy(h, c->st, sizeof(DevState), cudaMemcpyDeviceToHost));
  return 0;
}

// Grows the P table (prefix products of column scales) to hold `rows` rows.
// Stream-ordered (no host synchronisation), so growth never drains the queue.
int ensure_P(isnmf_online* c, int64_t rows) {
  if (rows <= c->Pcap) return 0;
  const int64_t cap = std::max<int64_t>(rows, 2 * c->Pcap + 64);
  double* np = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&np), size_t(cap) * c->K * sizeof(double), c->cs));
  if (c->P) {
    CU(cudaMemcpyAsync(np, c->P, size_t(c->Pcap) * c->K * sizeof(double), cudaMemcpyDeviceToDevice, c->cs));
    CU(cudaFreeAsync(c->P, c->cs));
  }
  c->P = np;
  c->Pcap = cap;
  return 0;
}

int ensure_trace(isnmf_online* c, int64_t n) {
  if (n <= c->tr_cap) return 0;
  const int64_t cap = std::max<int64_t>(n, 2 * c->tr_cap + 64);
  unsigned long long *t = nullptr, *ns = nullptr;
  double* o = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&t), size_t(cap) * sizeof(*t), c->cs));
  CU(cudaMallocAsync(reinterpret_cast<void**>(&ns), size_t(cap) * sizeof(*ns), c->cs));
  CU(cudaMallocAsync(reinterpret_cast<void**>(&o), size_t(cap) * sizeof(*o), c->cs));
  if (c->tr_cap) {
    CU(cudaMemcpyAsync(t, c->tr_t, c->tr_cap * sizeof(*t), cudaMemcpyDeviceToDevice, c->cs));
    CU(cudaMemcpyAsync(ns, c->tr_ns, c->tr_cap * sizeof(*ns), cudaMemcpyDeviceToDevice, c->cs));
    CU(cudaMemcpyAsync(o, c->tr_obj, c->tr_cap * sizeof(*o), cudaMemcpyDeviceToDevice, c->cs));
    CU(cudaFreeAsync(c->tr_t, c->cs));
    CU(cudaFreeAsync(c->tr_ns, c->cs));
    CU(cudaFreeAsync(c->tr_obj, c->cs));
  }
  c->tr_t = t;
  c->tr_ns = ns;
  c->tr_obj = o;
  c->tr_cap = cap;
  return 0;
}

// One block of nb frames inside a single mini-batch: K0? -> K1 -> K2 (-> K3).
FoldArgs fold_args(const isnmf_online* c) {
  FoldArgs r{};
  r.stats = c->stats;
  r.divpart = c->divpart;
  r.F = c->F;
  r.K = c->K;
  r.KP = c->KP;
  r.WS = c->WS;
  r.W64 = c->W64;
  r.pa = c->pa;
  r.pb = c->pb;
  r.A = c->A;
  r.B = c->B;
  r.W32 = c->W32;
  r.WB = c->WB;
  r.wb_kp = c->KP;
  r.P = c->P;
  r.cta_part = c->cta_part;
  r.rho = c->rho;
  r.st = c->st;
  r.halt = &c->st->halt;
  r.tr_t = c->tr_t;
  r.tr_obj = c->tr_obj;
  r.tr_ns = c->tr_ns;
  r.tr_cap = c->tr_cap;
  r.tprof = c->fold_prof;
  r.stats_cap = c->maxblk;
  r.p_cap = c->Pcap;
  return r;
}

int launch_block(isnmf_online* c, const float* dv, int64_t ldv, int nb, const uint64_t* widx_dev) {
  const int nblk = (nb + c->NT - 1) / c->NT;
  if (c->restart == ISNMF_RESTART_FRESH) {
    fresh_kernel<<<(nb + 127) / 128, 128, 0, c->cs>>>(c->cfg.seed, c->t_host, nb, c->K, c->u01);
    c->launches++;
  }
  SolveArgs a{};
  a.W32 = c->W32;
  a.ws = c->WS;
  a.WB = c->WB;
  a.F = c->F;
  a.K = c->K;
  a.V = dv;
  a.ldv = ldv;
  a.vsel = nullptr;
  a.v0 = 0;
  a.nframes = nb;
  a.iters = c->iters;
  a.eps = float(c->eps);
  a.epsd = c->eps;
  a.h0_mode = c->restart == ISNMF_RESTART_WARM ? 1 : 2;
  a.U = c->U;
  a.T = c->T;
  a.P = c->P;
  a.c_now = uint32_t(c->commits_host);
  a.widx = widx_dev;
  a.wbase = c->nstore ? int64_t(c->t_host % uint64_t(c->nstore)) : 0;
  a.wmod = c->nstore ? c->nstore : 1;
  a.u01 = c->u01;
  a.kst = c->st;
  a.Hout = c->Hlast + size_t(c->t_host % uint64_t(c->beta)) * c->K;
  a.write_store = c->restart == ISNMF_RESTART_WARM;
  a.check_h0 = 1;
  a.do_stats = 1;
  a.div_first = 0;
  a.stats = c->stats;
  a.divpart = c->divpart;
  a.stats_cap = c->maxblk;
  a.status = &c->st->status;
  a.halt = &c->st->halt;
  a.prof = c->phase_prof;
  const bool chained = c->chain_flags && c->plan.chain > 1 && nblk > 1;
  if (chained) {  // K1T: `chain` CTAs accumulate one statistics plane in rank order
    if (c->chain_epoch >= (1u << 18)) {  // keep stale words far behind every future target
      CU(cudaMemsetAsync(c->chain_flags, 0, size_t(c->maxblk) * sizeof(uint32_t), c->cs));
      c->chain_epoch = 0;
    }
    a.chain = c->plan.chain;
    a.chain_base = ++c->chain_epoch * kTcChainSpan;
    a.chain_flags = c->chain_flags;
  }
  if (c->prof) {
    while (c->ev_pool.size() < c->ev_used + 2) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      c->ev_pool.push_back(e);
    }
    CU(cudaEventRecord(c->ev_pool[c->ev_used], c->cs));
  }
  launch_solve(c->plan, nblk, a, c->cs, !c->prof);
  if (c->prof) {
    CU(cudaEventRecord(c->ev_pool[c->ev_used + 1], c->cs));
    c->ev_used += 2;
    c->prof_frames += nb;
  }
  const bool commit = (c->t_host + uint64_t(nb)) % uint64_t(c->beta) == 0;
  FoldArgs r = fold_args(c);
  r.nstat = chained ? (nblk + c->plan.chain - 1) / c->plan.chain : nblk;
  r.stats_tiled = chained ? 1 : c->plan.tiled ? 2 : 0;
  r.after_k1 = 1;
  r.ndiv = (c->plan.pair || c->plan.mpair) ? 2 * nblk : nblk;
  r.nframes = nb;
  r.do_commit = commit;
  r.eta = c->eta;
  if (c->prof) {
    while (c->ev_tail.size() < c->tail_used + 2) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      c->ev_tail.push_back(e);
    }
    CU(cudaEventRecord(c->ev_tail[c->tail_used], c->cs));
  }
  TRY(launch_fold(r, c->cs, !c->prof));
  c->launches += 2;
  if (commit) c->commits_host++;
  if (c->prof) {
    CU(cudaEventRecord(c->ev_tail[c->tail_used + 1], c->cs));
    c->tail_used += 2;
  }
  c->t_host += uint64_t(nb);
  CU(cudaGetLastError());
  return 0;
}

// Frames [0, n) of a device-resident span, split at mini-batch boundaries and,
// in warm mode, wherever a store column repeats inside a mini-batch (the
// reference's sequential loop would see the first visit's update).
int run_span(isnmf_online* c, const float* dv, int64_t ldv, int64_t n, const uint64_t* idx_host,
             const uint64_t* idx_dev) {
  int64_t pos = 0;
  std::unordered_set<uint64_t> seen;
  while (pos < n) {
    const int64_t room = int64_t(uint64_t(c->beta) - c->t_host % uint64_t(c->beta));
    int64_t nb = std::min<int64_t>(room, n - pos);
    if (c->restart == ISNMF_RESTART_WARM && !idx_host) nb = std::min<int64_t>(nb, c->nstore);
    if (c->restart == ISNMF_RESTART_WARM && idx_host) {
      seen.clear();
      for (int64_t j = 0; j < nb; ++j)
        if (!seen.insert(idx_host[pos + j]).second) {
          nb = j;
          break;
        }
    }
    TRY(launch_block(c, dv + pos * ldv, ldv, int(nb), idx_dev ? idx_dev + pos : nullptr));
    pos += nb;
  }
  return 0;
}

int online_enqueue(isnmf_online* c, const float* frames, int64_t ldv, int64_t n, const uint64_t* index,
                   uint64_t budget, double eta) {
  if (n < 0) return fail(ISNMF_E_INVALID_ARG, "online_run: n < 0");
  if (n > 0 && !frames) return fail(ISNMF_E_INVALID_ARG, "online_run: frames is NULL");
  if (ldv < c->F) return fail(ISNMF_E_INVALID_ARG, "online_run: ldv < F");
  c->eta = eta;
  const uint64_t room = c->t_host >= budget ? 0 : budget - c->t_host;
  const int64_t n_eff = uint64_t(n) <= room ? n : int64_t(room);
  if (n_eff == 0) return 0;
  if (c->restart == ISNMF_RESTART_WARM && index) {
    for (int64_t j = 0; j < n_eff; ++j)
      if (index[j] >= uint64_t(c->nstore))
        return fail(ISNMF_E_SHAPE_MISMATCH, "online_step: sample index outside warm activation store");
  }
  const int64_t commits_max = int64_t(c->commits_host) + n_eff / c->beta + 2;
  TRY(ensure_P(c, commits_max + 1));
  TRY(ensure_trace(c, commits_max - int64_t(c->trace_base) + 1));

  if (is_device_ptr(frames)) {
    uint64_t* idx_dev = nullptr;
    if (index) {
      TRY(dalloc(&idx_dev, n_eff));
      CU(cudaMemcpyAsync(idx_dev, index, n_eff * sizeof(uint64_t), cudaMemcpyHostToDevice, c->cs));
    }
    int rc = run_span(c, frames, ldv, n_eff, index, idx_dev);
    if (idx_dev) {
      cudaStreamSynchronize(c->cs);
      dfree(idx_dev);
    }
    return rc;
  }
  // host frames: chunked H2D on the copy stream, double-buffered
  if (!c->vbuf[0]) {
    for (int i = 0; i < 2; ++i) {
      TRY(dalloc(&c->vbuf[i], size_t(c->chunk) * c->F));
      TRY(dalloc(&c->ibuf[i], size_t(c->chunk)));
      CU(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming));
      CU(cudaEventRecord(c->ev_free[i], c->cs));
    }
  }
  int64_t pos = 0;
  int buf = 0;
  // Chunk sizes ramp up from one mini-batch so the first copy (not overlapped) is short,
  // growing by ramp_factor() per chunk: at config 3 (1/8) a copy of 9/8 s frames takes
  // about as long as the compute of the previous s frames (pinned H2D ~55 GB/s = ~0.9x
  // the consumption rate), so the compute stream does not wait on the copy stream while
  // the chunks grow (doubling made it wait ~9 ms per 2.7M-frame pass).
  double ramp = double(c->beta);
  while (pos < n_eff) {
    const int64_t rb = std::max<int64_t>(int64_t(c->beta), int64_t(ramp / c->beta) * c->beta);
    // ... and shrink towards the end (a fraction of what is left, whole mini-batches):
    // the last chunk's compute (copy-bound shapes) or copy (compute-bound ones) is not
    // overlapped, so it must be short — a 64-mini-batch last chunk cost 8 ms per config-3 pass.
    // With two buffers the copy of chunk i+1 waits for the compute of chunk i-1, which runs
    // beside the copy of chunk i: when copy and compute are balanced (config 3 with K1C:
    // compute = 0.82 x copy per frame) a chunk must not be much shorter than its predecessor or
    // the copy engine idles — quarters (ratio 0.75) cost ~2.5 ms per pass, eighths (0.875) do not.
    const int64_t rem = n_eff - pos;
    const int64_t tail = std::max<int64_t>(int64_t(c->beta), (rem / tail_div(c->K, c->iters)) / c->beta * c->beta);
    const int64_t cf = std::min<int64_t>(std::min<int64_t>(std::min<int64_t>(c->chunk, rb), tail), rem);
    ramp *= ramp_factor(c->K, c->iters);
    CU(cudaStreamWaitEvent(c->xs, c->ev_free[buf], 0));
    if (ldv == c->F)  // contiguous frames: one linear DMA (2D copies run far below PCIe speed)
      CU(cudaMemcpyAsync(c->vbuf[buf], frames + pos * ldv, size_t(cf) * c->F * sizeof(float),
                         cudaMemcpyHostToDevice, c->xs));
    else
      CU(cudaMemcpy2DAsync(c->vbuf[buf], size_t(c->F) * sizeof(float), frames + pos * ldv,
                           size_t(ldv) * sizeof(float), size_t(c->F) * sizeof(float), size_t(cf),
                           cudaMemcpyHostToDevice, c->xs));
    if (index)
      CU(cudaMemcpyAsync(c->ibuf[buf], index + pos, size_t(cf) * sizeof(uint64_t), cudaMemcpyHostToDevice, c->xs));
    CU(cudaEventRecord(c->ev_copied[buf], c->xs));
    CU(cudaStreamWaitEvent(c->cs, c->ev_copied[buf], 0));
    TRY(run_span(c, c->vbuf[buf], c->F, cf, index ? index + pos : nullptr, index ? c->ibuf[buf] : nullptr));
    CU(cudaEventRecord(c->ev_free[buf], c->cs));
    pos += cf;
    buf ^= 1;
  }
  return 0;
}

int online_finish(isnmf_online* c, int32_t* stopped) {
  DevState h;
  TRY(read_state(c, &h));
  c->t_host = h.t;
  c->commits_host = h.commits;
  if (stopped) *stopped = int32_t(h.halt != 0);
  if (h.status) {
    // report once, then clear: the reference's exceptions leave the state usable
    // (solve_h throws before it mutates anything), so the context must be too
    const unsigned int zero = 0;
    CU(cudaMemcpy(reinterpret_cast<char*>(c->st) + offsetof(DevState, status), &zero, sizeof(zero),
                  cudaMemcpyHostToDevice));
    return status_to_code(h.status, "online", h.t);
  }
  return 0;
}

}  // namespace

extern "C" {

const char* isnmf_last_error(void) { return g_err.c_str(); }

int isnmf_device_info(char* buf, int64_t cap) {
  int dev = 0;
  cudaDeviceProp p;
  CU(cudaGetDevice(&dev));
  CU(cudaGetDeviceProperties(&p, dev));
  std::string variants;
  for (int i = 0; i < kNumVariants; ++i)
    variants += (i ? "," : "") + std::to_string(g_variants[i].TK * 4) + "x" + std::to_string(g_variants[i].TN * 4);
  const int n = snprintf(buf, size_t(cap),
                         "{\"device\":\"%s\",\"sm\":\"%d.%d\",\"sms\":%d,\"smem_optin\":%zu,\"arch\":\"sm_100a\","
                         "\"solve_variants_KPxNT\":\"%s\"}",
                         p.name, p.major, p.minor, p.multiProcessorCount, p.sharedMemPerBlockOptin, variants.c_str());
  return n < cap ? 0 : fail(ISNMF_E_INVALID_ARG, "device_info: buffer too small");
}

int isnmf_online_create(isnmf_online** out, const isnmf_online_config* cfg) {
  if (!out || !cfg) return fail(ISNMF_E_INVALID_ARG, "online_create: NULL argument");
  *out = nullptr;
  if (cfg->F < 1 || cfg->K < 1) return fail(ISNMF_E_SHAPE_MISMATCH, "online_create: empty dictionary");
  if (cfg->beta < 1) return fail(ISNMF_E_NEGATIVE_INPUT, "config: beta must be >= 1");
  if (cfg->inner_iters < 1) return fail(ISNMF_E_NEGATIVE_INPUT, "online_create: inner_iters must be >= 1");
  if (!(cfg->epsilon > 0.0)) return fail(ISNMF_E_NEGATIVE_INPUT, "config: epsilon must be > 0");
  if (cfg->restart != ISNMF_RESTART_WARM && cfg->restart != ISNMF_RESTART_FRESH)
    return fail(ISNMF_E_INVALID_ARG, "online_create: bad restart mode");
  if (cfg->restart == ISNMF_RESTART_WARM && cfg->n_store < 1)
    return fail(ISNMF_E_EMPTY_DATASET, "online: warm restarts need an in-memory dataset");
  auto* c = new isnmf_online;
  c->cfg = *cfg;
  c->F = int(cfg->F);
  c->K = int(cfg->K);
  c->beta = cfg->beta;
  c->iters = cfg->inner_iters;
  c->restart = cfg->restart;
  c->eps = cfg->epsilon;
  c->nstore = cfg->restart == ISNMF_RESTART_WARM ? cfg->n_store : 0;
  c->chunk = cfg->max_chunk > 0 ? cfg->max_chunk : int64_t(64) * cfg->beta;
  int rc = plan_solve(c->F, c->K, c->beta, &c->plan, (cfg->flags & ISNMF_FLAG_GENERIC_SOLVE) != 0, true,
                      cfg->flags);
  auto bail = [&](int code) {
    std::string keep = g_err;
    online_free(c);
    g_err = keep;
    return code;
  };
  if (rc) return bail(rc);
  c->KP = c->plan.KP;
  c->NT = c->plan.NT;
  c->WS = c->plan.WS;
  c->maxblk = (c->beta + c->NT - 1) / c->NT;
  const size_t FK = size_t(c->F) * c->K;
  if (cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->xs, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(ISNMF_E_CUDA, "online_create: stream creation failed (%s)",
                     cudaGetErrorString(cudaGetLastError())));
  if ((rc = dalloc(&c->st, 1)) || (rc = dalloc(&c->W64, FK)) || (rc = dalloc(&c->A, FK)) ||
      (rc = dalloc(&c->B, FK)) || (rc = dalloc(&c->pa, FK)) || (rc = dalloc(&c->pb, FK)) ||
      (rc = dalloc(&c->cta_part, size_t(fold_parts(c->K)))) ||
      (rc = dalloc(&c->W32, size_t(c->F) * c->WS)) ||
      (rc = dalloc(&c->stats, size_t(c->maxblk) * 2 * ((c->F + 15) & ~int64_t(15)) * c->KP + 4)) ||
      (rc = dalloc(&c->divpart, 2 * size_t(c->maxblk))) ||
      (c->plan.chain > 1 && (rc = dalloc(&c->chain_flags, size_t(c->maxblk)))) ||
      (c->plan.pair && (rc = dalloc(&c->WB, size_t(2) * 2 * c->KP * kWbRows))) ||
      (rc = dalloc(&c->Hlast, size_t(c->beta) * c->K)))
    return bail(rc);
  if (c->restart == ISNMF_RESTART_FRESH && (rc = dalloc(&c->u01, size_t(c->beta) * c->K))) return bail(rc);
  if (c->restart == ISNMF_RESTART_WARM &&
      ((rc = dalloc(&c->U, size_t(c->nstore) * c->K)) || (rc = dalloc(&c->T, size_t(c->nstore)))))
    return bail(rc);
  if ((rc = ensure_P(c, 64)) || (rc = ensure_trace(c, 64))) return bail(rc);
  DevState h{};
  h.last_delta = INFINITY;
  h.kmeanw = 1.0;
  if (cudaMemcpy(c->st, &h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(c->W32, 0, size_t(c->F) * c->WS * sizeof(float)) != cudaSuccess ||
      (c->WB && cudaMemset(c->WB, 0, size_t(2) * 2 * c->KP * kWbRows * sizeof(float)) != cudaSuccess) ||
      (c->chain_flags && cudaMemset(c->chain_flags, 0, size_t(c->maxblk) * sizeof(uint32_t)) != cudaSuccess) ||
      cudaMemset(c->pa, 0, FK * sizeof(double)) != cudaSuccess ||
      cudaMemset(c->pb, 0, FK * sizeof(double)) != cudaSuccess ||
      cudaMemset(c->Hlast, 0, size_t(c->beta) * c->K * sizeof(float)) != cudaSuccess)
    return bail(fail(ISNMF_E_CUDA, "online_create: init failed (%s)", cudaGetErrorString(cudaGetLastError())));
  if ((rc = settle())) return bail(rc);
  fill_f64<<<64, 256, 0, c->cs>>>(c->P, c->Pcap * c->K, 1.0);
  if (c->restart == ISNMF_RESTART_WARM) {
    fill_f64<<<592, 256, 0, c->cs>>>(c->U, c->nstore * c->K, 1.0);
    fill_u32<<<592, 256, 0, c->cs>>>(c->T, c->nstore, 0u);
  }
  mark_origin<<<1, 1, 0, c->cs>>>(c->st);
  if (cudaStreamSynchronize(c->cs) != cudaSuccess)
    return bail(fail(ISNMF_E_CUDA, "online_create: %s", cudaGetErrorString(cudaGetLastError())));
  *out = c;
  return 0;
}

int isnmf_online_destroy(isnmf_online* c) { return online_free(c); }

int isnmf_online_set_dictionary(isnmf_online* c, const double* w, const double* a, const double* b) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  const int64_t F = c->F, K = c->K;
  std::vector<double> rm(size_t(F * K));
  CU(cudaStreamSynchronize(c->cs));
  if (w) {
    CU(cudaMemcpy(c->W64, w, rm.size() * sizeof(double), cudaMemcpyHostToDevice));
    std::vector<float> w32(size_t(F) * c->WS, 0.0f);
    double sum = 0.0;
    for (int64_t k = 0; k < K; ++k)
      for (int64_t f = 0; f < F; ++f) {
        w32[f * c->WS + k] = float(w[k * F + f]);
        sum += w[k * F + f];
      }
    CU(cudaMemcpy(c->W32, w32.data(), w32.size() * sizeof(float), cudaMemcpyHostToDevice));
    if (c->WB) {  // K1C's W^T halves (the layout K2 keeps up to date at every commit)
      std::vector<float> wb(size_t(2) * 2 * c->KP * kWbRows, 0.0f);
      for (int64_t k = 0; k < K; ++k)
        for (int64_t f = 0; f < std::min<int64_t>(F, 2 * kWbRows); ++f) {
          const float x = w32[f * c->WS + k];
          float hi;
          uint32_t u;
          std::memcpy(&u, &x, 4);
          u &= 0xffffe000u;
          std::memcpy(&hi, &u, 4);
          const size_t half = size_t(f / kWbRows) * 2 * c->KP * kWbRows;
          wb[half + wb_offset(int(k), int(f % kWbRows))] = x;
          wb[half + wb_offset(c->KP + int(k), int(f % kWbRows))] = x - hi;
        }
      CU(cudaMemcpy(c->WB, wb.data(), wb.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    const double kmeanw = double(K) * (sum / double(F * K));
    CU(cudaMemcpy(reinterpret_cast<char*>(c->st) + offsetof(DevState, kmeanw), &kmeanw, sizeof(double),
                  cudaMemcpyHostToDevice));
  }
  if (a) CU(cudaMemcpy(c->A, a, rm.size() * sizeof(double), cudaMemcpyHostToDevice));
  if (b) CU(cudaMemcpy(c->B, b, rm.size() * sizeof(double), cudaMemcpyHostToDevice));
  return settle();
}

int isnmf_online_get_dictionary(isnmf_online* c, double* w, double* a, double* b) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  const int64_t F = c->F, K = c->K;
  std::vector<double> rm(size_t(F * K));
  CU(cudaStreamSynchronize(c->cs));
  double* src[3] = {c->W64, c->A, c->B};
  double* dst[3] = {w, a, b};
  for (int i = 0; i < 3; ++i)
    if (dst[i]) CU(cudaMemcpy(dst[i], src[i], rm.size() * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int isnmf_online_set_pending(isnmf_online* c, const double* pa, const double* pb, double pending_div,
                             uint64_t pending_count) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  const int64_t F = c->F, K = c->K;
  std::vector<double> rm(size_t(F * K));
  CU(cudaStreamSynchronize(c->cs));
  if (pa) CU(cudaMemcpy(c->pa, pa, rm.size() * sizeof(double), cudaMemcpyHostToDevice));
  if (pb) CU(cudaMemcpy(c->pb, pb, rm.size() * sizeof(double), cudaMemcpyHostToDevice));
  DevState h;
  CU(cudaMemcpy(&h, c->st, sizeof(h), cudaMemcpyDeviceToHost));
  h.pending_div = pending_div;
  h.pending_count = pending_count;
  CU(cudaMemcpy(c->st, &h, sizeof(h), cudaMemcpyHostToDevice));
  return settle();
}

int isnmf_online_get_pending(isnmf_online* c, double* pa, double* pb, double* pending_div, uint64_t* pending_count) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  const int64_t F = c->F, K = c->K;
  std::vector<double> rm(size_t(F * K));
  CU(cudaStreamSynchronize(c->cs));
  if (pa) CU(cudaMemcpy(pa, c->pa, rm.size() * sizeof(double), cudaMemcpyDeviceToHost));
  if (pb) CU(cudaMemcpy(pb, c->pb, rm.size() * sizeof(double), cudaMemcpyDeviceToHost));
  DevState h;
  CU(cudaMemcpy(&h, c->st, sizeof(h), cudaMemcpyDeviceToHost));
  if (pending_div) *pending_div = h.pending_div;
  if (pending_count) *pending_count = h.pending_count;
  return 0;
}

int isnmf_online_set_counters(isnmf_online* c, uint64_t t, uint64_t commits, double rho) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  if (!(rho >= 0.0)) return fail(ISNMF_E_NEGATIVE_INPUT, "rho must be >= 0");
  CU(cudaStreamSynchronize(c->cs));
  const uint64_t c_old = c->commits_host;
  TRY(ensure_P(c, int64_t(std::max(commits, c_old)) + 2));
  if (commits != c_old) {
    // P[commits] <- 1 and re-tag the warm store at its current values
    if (c->restart == ISNMF_RESTART_WARM)
      warm_rebase<<<592, 256, 0, c->cs>>>(c->U, c->T, c->P, c->nstore, c->K, uint32_t(c_old), uint32_t(commits));
    fill_f64<<<1, 256, 0, c->cs>>>(c->P + size_t(commits) * c->K, c->K, 1.0);
    if (c->restart == ISNMF_RESTART_WARM) {
      // tags now equal `commits`, whose P row is 1: values unchanged
    }
    CU(cudaStreamSynchronize(c->cs));
  }
  DevState h;
  CU(cudaMemcpy(&h, c->st, sizeof(h), cudaMemcpyDeviceToHost));
  h.t = t;
  h.commits = commits;
  h.trace_base = commits;
  h.halt = 0;
  CU(cudaMemcpy(c->st, &h, sizeof(h), cudaMemcpyHostToDevice));
  c->t_host = t;
  c->commits_host = commits;
  c->trace_base = commits;
  c->rho = rho;
  return settle();
}

int isnmf_online_get_counters(isnmf_online* c, uint64_t* t, uint64_t* commits, double* rho, double* last_delta,
                              double* last_obj) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  DevState h;
  TRY(read_state(c, &h));
  if (t) *t = h.t;
  if (commits) *commits = h.commits;
  if (rho) *rho = c->rho;
  if (last_delta) *last_delta = h.last_delta;
  if (last_obj) *last_obj = h.last_obj;
  return 0;
}

int isnmf_online_set_warm_h(isnmf_online* c, const double* warm_h) {
  if (!c || !warm_h) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  if (c->restart != ISNMF_RESTART_WARM) return fail(ISNMF_E_INVALID_ARG, "set_warm_h: context is not warm");
  CU(cudaStreamSynchronize(c->cs));
  CU(cudaMemcpy(c->U, warm_h, size_t(c->nstore) * c->K * sizeof(double), cudaMemcpyHostToDevice));
  TRY(settle());
  fill_u32<<<592, 256, 0, c->cs>>>(c->T, c->nstore, uint32_t(c->commits_host));
  fill_f64<<<1, 256, 0, c->cs>>>(c->P + size_t(c->commits_host) * c->K, c->K, 1.0);
  CU(cudaStreamSynchronize(c->cs));
  return 0;
}

int isnmf_online_fill_warm_h(isnmf_online* c, double value) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  if (c->restart != ISNMF_RESTART_WARM) return fail(ISNMF_E_INVALID_ARG, "fill_warm_h: context is not warm");
  fill_f64<<<592, 256, 0, c->cs>>>(c->U, c->nstore * c->K, value);
  fill_u32<<<592, 256, 0, c->cs>>>(c->T, c->nstore, uint32_t(c->commits_host));
  fill_f64<<<1, 256, 0, c->cs>>>(c->P + size_t(c->commits_host) * c->K, c->K, 1.0);
  CU(cudaStreamSynchronize(c->cs));
  return 0;
}

int isnmf_online_get_warm_h(isnmf_online* c, double* warm_h) {
  if (!c || !warm_h) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  if (c->restart != ISNMF_RESTART_WARM) return fail(ISNMF_E_INVALID_ARG, "get_warm_h: context is not warm");
  double* d = nullptr;
  TRY(dalloc(&d, size_t(c->nstore) * c->K));
  CU(cudaStreamSynchronize(c->cs));
  DevState h;
  CU(cudaMemcpy(&h, c->st, sizeof(h), cudaMemcpyDeviceToHost));
  warm_read<<<592, 256, 0, c->cs>>>(c->U, c->T, c->P, c->nstore, c->K, uint32_t(h.commits), d);
  CU(cudaStreamSynchronize(c->cs));
  CU(cudaMemcpy(warm_h, d, size_t(c->nstore) * c->K * sizeof(double), cudaMemcpyDeviceToHost));
  dfree(d);
  return 0;
}

int isnmf_online_enqueue(isnmf_online* c, const float* frames, int64_t ldv, int64_t n, const uint64_t* index,
                         uint64_t budget, double eta) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  return online_enqueue(c, frames, ldv, n, index, budget, eta);
}

int isnmf_online_synchronize(isnmf_online* c) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  return online_finish(c, nullptr);
}

int isnmf_online_run(isnmf_online* c, const float* frames, int64_t ldv, int64_t n, const uint64_t* index,
                     uint64_t budget, double eta, int32_t* stopped) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  int rc = online_enqueue(c, frames, ldv, n, index, budget, eta);
  int rc2 = online_finish(c, stopped);
  return rc ? rc : rc2;
}

int isnmf_online_commit(isnmf_online* c) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  TRY(ensure_P(c, int64_t(c->commits_host) + 2));
  TRY(ensure_trace(c, int64_t(c->commits_host - c->trace_base) + 2));
  FoldArgs r = fold_args(c);
  r.nstat = 0;
  r.ndiv = 0;
  r.nframes = 0;
  r.do_commit = 1;
  r.eta = 0.0;
  TRY(launch_fold(r, c->cs));
  c->launches += 1;
  c->commits_host++;
  CU(cudaGetLastError());
  return online_finish(c, nullptr);
}

void* isnmf_host_alloc(int64_t bytes) {
  void* p = nullptr;
  if (bytes <= 0 || cudaHostAlloc(&p, size_t(bytes), cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    fail(ISNMF_E_CUDA, "host_alloc: %lld bytes failed", (long long)bytes);
    return nullptr;
  }
  return p;
}

void isnmf_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int isnmf_online_get_trace(isnmf_online* c, uint64_t* samples, double* obj, double* seconds, int64_t cap,
                           int64_t* n) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  DevState h;
  TRY(read_state(c, &h));
  const int64_t cnt = std::min<int64_t>(int64_t(h.commits - h.trace_base), std::min<int64_t>(cap, c->tr_cap));
  if (n) *n = std::max<int64_t>(cnt, 0);
  if (cnt <= 0) return 0;
  std::vector<unsigned long long> t(static_cast<size_t>(cnt)), ns(static_cast<size_t>(cnt));
  std::vector<double> o(static_cast<size_t>(cnt));
  CU(cudaMemcpy(t.data(), c->tr_t, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(ns.data(), c->tr_ns, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(o.data(), c->tr_obj, cnt * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < cnt; ++i) {
    if (samples) samples[i] = t[size_t(i)];
    if (obj) obj[i] = o[size_t(i)];
    if (seconds) seconds[i] = double(ns[size_t(i)] - h.origin_ns) * 1e-9;
  }
  return 0;
}

int isnmf_online_clear_trace(isnmf_online* c) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  DevState h;
  TRY(read_state(c, &h));
  h.trace_base = h.commits;
  CU(cudaMemcpy(c->st, &h, sizeof(h), cudaMemcpyHostToDevice));
  TRY(settle());
  c->trace_base = h.commits;
  mark_origin<<<1, 1, 0, c->cs>>>(c->st);
  CU(cudaStreamSynchronize(c->cs));
  return 0;
}

int isnmf_online_get_last_h(isnmf_online* c, double* h, int64_t n) {
  if (!c || !h) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  if (n < 0 || n > c->beta) return fail(ISNMF_E_INVALID_ARG, "get_last_h: n must be <= beta");
  std::vector<float> tmp(size_t(n) * c->K);
  CU(cudaStreamSynchronize(c->cs));
  CU(cudaMemcpy(tmp.data(), c->Hlast, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < tmp.size(); ++i) h[i] = tmp[i];
  return 0;
}

int64_t isnmf_online_launch_count(isnmf_online* c) { return c ? c->launches : -1; }

int isnmf_online_solver(isnmf_online* c, char* buf, int64_t cap) {
  if (!c || !buf || cap < 1) return fail(ISNMF_E_INVALID_ARG, "online_solver: NULL argument");
  const SolvePlan& p = c->plan;
  const char* name = p.pair                                      ? "K1C"
                     : p.mpair                                   ? "K1P"
                     : p.tiled                                   ? "K1M"
                     : p.var                                     ? "K1"
                     : p.large && p.threads == kTcThreads        ? "K1T"
                     : p.large                                   ? "K1L"
                                                                 : "generic";
  std::snprintf(buf, size_t(cap), "%s", name);
  return 0;
}

#ifdef ISNMF_PC_TRACE
// K1C progress trace (ISNMF_PC_TRACE builds, `make trace`): maps a host buffer of cap
// words the kernel writes its per-warp progress into; read it with out != NULL at any
// time (no synchronisation: the point is to see where a stuck launch waits)
int isnmf_debug_pc_trace(long long* out, int64_t cap) {
  if (!g_trace_host) {
    CU(cudaHostAlloc(reinterpret_cast<void**>(&g_trace_host), size_t(cap) * 8, cudaHostAllocMapped));
    std::memset(g_trace_host, 0, size_t(cap) * 8);
    unsigned long long* dp = nullptr;
    CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), g_trace_host, 0));
    if (pc_trace_set(dp)) return fail(ISNMF_E_UNSUPPORTED, "not an ISNMF_PC_TRACE build");
    return 0;
  }
  if (out) std::memcpy(out, g_trace_host, size_t(cap) * 8);
  return 0;
}

#endif

#ifdef ISNMF_PHASE_PROF
// Debug hook of ISNMF_PHASE_PROF builds: per-(CTA, warp) cycles per K1 phase.
int isnmf_debug_phase_prof(isnmf_online* c, long long* out, int64_t cap, int32_t reset) {
  const size_t n = size_t(c->maxblk) * kWarps * 8;
  if (!c->phase_prof) {
    CU(cudaMalloc(&c->phase_prof, n * sizeof(long long)));
    CU(cudaMemset(c->phase_prof, 0, n * sizeof(long long)));
  }
  CU(cudaStreamSynchronize(c->cs));
  if (out) CU(cudaMemcpy(out, c->phase_prof, std::min<size_t>(n, size_t(cap)) * sizeof(long long),
                         cudaMemcpyDeviceToHost));
  if (reset) CU(cudaMemset(c->phase_prof, 0, n * sizeof(long long)));
  return 0;
}

// K1M stamps of CTA 0 in the batch / stateless passes (the last tile the CTA ran): [warp][64]
int isnmf_debug_work_prof(long long* out, int64_t cap) {
  const size_t n = 16 * 64;
  if (!g_work_prof) {
    CU(cudaMalloc(&g_work_prof, n * sizeof(long long)));
    CU(cudaMemset(g_work_prof, 0, n * sizeof(long long)));
  }
  CU(cudaDeviceSynchronize());
  if (out) CU(cudaMemcpy(out, g_work_prof, std::min<size_t>(n, size_t(cap)) * sizeof(long long), cudaMemcpyDeviceToHost));
  return 0;
}

// per-CTA globaltimer stamps of the last fold_commit_kernel launch: [K*kFoldCluster][8]
int isnmf_debug_fold_prof(isnmf_online* c, long long* out, int64_t cap) {
  const size_t n = size_t(c->K) * kFoldCluster * 8;
  if (!c->fold_prof) {
    CU(cudaMalloc(&c->fold_prof, n * sizeof(long long)));
    CU(cudaMemset(c->fold_prof, 0, n * sizeof(long long)));
  }
  CU(cudaStreamSynchronize(c->cs));
  if (out) CU(cudaMemcpy(out, c->fold_prof, std::min<size_t>(n, size_t(cap)) * sizeof(long long),
                         cudaMemcpyDeviceToHost));
  return 0;
}
#endif

int isnmf_online_profile_begin(isnmf_online* c, int32_t per_kernel) {
  if (!c) return fail(ISNMF_E_INVALID_ARG, "NULL context");
  for (int i = 0; i < 2; ++i)
    if (!c->ev_span[i]) CU(cudaEventCreate(&c->ev_span[i]));
  c->prof = per_kernel != 0;
  c->span_open = true;
  c->ev_used = 0;
  c->tail_used = 0;
  c->prof_frames = 0;
  CU(cudaEventRecord(c->ev_span[0], c->cs));
  return 0;
}

int isnmf_online_profile_end(isnmf_online* c, double* solve_ms, int64_t* solve_launches, int64_t* solve_frames,
                             double* span_ms, double* tail_ms) {
  if (!c || !c->span_open) return fail(ISNMF_E_INVALID_ARG, "profile_end without profile_begin");
  CU(cudaEventRecord(c->ev_span[1], c->cs));
  CU(cudaEventSynchronize(c->ev_span[1]));
  double tot = 0.0;
  for (size_t i = 0; i + 1 < c->ev_used; i += 2) {
    float ms = 0.0f;
    CU(cudaEventElapsedTime(&ms, c->ev_pool[i], c->ev_pool[i + 1]));
    tot += ms;
  }
  float span = 0.0f;
  CU(cudaEventElapsedTime(&span, c->ev_span[0], c->ev_span[1]));
  double tail = 0.0;
  for (size_t i = 0; i + 1 < c->tail_used; i += 2) {
    float ms = 0.0f;
    CU(cudaEventElapsedTime(&ms, c->ev_tail[i], c->ev_tail[i + 1]));
    tail += ms;
  }
  if (tail_ms) *tail_ms = tail;
  if (solve_ms) *solve_ms = tot;
  if (solve_launches) *solve_launches = int64_t(c->ev_used / 2);
  if (solve_frames) *solve_frames = c->prof_frames;
  if (span_ms) *span_ms = span;
  c->prof = false;
  c->span_open = false;
  return 0;
}

}  // extern "C"

// ===========================================================================
// Stateless kernels (kernels.hpp) and the batch trainer (batch.hpp)
// ===========================================================================
namespace {

__global__ void is_div_kernel(const double* y, const double* x, int64_t n, double eps, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += is_term_d((y[i] - x[i]) / (eps + x[i]));
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void update_w_kernel(const double* a, const double* b, const double* wp, int64_t n, double* w,
                                unsigned int* status) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if (b[i] > 0.0)
      w[i] = sqrt(a[i] / b[i]);
    else if (a[i] > 0.0)
      atomicOr(status, ST_INCONSISTENT);
    else
      w[i] = wp[i];
  }
}

// model.hpp:73-86 on column-major W/A/B (F x K) and optional warm_h (K x N).
__global__ void rescale_kernel(double* w, double* a, double* b, int64_t F, int64_t K, double* h, int64_t N,
                               unsigned int* status) {
  const int64_t k = blockIdx.x;
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) s += w[k * F + f];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const double sc = sh[0];
  if (!(sc > 0.0)) {
    if (threadIdx.x == 0) atomicOr(status, ST_ZERO_COLUMN);
    return;
  }
  for (int64_t f = threadIdx.x; f < F; f += blockDim.x) {
    w[k * F + f] /= sc;
    a[k * F + f] /= sc;
    b[k * F + f] *= sc;
  }
  if (h)
    for (int64_t n = threadIdx.x; n < N; n += blockDim.x) h[n * K + k] *= sc;
}

// Deterministic fp64 sum of an F x N fp32 matrix with leading dimension ld:
// block b sums a fixed element range (thread-strided, block tree), then one
// block adds the partials in block order.
constexpr int kSumBlocks = 296, kSumThreads = 256;
__global__ void sum_f32_partial(const float* v, int64_t ld, int64_t F, int64_t N, double* part) {
  __shared__ double sh[kSumThreads];
  const int64_t n = F * N, per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = blockIdx.x * per, e1 = std::min<int64_t>(n, e0 + per);
  double s = 0.0;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kSumThreads) {
    const int64_t j = e / F, f = e - j * F;
    s += double(v[j * ld + f]);
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kSumThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void sum_partials(const double* part, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

struct BatchProfile {
  bool on = false;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  double device_ms = 0.0;
  int64_t launches = 0;
};
BatchProfile g_prof;

// A device workspace for the fused solve over an arbitrary set of frames.
struct SolveWork {
  int F = 0, K = 0, WS = 0, KP = 0, NT = 0;
  SolvePlan plan;
  int seg_blocks = 0;
  cudaStream_t s = nullptr;
  DevState* st = nullptr;
  float* W32 = nullptr;
  double* W64 = nullptr;
  double *pa = nullptr, *pb = nullptr, *A = nullptr, *B = nullptr, *cta_part = nullptr;
  double *P = nullptr, *scale = nullptr;
  float* stats = nullptr;
  double* divpart = nullptr;
  unsigned int* halt = nullptr;
  double* obj_trace = nullptr;  // batch: objective of (W_{e-1}, H_{e-1}) recorded by epoch e's commit
  long long obj_cap = 0;
  int64_t launches = 0;

  ~SolveWork() {
    if (s) cudaStreamSynchronize(s);
    void* ptrs[] = {st, W32, W64, pa, pb, A, B, cta_part, P, scale, stats, divpart, halt, obj_trace};
    for (void* p : ptrs) dfree(p);
    if (s) cudaStreamDestroy(s);
  }

  int init(int64_t F_, int64_t K_, int64_t frames) {
    F = int(F_);
    K = int(K_);
    TRY(plan_solve(F, K, frames, &plan));
    KP = plan.KP;
    NT = plan.NT;
    WS = plan.WS;
    seg_blocks = device_sms() * 4;
    CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t FK = size_t(F) * K;
    TRY(dalloc(&st, 1));
    TRY(dalloc(&W32, size_t(F) * WS));
    TRY(dalloc(&W64, FK));
    TRY(dalloc(&pa, FK));
    TRY(dalloc(&pb, FK));
    TRY(dalloc(&A, FK));
    TRY(dalloc(&B, FK));
    TRY(dalloc(&cta_part, size_t(fold_parts(K))));
    TRY(dalloc(&P, 2 * size_t(K)));
    TRY(dalloc(&scale, size_t(K)));
    TRY(dalloc(&stats, size_t(seg_blocks) * 2 * ((F + 15) & ~int64_t(15)) * KP + 4));
    TRY(dalloc(&divpart, size_t(seg_blocks)));
    TRY(dalloc(&halt, 1));
    CU(cudaMemset(halt, 0, sizeof(unsigned int)));
    CU(cudaMemset(pa, 0, FK * sizeof(double)));
    CU(cudaMemset(pb, 0, FK * sizeof(double)));
    CU(cudaMemset(A, 0, FK * sizeof(double)));
    CU(cudaMemset(B, 0, FK * sizeof(double)));
    DevState h{};
    h.last_delta = INFINITY;
    CU(cudaMemcpy(st, &h, sizeof(h), cudaMemcpyHostToDevice));
    return settle();
  }

  // W from host column-major fp64 (F x K)
  int set_w(const double* w) {
    CU(cudaMemcpy(W64, w, size_t(F) * K * sizeof(double), cudaMemcpyHostToDevice));
    std::vector<float> w32(size_t(F) * WS, 0.0f);
    for (int64_t k = 0; k < K; ++k)
      for (int64_t f = 0; f < F; ++f) w32[f * WS + k] = float(w[k * F + f]);
    CU(cudaMemcpy(W32, w32.data(), w32.size() * sizeof(float), cudaMemcpyHostToDevice));
    return settle();
  }

  // One fused pass over frames [0, n) of V (device, ld ldv): h0 from H (device
  // [n][K]) scaled by hscale, `iters` MM iterations, H written back in place;
  // statistics reduced into pa/pb and the divergence into st->pending_div.  With
  // `commit` the last fold also commits (batch: rho = 0, column scales -> scale,
  // epoch bookkeeping on the device, eta stop through the halt flag).
  // K1M (tiled) covers all n frames in one launch of one CTA per SM; the other
  // kernels run segments of seg_blocks CTAs, each followed by a fold.
  int pass(const float* V, int64_t ldv, int64_t n, float* H, int iters, double eps, const double* hscale,
           bool stats_on, bool div_first, bool check_h0, bool commit = false, double eta = 0.0,
           const unsigned int* halt_in = nullptr) {
    const int64_t seg = plan.tiled ? std::max<int64_t>(n, 1) : int64_t(seg_blocks) * NT;
    for (int64_t s0 = 0; s0 < n; s0 += seg) {
      const int64_t ns = std::min<int64_t>(n - s0, seg);
      const int64_t tiles = (ns + NT - 1) / NT;
      const int nblk = int(plan.tiled ? std::min<int64_t>(tiles, device_sms()) : tiles);
      SolveArgs a{};
      a.W32 = W32;
      a.F = F;
      a.K = K;
      a.V = V;
      a.ldv = ldv;
      a.v0 = s0;
      a.nframes = int(ns);
      a.iters = iters;
      a.eps = float(eps);
      a.epsd = eps;
      a.h0_mode = 0;
      a.H0 = H + s0 * K;
      a.hscale = hscale;
      a.Hout = H + s0 * K;
      a.check_h0 = check_h0;
      a.do_stats = 1;
      a.div_first = div_first;
      a.stats = stats_on ? stats : nullptr;
      a.divpart = divpart;
      a.stats_cap = seg_blocks;
      a.status = &st->status;
      a.halt = halt_in ? halt_in : halt;
#ifdef ISNMF_PHASE_PROF
      a.prof = iters > 0 ? g_work_prof : nullptr;  // (not the final objective-only pass)
#endif
      if (nblk > 0) {
        launch_solve(plan, nblk, a, s);
        launches++;
      }
      FoldArgs r = fold_args();
      r.halt = halt_in ? const_cast<unsigned int*>(halt_in) : halt;
      r.nstat = stats_on ? nblk : 0;
      r.stats_tiled = plan.tiled ? 2 : 0;
      r.ndiv = nblk;
      r.nframes = int(ns);
      r.do_commit = commit && s0 + seg >= n;
      if (r.do_commit) {
        r.rho = 0.0;
        r.scale_out = scale;
        r.batch_mode = 1;
        r.eta = eta;
        r.tr_obj = obj_trace;
        r.tr_cap = obj_cap;
      }
      TRY(launch_fold(r, s));
      launches++;
      CU(cudaGetLastError());
    }
    return 0;
  }

  FoldArgs fold_args() const {
    FoldArgs r{};
    r.stats = stats;
    r.divpart = divpart;
    r.F = F;
    r.K = K;
    r.KP = KP;
    r.WS = WS;
    r.W64 = W64;
    r.pa = pa;
    r.pb = pb;
    r.A = A;
    r.B = B;
    r.W32 = W32;
    r.P = P;
    r.cta_part = cta_part;
    r.st = st;
    r.halt = halt;
    r.stats_cap = seg_blocks;
    return r;
  }

  int state(DevState* h) {
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpy(h, st, sizeof(DevState), cudaMemcpyDeviceToHost));
    return 0;
  }
};

int upload_frames(const double* v, int64_t F, int64_t N, float** dv) {
  std::vector<float> v32(size_t(F) * N);
  for (size_t i = 0; i < v32.size(); ++i) v32[i] = float(v[i]);
  TRY(dalloc(dv, v32.size()));
  CU(cudaMemcpy(*dv, v32.data(), v32.size() * sizeof(float), cudaMemcpyHostToDevice));
  return settle();
}

int upload_h(const double* h, int64_t K, int64_t N, float** dh) {
  std::vector<float> h32(size_t(K) * N);
  for (size_t i = 0; i < h32.size(); ++i) h32[i] = float(h[i]);
  TRY(dalloc(dh, std::max<size_t>(1, h32.size())));
  if (!h32.empty()) CU(cudaMemcpy(*dh, h32.data(), h32.size() * sizeof(float), cudaMemcpyHostToDevice));
  return settle();
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { dfree(p); }
};

}  // namespace

extern "C" {

int isnmf_is_divergence(const double* y, int64_t ny, const double* x, int64_t nx, double eps, double* out) {
  if (!out) return fail(ISNMF_E_INVALID_ARG, "NULL out");
  if (ny != nx) return fail(ISNMF_E_SHAPE_MISMATCH, "is_divergence: %lld vs %lld", (long long)ny, (long long)nx);
  if (!(eps > 0.0)) return fail(ISNMF_E_NEGATIVE_INPUT, "epsilon must be > 0");
  for (int64_t i = 0; i < ny; ++i)
    if (y[i] < 0.0 || x[i] < 0.0) return fail(ISNMF_E_NEGATIVE_INPUT, "is_divergence: negative entry");
  DevBuf dy, dx, dout;
  TRY(dalloc(reinterpret_cast<double**>(&dy.p), ny));
  TRY(dalloc(reinterpret_cast<double**>(&dx.p), ny));
  TRY(dalloc(reinterpret_cast<double**>(&dout.p), 1));
  if (ny) {
    CU(cudaMemcpy(dy.p, y, ny * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dx.p, x, ny * sizeof(double), cudaMemcpyHostToDevice));
  }
  is_div_kernel<<<1, 256>>>(static_cast<double*>(dy.p), static_cast<double*>(dx.p), ny, eps,
                            static_cast<double*>(dout.p));
  CU(cudaGetLastError());
  CU(cudaMemcpy(out, dout.p, sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

static int stateless(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N, int iters,
                     double eps, bool stats, bool check_h0, double* h_out, double* a_out, double* b_out,
                     double* div_out) {
  if (!v || !w || !h) return fail(ISNMF_E_INVALID_ARG, "NULL input");
  if (!(eps > 0.0)) return fail(ISNMF_E_NEGATIVE_INPUT, "epsilon must be > 0");
  if (F < 1 || K < 1 || N < 0) return fail(ISNMF_E_SHAPE_MISMATCH, "inconsistent shapes");
  SolveWork wk;
  TRY(wk.init(F, K, std::max<int64_t>(N, 1)));
  TRY(wk.set_w(w));
  float *dv = nullptr, *dh = nullptr;
  TRY(upload_frames(v, F, N, &dv));
  DevBuf bv, bh;
  bv.p = dv;
  TRY(upload_h(h, K, N, &dh));
  bh.p = dh;
  TRY(wk.pass(dv, F, N, dh, iters, eps, nullptr, stats, false, check_h0));
  DevState st;
  TRY(wk.state(&st));
  if (st.status) return status_to_code(st.status, "solve_h", 0);
  if (h_out) {
    std::vector<float> h32(size_t(K) * N);
    if (N) CU(cudaMemcpy(h32.data(), dh, h32.size() * sizeof(float), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < h32.size(); ++i) h_out[i] = h32[i];
  }
  if (a_out || b_out) {
    if (a_out) CU(cudaMemcpy(a_out, wk.pa, size_t(F) * K * sizeof(double), cudaMemcpyDeviceToHost));
    if (b_out) CU(cudaMemcpy(b_out, wk.pb, size_t(F) * K * sizeof(double), cudaMemcpyDeviceToHost));
  }
  if (div_out) *div_out = st.pending_div;
  return 0;
}

int isnmf_objective(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N, double eps,
                    double* out) {
  if (!out) return fail(ISNMF_E_INVALID_ARG, "NULL out");
  if (N == 0) return fail(ISNMF_E_EMPTY_DATASET, "objective: no columns");
  double d = 0.0;
  TRY(stateless(v, w, h, F, K, N, 0, eps, false, false, nullptr, nullptr, nullptr, &d));
  *out = d / double(N);
  return 0;
}

int isnmf_solve_h(const double* v, const double* w, const double* h0, int64_t F, int64_t K, int64_t N, int iters,
                  double eps, double* h_out) {
  if (!h_out) return fail(ISNMF_E_INVALID_ARG, "NULL out");
  if (iters < 0) return fail(ISNMF_E_NEGATIVE_INPUT, "solve_h: iters < 0");
  for (int64_t i = 0; i < K * N; ++i)
    if (!(h0[i] > 0.0)) return fail(ISNMF_E_NON_POSITIVE_INIT, "solve_h: h0 must be positive");
  return stateless(v, w, h0, F, K, N, iters, eps, false, true, h_out, nullptr, nullptr, nullptr);
}

int isnmf_batch_stats(const double* v, const double* w, const double* h, int64_t F, int64_t K, int64_t N, double eps,
                      double* a_out, double* b_out) {
  if (!a_out || !b_out) return fail(ISNMF_E_INVALID_ARG, "NULL out");
  return stateless(v, w, h, F, K, N, 0, eps, true, false, nullptr, a_out, b_out, nullptr);
}

int isnmf_update_w(const double* a, const double* b, const double* w_prev, int64_t F, int64_t K, double* w_out) {
  if (!a || !b || !w_prev || !w_out) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  const int64_t n = F * K;
  DevBuf da, db, dw, dout, dst;
  TRY(dalloc(reinterpret_cast<double**>(&da.p), n));
  TRY(dalloc(reinterpret_cast<double**>(&db.p), n));
  TRY(dalloc(reinterpret_cast<double**>(&dw.p), n));
  TRY(dalloc(reinterpret_cast<double**>(&dout.p), n));
  TRY(dalloc(reinterpret_cast<unsigned int**>(&dst.p), 1));
  CU(cudaMemset(dst.p, 0, sizeof(unsigned int)));
  CU(cudaMemcpy(da.p, a, n * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(db.p, b, n * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(dw.p, w_prev, n * sizeof(double), cudaMemcpyHostToDevice));
  update_w_kernel<<<std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256)), 256>>>(
      static_cast<double*>(da.p), static_cast<double*>(db.p), static_cast<double*>(dw.p), n,
      static_cast<double*>(dout.p), static_cast<unsigned int*>(dst.p));
  CU(cudaGetLastError());
  unsigned int stt = 0;
  CU(cudaMemcpy(&stt, dst.p, sizeof(stt), cudaMemcpyDeviceToHost));
  if (stt) return status_to_code(stt, "update_w", 0);
  CU(cudaMemcpy(w_out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int isnmf_rescale_dictionary(double* w, double* a, double* b, int64_t F, int64_t K, double* warm_h, int64_t N) {
  if (!w || !a || !b) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  const int64_t n = F * K;
  DevBuf dw, da, db, dh, dst;
  TRY(dalloc(reinterpret_cast<double**>(&dw.p), n));
  TRY(dalloc(reinterpret_cast<double**>(&da.p), n));
  TRY(dalloc(reinterpret_cast<double**>(&db.p), n));
  TRY(dalloc(reinterpret_cast<unsigned int**>(&dst.p), 1));
  CU(cudaMemset(dst.p, 0, sizeof(unsigned int)));
  CU(cudaMemcpy(dw.p, w, n * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(da.p, a, n * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(db.p, b, n * sizeof(double), cudaMemcpyHostToDevice));
  if (warm_h) {
    TRY(dalloc(reinterpret_cast<double**>(&dh.p), K * N));
    if (K * N) CU(cudaMemcpy(dh.p, warm_h, K * N * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (K > 0)
    rescale_kernel<<<int(K), 256>>>(static_cast<double*>(dw.p), static_cast<double*>(da.p),
                                    static_cast<double*>(db.p), F, K, static_cast<double*>(dh.p), N,
                                    static_cast<unsigned int*>(dst.p));
  CU(cudaGetLastError());
  unsigned int stt = 0;
  CU(cudaMemcpy(&stt, dst.p, sizeof(stt), cudaMemcpyDeviceToHost));
  if (stt) return status_to_code(stt, "rescale_dictionary", 0);
  CU(cudaMemcpy(w, dw.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(a, da.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(b, db.p, n * sizeof(double), cudaMemcpyDeviceToHost));
  if (warm_h && K * N) CU(cudaMemcpy(warm_h, dh.p, K * N * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

// batch_train (batch.hpp:84-143).  Per epoch e: one fused pass (objective of
// the incoming (W, H) from the first Lambda, one MM update of every column of
// H, statistics of the updated H), then W = sqrt(A/B) and the l1 rescale whose
// column scales multiply H on the next read.  The objective of epoch e is thus
// measured during epoch e+1's pass (shared Lambda, 12FKN per epoch instead of
// the reference's 14FKN); a final divergence-only pass closes the last epoch.
int isnmf_batch_train(const float* v, int64_t ldv, int64_t F, int64_t N, int64_t K, const double* w0,
                      const double* h0, uint64_t max_epochs, double eps, double eta, double* w_out, double* h_out,
                      double* obj_trace, uint64_t* epochs, double* initial_obj, double* last_delta) {
  if (!v || !w0 || !h0 || !w_out || !h_out) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  if (N == 0) return fail(ISNMF_E_EMPTY_DATASET, "batch_train: empty dataset");
  if (F < 1 || K < 1 || ldv < F) return fail(ISNMF_E_SHAPE_MISMATCH, "batch_train: inconsistent V/W0/H0 shapes");
  if (!(eps > 0.0)) return fail(ISNMF_E_NEGATIVE_INPUT, "config: epsilon must be > 0");
  for (int64_t i = 0; i < F * K; ++i)
    if (!(w0[i] > 0.0)) return fail(ISNMF_E_NON_POSITIVE_INIT, "batch_train: w0 and h0 must be strictly positive");
  SolveWork wk;
  TRY(wk.init(F, K, N));
  TRY(wk.set_w(w0));
  DevBuf bv, bh, bh64;
  const float* dv = v;
  int64_t dld = ldv;
  if (!is_device_ptr(v)) {
    float* tmp = nullptr;
    TRY(dalloc(&tmp, size_t(F) * N));
    if (ldv == F)  // contiguous frames: one linear DMA (2D copies run far below PCIe speed)
      CU(cudaMemcpy(tmp, v, size_t(F) * N * sizeof(float), cudaMemcpyHostToDevice));
    else
      CU(cudaMemcpy2D(tmp, size_t(F) * sizeof(float), v, size_t(ldv) * sizeof(float), size_t(F) * sizeof(float),
                      size_t(N), cudaMemcpyHostToDevice));
    bv.p = tmp;
    dv = tmp;
    dld = F;
  }
  // H0 goes up as the caller's fp64 and is converted (and checked: h0 > 0) on the device; the
  // same fp64 buffer takes the final H back
  float* dh = nullptr;
  double* dh64 = nullptr;
  TRY(dalloc(&dh, size_t(K) * N));
  bh.p = dh;
  TRY(dalloc(&dh64, size_t(K) * N));
  bh64.p = dh64;
  CU(cudaMemcpy(dh64, h0, size_t(K) * N * sizeof(double), cudaMemcpyHostToDevice));
  TRY(settle());  // (pageable copies return once staged: the DMAs of V and H0 must have landed)
  CU(cudaMemsetAsync(wk.halt, 0, sizeof(unsigned int), wk.s));
  h_to_f32<<<1184, 256, 0, wk.s>>>(dh64, dh, K * N, wk.halt);
  {
    unsigned int bad = 0;
    CU(cudaMemcpyAsync(&bad, wk.halt, sizeof(bad), cudaMemcpyDeviceToHost, wk.s));
    CU(cudaMemsetAsync(wk.halt, 0, sizeof(unsigned int), wk.s));
    CU(cudaStreamSynchronize(wk.s));
    if (bad) return fail(ISNMF_E_NON_POSITIVE_INIT, "batch_train: w0 and h0 must be strictly positive");
  }
  // the column scales of the last commit multiply H on its next read (rescale_dictionary's
  // H compensation, model.hpp:84, applied lazily)
  fill_f64<<<1, 256, 0, wk.s>>>(wk.scale, K, 1.0);
  fill_f64<<<1, 256, 0, wk.s>>>(wk.P, 2 * K, 1.0);
  wk.obj_cap = (long long)max_epochs + 1;
  TRY(dalloc(&wk.obj_trace, size_t(wk.obj_cap)));
  if (g_prof.on) CU(cudaEventRecord(g_prof.ev[0], wk.s));
  // Every epoch is enqueued without a host round trip (batch.hpp:104-141): K1 runs one MM
  // iteration over all N frames with the objective of the incoming (W_{e-1}, H_{e-1})
  // from its first Lam and the statistics of the updated H; K2 folds them and commits
  // with rho = 0 (A, B = the statistics, W = sqrt(A/B), l1 rescale).  K2's last CTA
  // records the objective, raises DivergedObjective (batch.hpp:129-131) and sets the
  // halt flag on ||dW||_F < eta, after which every queued kernel returns at once.
  for (uint64_t e = 1; e <= max_epochs; ++e)
    TRY(wk.pass(dv, dld, N, dh, 1, eps, wk.scale, true, true, false, true, eta));
  DevState h{};
  TRY(wk.state(&h));
  const uint64_t done = h.commits;
  std::vector<double> tr(size_t(wk.obj_cap));
  CU(cudaMemcpy(tr.data(), wk.obj_trace, tr.size() * sizeof(double), cudaMemcpyDeviceToHost));
  if (h.status & ST_DIVERGED)
    return fail(ISNMF_E_DIVERGED_OBJECTIVE, "batch_train: objective increased at epoch %llu",
                (unsigned long long)done);
  if (h.status) return status_to_code(h.status, "batch_train", done);
  const double delta = h.last_delta;
  // final objective of (W_e, H_e): a divergence-only pass that also applies the last
  // rescale to H (the halt flag is cleared so it runs after an eta stop)
  h.pending_div = 0.0;
  h.pending_count = 0;
  CU(cudaMemcpy(wk.st, &h, sizeof(h), cudaMemcpyHostToDevice));
  CU(cudaMemset(wk.halt, 0, sizeof(unsigned int)));
  TRY(wk.pass(dv, dld, N, dh, 0, eps, wk.scale, false, false, false));
  if (g_prof.on) CU(cudaEventRecord(g_prof.ev[1], wk.s));
  TRY(wk.state(&h));
  if (h.status) return status_to_code(h.status, "batch_train", done);
  const double obj = h.pending_div / double(N);
  if (done >= 1) {
    const double prev = tr[done - 1];
    if (obj > prev + 1e-6 * prev + 1e-15)
      return fail(ISNMF_E_DIVERGED_OBJECTIVE, "batch_train: objective increased at epoch %llu",
                  (unsigned long long)done);
    if (initial_obj) *initial_obj = tr[0];
    if (obj_trace) {
      for (uint64_t i = 0; i + 1 < done; ++i) obj_trace[i] = tr[i + 1];
      obj_trace[done - 1] = obj;
    }
  } else if (initial_obj) {
    *initial_obj = obj;
  }
  CU(cudaMemcpy(w_out, wk.W64, size_t(F) * K * sizeof(double), cudaMemcpyDeviceToHost));
  h_to_f64<<<1184, 256, 0, wk.s>>>(dh, dh64, K * N);
  CU(cudaStreamSynchronize(wk.s));
  CU(cudaMemcpy(h_out, dh64, size_t(K) * N * sizeof(double), cudaMemcpyDeviceToHost));
  if (epochs) *epochs = done;
  if (last_delta) *last_delta = delta;
  if (g_prof.on) {
    float ms = 0.0f;
    CU(cudaEventElapsedTime(&ms, g_prof.ev[0], g_prof.ev[1]));
    g_prof.device_ms = ms;
    g_prof.launches = wk.launches;
  }
  return 0;
}

// Device time of the last isnmf_batch_train call (CUDA events on its stream
// around the enqueued epochs and the final objective pass, i.e. without the
// V / H uploads and downloads) and the kernels it launched; profiling only.
int isnmf_batch_profile(int32_t enable, double* device_ms, int64_t* launches) {
  if (enable >= 0) {
    if (!g_prof.ev[0]) {
      CU(cudaEventCreate(&g_prof.ev[0]));
      CU(cudaEventCreate(&g_prof.ev[1]));
    }
    g_prof.on = enable != 0;
  }
  if (device_ms) *device_ms = g_prof.device_ms;
  if (launches) *launches = g_prof.launches;
  return 0;
}

// harness.hpp:17-37.  H0 = max(mean test, eps)/(K mean W) * uniform_open01 from
// the reference stream mt19937_64(splitmix64(mix_seed(seed, 0xE7A1))), filled
// column-major; the stream is sequential, so it is drawn on the host (std::
// mt19937_64 is specified bit-exactly by the standard) and uploaded; the scale
// is applied on the device (hscale).  The MM iterations and the divergence of
// the final fit run in the fused solve kernel at frozen W.
int isnmf_evaluate_heldout(const float* test, int64_t ldt, int64_t F, int64_t N, const double* w, int64_t K,
                           double eps, int32_t inner_iters, uint64_t seed, double* out) {
  if (!test || !w || !out) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  if (F < 1 || K < 1 || ldt < F) return fail(ISNMF_E_SHAPE_MISMATCH, "evaluate_heldout: W rows vs test rows");
  if (N == 0) return fail(ISNMF_E_EMPTY_DATASET, "evaluate_heldout: empty test set");
  if (!(eps > 0.0)) return fail(ISNMF_E_NEGATIVE_INPUT, "epsilon must be > 0");
  if (inner_iters < 0) return fail(ISNMF_E_INVALID_ARG, "evaluate_heldout: inner_iters < 0");
  double wsum = 0.0;
  for (int64_t i = 0; i < F * K; ++i) wsum += w[i];
  const double wmean = wsum / double(F * K);
  SolveWork wk;
  TRY(wk.init(F, K, N));
  TRY(wk.set_w(w));
  DevBuf bv, bh, bs, bp;
  const float* dv = test;
  int64_t dld = ldt;
  if (!is_device_ptr(test)) {
    float* tmp = nullptr;
    TRY(dalloc(&tmp, size_t(F) * N));
    CU(cudaMemcpy2D(tmp, size_t(F) * sizeof(float), test, size_t(ldt) * sizeof(float), size_t(F) * sizeof(float),
                    size_t(N), cudaMemcpyHostToDevice));
    TRY(settle());
    bv.p = tmp;
    dv = tmp;
    dld = F;
  }
  // scale = max(mean(test), eps) / (K * mean(W)), the mean reduced on the device
  double* part = nullptr;
  TRY(dalloc(&part, kSumBlocks + 1));
  bp.p = part;
  sum_f32_partial<<<kSumBlocks, kSumThreads, 0, wk.s>>>(dv, dld, F, N, part);
  sum_partials<<<1, 32, 0, wk.s>>>(part, kSumBlocks, part + kSumBlocks);
  double tsum = 0.0;
  CU(cudaMemcpyAsync(&tsum, part + kSumBlocks, sizeof(double), cudaMemcpyDeviceToHost, wk.s));
  // uniforms (host stream, overlapped with the reduction)
  std::vector<float> u(size_t(K) * N);
  {
    auto sm = [](uint64_t x) {
      x += 0x9e3779b97f4a7c15ULL;
      x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
      x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
      return x ^ (x >> 31);
    };
    const uint64_t stream = sm(sm(seed) ^ sm(~uint64_t(0xE7A1)));
    std::mt19937_64 g(sm(stream));
    for (size_t i = 0; i < u.size(); ++i) u[i] = float(1.0 - double(g() >> 11) * 0x1.0p-53);
  }
  CU(cudaStreamSynchronize(wk.s));
  const double scale = std::max(tsum / double(F * N), eps) / (double(K) * wmean);
  float* dh = nullptr;
  TRY(dalloc(&dh, u.size()));
  bh.p = dh;
  CU(cudaMemcpyAsync(dh, u.data(), u.size() * sizeof(float), cudaMemcpyHostToDevice, wk.s));
  double* dscale = nullptr;
  TRY(dalloc(&dscale, size_t(K)));
  bs.p = dscale;
  fill_f64<<<1, 256, 0, wk.s>>>(dscale, K, scale);
  TRY(wk.pass(dv, dld, N, dh, inner_iters, eps, dscale, false, false, true));
  DevState h{};
  TRY(wk.state(&h));
  if (h.status) return status_to_code(h.status, "evaluate_heldout", 0);
  *out = h.pending_div / double(N);
  return 0;
}

// audio.hpp:121-153 (stft_power) on the device in fp64
int isnmf_stft_power(const double* samples, int64_t n_samples, int32_t window, int32_t hop, double* power,
                     int64_t frames_cap, int64_t* frames_out) {
  if (window < 2 || window % 2 != 0) return fail(ISNMF_E_UNSUPPORTED_FORMAT, "stft_power: window must be even and >= 2");
  if (hop < 1 || hop > window) return fail(ISNMF_E_UNSUPPORTED_FORMAT, "stft_power: need 1 <= hop <= window");
  if (n_samples < window) return fail(ISNMF_E_TOO_SHORT, "stft_power: signal shorter than one window");
  if (!samples || !power || !frames_out) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  const int64_t frames = (n_samples - window) / hop + 1;
  const int bins = window / 2 + 1;
  *frames_out = frames;
  if (frames > frames_cap) return fail(ISNMF_E_INVALID_ARG, "stft_power: output holds %lld frames, need %lld",
                                       (long long)frames_cap, (long long)frames);
  int logW = 0;
  while ((1 << logW) < window) ++logW;
  const bool pow2 = (1 << logW) == window && window <= 4096;
  if (!pow2 && size_t(window) * sizeof(double) + 4096 > size_t(smem_optin()))
    return fail(ISNMF_E_UNSUPPORTED, "stft_power: window %d too large", window);
  std::vector<double> win(static_cast<size_t>(window));
  std::vector<double2> tw(static_cast<size_t>(window));
  for (int i = 0; i < window; ++i) {
    win[size_t(i)] = std::sin(M_PI * (i + 0.5) / window);
    const double ang = -2.0 * M_PI * double(i) / double(window);
    tw[size_t(i)] = make_double2(std::cos(ang), std::sin(ang));
  }
  cudaStream_t st = nullptr;
  CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DevBuf bs, bw, bt, bp;
  double *ds = nullptr, *dw = nullptr, *dp = nullptr;
  double2* dt = nullptr;
  int rc = 0;
  if ((rc = dalloc(&ds, size_t(n_samples))) || (rc = dalloc(&dw, size_t(window))) ||
      (rc = dalloc(&dt, size_t(window))) || (rc = dalloc(&dp, size_t(frames) * bins))) {
    dfree(ds);
    dfree(dw);
    dfree(dt);
    dfree(dp);
    cudaStreamDestroy(st);
    return rc;
  }
  bs.p = ds;
  bw.p = dw;
  bt.p = dt;
  bp.p = dp;
  CU(cudaMemcpyAsync(ds, samples, size_t(n_samples) * sizeof(double), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dw, win.data(), win.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(dt, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice, st));
  for (int64_t f0 = 0; f0 < frames; f0 += 1 << 30) {  // grid.x limit
    const int nb = int(std::min<int64_t>(frames - f0, int64_t(1) << 30));
    if (pow2) {
      const size_t sm = size_t(window) * sizeof(double2);
      if (sm > 48 * 1024) CU(cudaFuncSetAttribute(stft_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      stft_fft_kernel<<<nb, kStftThreads, sm, st>>>(ds + f0 * hop, window, logW, hop, dw, dt, dp + f0 * bins, bins);
    } else {
      const size_t sm = size_t(window) * sizeof(double);
      if (sm > 48 * 1024) CU(cudaFuncSetAttribute(stft_dft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
      stft_dft_kernel<<<nb, kStftThreads, sm, st>>>(ds + f0 * hop, window, hop, dw, dt, dp + f0 * bins, bins);
    }
    CU(cudaGetLastError());
  }
  CU(cudaMemcpyAsync(power, dp, size_t(frames) * bins * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  CU(cudaStreamDestroy(st));
  return 0;
}

// audio.hpp:164-187 (discard_silence): the indices of the retained frames
int isnmf_discard_silence(const double* spec, int64_t bins, int64_t frames, double threshold_db, int64_t* keep,
                          int64_t* n_keep) {
  if (!spec || !keep || !n_keep) return fail(ISNMF_E_INVALID_ARG, "NULL argument");
  if (bins < 1 || frames < 1) return fail(ISNMF_E_ALL_SILENT, "discard_silence: every frame is silent");
  DevBuf bspec, bpow, bkeep, bcnt;
  const double* dspec = spec;
  if (!is_device_ptr(spec)) {
    double* tmp = nullptr;
    TRY(dalloc(&tmp, size_t(bins) * frames));
    bspec.p = tmp;
    CU(cudaMemcpy(tmp, spec, size_t(bins) * frames * sizeof(double), cudaMemcpyHostToDevice));
    dspec = tmp;
  }
  double* dpow = nullptr;
  int64_t* dkeep = nullptr;
  int64_t* dcnt = nullptr;
  TRY(dalloc(&dpow, size_t(frames)));
  bpow.p = dpow;
  TRY(dalloc(&dkeep, size_t(frames)));
  bkeep.p = dkeep;
  TRY(dalloc(&dcnt, 2));
  bcnt.p = dcnt;
  frame_power_kernel<<<int(std::min<int64_t>((frames + 7) / 8, 4096)), 256>>>(dspec, bins, frames, dpow);
  silence_select_kernel<<<1, kSelThreads>>>(dpow, frames, threshold_db, dkeep, dcnt,
                                            reinterpret_cast<int*>(dcnt + 1));
  CU(cudaGetLastError());
  int64_t hc[2] = {0, 0};
  CU(cudaMemcpy(hc, dcnt, sizeof(hc), cudaMemcpyDeviceToHost));
  if (int(hc[1] & 0xffffffff) != 0 || hc[0] == 0) return fail(ISNMF_E_ALL_SILENT, "discard_silence: every frame is silent");
  CU(cudaMemcpy(keep, dkeep, size_t(hc[0]) * sizeof(int64_t), cudaMemcpyDeviceToHost));
  *n_keep = hc[0];
  return 0;
}

}  // extern "C"

// K1M instantiations (csrc/kernels_mma.cuh) in their own translation unit, so
// the engine library's two halves compile in parallel (Makefile).  engine.cu
// reaches them only through mma_kernel().
#define ISNMF_TEMPLATES_ONLY  // the non-template kernels live in engine.cu's translation unit
#ifndef ISNMF_MMA_MULTI
#define ISNMF_MMA_MULTI false  // single-tile (online) instantiations; mma_multi_table.cu: true
#endif
#include "kernels_mma.cuh"

namespace isnmf_dev {

using MmFn = void (*)(const SolveArgs);
#define MM(kb, fg, nw) solve_mma_kernel<kb, fg, nw, ISNMF_MMA_MULTI>
#define MMROW(fg, nw) {MM(1, fg, nw), MM(2, fg, nw), MM(3, fg, nw), MM(4, fg, nw), MM(5, fg, nw), MM(6, fg, nw), MM(7, fg, nw)}
static const MmFn g_mma[2][2][7] = {{MMROW(1, 8), MMROW(2, 8)}, {MMROW(1, 12), MMROW(2, 12)}};
#undef MMROW
#undef MM

#if ISNMF_MMA_MULTI
MmFn mma_multi_kernel(int nw, int fg, int kb) { return g_mma[nw == 12 ? 1 : 0][fg - 1][kb - 1]; }
#else
MmFn mma_multi_kernel(int nw, int fg, int kb);
// the K1M kernel for nw in {8, 12} warps, fg in {1, 2} frame groups, kb in 1..7 k blocks;
// multi: the multi-tile (batch) instantiation (csrc/mma_multi_table.cu)
MmFn mma_kernel(int nw, int fg, int kb, bool multi) {
  return multi ? mma_multi_kernel(nw, fg, kb) : g_mma[nw == 12 ? 1 : 0][fg - 1][kb - 1];
}
#endif

}  // namespace isnmf_dev

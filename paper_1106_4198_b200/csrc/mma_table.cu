// K1M instantiations (csrc/kernels_mma.cuh) in their own translation unit, so
// the engine library's two halves compile in parallel (Makefile).  engine.cu
// reaches them only through mma_kernel().
#define ISNMF_TEMPLATES_ONLY  // the non-template kernels live in engine.cu's translation unit
#include "kernels_mma.cuh"

namespace isnmf_dev {

using MmFn = void (*)(const SolveArgs);
#define MM(kb, fg, nw) solve_mma_kernel<kb, fg, nw>
#define MMROW(fg, nw) {MM(1, fg, nw), MM(2, fg, nw), MM(3, fg, nw), MM(4, fg, nw), MM(5, fg, nw), MM(6, fg, nw), MM(7, fg, nw)}
static const MmFn g_mma[2][2][7] = {{MMROW(1, 8), MMROW(2, 8)}, {MMROW(1, 12), MMROW(2, 12)}};
#undef MMROW
#undef MM

// the K1M kernel for nw in {8, 12} warps, fg in {1, 2} frame groups, kb in 1..7 k blocks
MmFn mma_kernel(int nw, int fg, int kb) { return g_mma[nw == 12 ? 1 : 0][fg - 1][kb - 1]; }

}  // namespace isnmf_dev

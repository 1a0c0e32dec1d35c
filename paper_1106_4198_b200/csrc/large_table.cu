// Large-K solve kernels (K1L csrc/kernels_large.cuh, K1T csrc/kernels_large_tc.cuh)
// in their own translation unit so the engine library compiles in parallel;
// engine.cu reaches them only through large_kernel() / large_tc_kernel().
#define ISNMF_TEMPLATES_ONLY  // the non-template kernels live in engine.cu's translation unit
#include "kernels_large_tc.cuh"

namespace isnmf_dev {

using LargeFn = void (*)(const SolveArgs);

#define LG(m, n) solve_large_kernel<m, n>
static const LargeFn g_large[2][8] = {{LG(1, 1), LG(1, 2), LG(1, 3), LG(1, 4), LG(1, 5), LG(1, 6), LG(1, 7), LG(1, 8)},
                                      {LG(2, 1), LG(2, 2), LG(2, 3), LG(2, 4), LG(2, 5), LG(2, 6), LG(2, 7), LG(2, 8)}};
#undef LG
static const LargeFn g_large_tc[7] = {solve_large_tc_kernel<1>, solve_large_tc_kernel<2>, solve_large_tc_kernel<3>,
                                      solve_large_tc_kernel<4>, solve_large_tc_kernel<5>, solve_large_tc_kernel<6>,
                                      solve_large_tc_kernel<7>};

// K1L for MBW m-blocks of 128 k (1, 2) and NB frame blocks of 8 (1..8)
LargeFn large_kernel(int mbw, int nb) { return g_large[mbw - 1][nb - 1]; }
// K1T (tcgen05 phase B) for NB frame blocks of 8 (1..7)
LargeFn large_tc_kernel(int nb) { return g_large_tc[nb - 1]; }

}  // namespace isnmf_dev

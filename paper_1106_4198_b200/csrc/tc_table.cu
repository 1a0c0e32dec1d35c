// K1C instantiations (csrc/kernels_tc.cuh) in their own translation unit, so the
// engine library compiles in parallel (Makefile); engine.cu reaches them through
// pair_kernel().
#define ISNMF_TEMPLATES_ONLY  // the non-template kernels live in engine.cu's translation unit
#include "kernels_tc.cuh"

namespace isnmf_dev {

using PairFn = void (*)(const SolveArgs);
static const PairFn g_pair[5] = {solve_pair_kernel<3>, solve_pair_kernel<4>, solve_pair_kernel<5>,
                                 solve_pair_kernel<6>, solve_pair_kernel<7>};

// K1C for kb k blocks of 8 (3..7: 17 <= K <= 56)
PairFn pair_kernel(int kb) { return g_pair[kb - 3]; }
size_t pair_smem(int kb) {
  switch (kb) {
    case 3: return PcShape<3>::smem_bytes();
    case 4: return PcShape<4>::smem_bytes();
    case 5: return PcShape<5>::smem_bytes();
    case 6: return PcShape<6>::smem_bytes();
    default: return PcShape<7>::smem_bytes();
  }
}

#ifdef ISNMF_PC_TRACE
// trace buffer (mapped host memory, [CTA][10 warps]) for the next K1C launches
int pc_trace_set(unsigned long long* dev_ptr) {
  return cudaMemcpyToSymbol(g_pc_trace, &dev_ptr, sizeof(dev_ptr)) == cudaSuccess ? 0 : 1;
}
#else
int pc_trace_set(unsigned long long*) { return 1; }
#endif

}  // namespace isnmf_dev

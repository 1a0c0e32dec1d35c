// FFMA register-tile solve variants (csrc/kernels.cuh solve_kernel<TK, TN>) in
// their own translation unit so the engine library compiles in parallel;
// engine.cu reaches them only through ffma_kernel().
#define ISNMF_TEMPLATES_ONLY  // the non-template kernels live in engine.cu's translation unit
#include "kernels.cuh"

namespace isnmf_dev {

using SolveFn = void (*)(const SolveArgs);

#define V(tk, tn) \
  if (TK == tk && TN == tn) return solve_kernel<tk, tn>;
SolveFn ffma_kernel(int TK, int TN) {
#ifdef ISNMF_MIN_VARIANTS  // fast experimental builds: the headline shape only
  V(13, 7) V(5, 2) V(3, 1)
#else
  V(1, 1) V(1, 2) V(1, 4) V(1, 7) V(1, 8)
  V(2, 1) V(2, 2) V(2, 4) V(2, 7) V(2, 8)
  V(3, 1) V(3, 2) V(3, 4) V(3, 7) V(3, 8)
  V(5, 1) V(5, 2) V(5, 4) V(5, 7) V(5, 8)
  V(8, 1) V(8, 2) V(8, 4) V(8, 7) V(8, 8)
  V(13, 1) V(13, 2) V(13, 4) V(13, 7) V(13, 8)
  V(16, 1) V(16, 2) V(16, 4) V(16, 7)
#endif
  return nullptr;
}
#undef V

}  // namespace isnmf_dev

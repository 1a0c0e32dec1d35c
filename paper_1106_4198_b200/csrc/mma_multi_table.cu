// K1M multi-tile instantiations (the batch path: CTAs loop over frame tiles), in their
// own translation unit so they compile in parallel with the single-tile table.
#define ISNMF_MMA_MULTI true
#include "mma_table.cu"

// Explicit instantiations: K2 power-iteration kernels, K = 8, cluster mode = true.
#define SNOP_PHASE_SYM g_phase_cycles_ecl
#include "si_kernels.cuh"

namespace snop_si {
SNOP_INST_PI(8, 32, true)
SNOP_INST_PI(8, 64, true)
SNOP_INST_PI(8, 128, true)
SNOP_INST_PI(8, 256, true)
}  // namespace snop_si

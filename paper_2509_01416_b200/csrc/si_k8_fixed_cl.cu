// Explicit instantiations: K1 fixed-source kernels, K = 8, cluster mode = true.
#define SNOP_PHASE_SYM g_phase_cycles_fcl
#include "si_kernels.cuh"

namespace snop_si {
SNOP_INST_SI(SNOP_K, 32, true)
SNOP_INST_SI(SNOP_K, 64, true)
SNOP_INST_SI(SNOP_K, 128, true)
SNOP_INST_SI(SNOP_K, 256, true)
}  // namespace snop_si

// Explicit instantiations: K2 power-iteration kernels, K = 8, cluster mode = false.
#include "si_kernels.cuh"

namespace snop_si {
SNOP_INST_PI(8, 32, false)
SNOP_INST_PI(8, 64, false)
SNOP_INST_PI(8, 128, false)
SNOP_INST_PI(8, 256, false)
SNOP_INST_PI(8, 512, false)
}  // namespace snop_si

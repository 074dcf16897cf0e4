// Explicit instantiations: K1 fixed-source kernels, K = 8, cluster mode = false.
#include "si_kernels.cuh"

namespace snop_si {
SNOP_INST_SI(8, 32, false)
SNOP_INST_SI(8, 64, false)
SNOP_INST_SI(8, 128, false)
SNOP_INST_SI(8, 256, false)
SNOP_INST_SI(8, 512, false)
}  // namespace snop_si

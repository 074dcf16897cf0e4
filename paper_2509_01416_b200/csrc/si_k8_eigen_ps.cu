// Explicit instantiations: K2 power-iteration kernels in pair-split cluster mode, K = 8.
#define SNOP_PHASE_SYM g_phase_cycles_eigen_ps
#include "si_kernels.cuh"

namespace snop_si {
SNOP_INST_PS(SNOP_K, 32)
SNOP_INST_PS(SNOP_K, 64)
SNOP_INST_PS(SNOP_K, 128)
SNOP_INST_PS(SNOP_K, 256)
SNOP_INST_PS(SNOP_K, 512)
}  // namespace snop_si

#ifdef SNOP_PHASE_TIMING
extern "C" int snop_internal_phase_cycles_eigen_ps(unsigned long long* out /* [2][10] */, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, snop_dev::g_phase_cycles_eigen_ps, sizeof(unsigned long long) * 20);
  if (reset) {
    unsigned long long z[20] = {};
    cudaMemcpyToSymbol(snop_dev::g_phase_cycles_eigen_ps, z, sizeof(z));
  }
  return (int)e;
}
#endif

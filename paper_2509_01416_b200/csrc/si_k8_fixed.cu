// Explicit instantiations: K1 fixed-source kernels, K = 8, cluster mode = false.
#include "si_kernels.cuh"

namespace snop_si {
SNOP_INST_SI(SNOP_K, 32, false)
SNOP_INST_SI(SNOP_K, 64, false)
SNOP_INST_SI(SNOP_K, 128, false)
SNOP_INST_SI(SNOP_K, 256, false)
SNOP_INST_SI(SNOP_K, 512, false)
}  // namespace snop_si

#ifdef SNOP_PHASE_TIMING
extern "C" int snop_internal_phase_cycles(unsigned long long* out /* [2][10] */, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, snop_dev::g_phase_cycles, sizeof(unsigned long long) * 20);
  if (reset) {
    unsigned long long z[20] = {};
    cudaMemcpyToSymbol(snop_dev::g_phase_cycles, z, sizeof(z));
  }
  return (int)e;
}
#endif

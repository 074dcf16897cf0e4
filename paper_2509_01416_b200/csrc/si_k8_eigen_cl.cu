// Explicit instantiations: K2 power-iteration kernels, K = 8, cluster mode = true.
#define SNOP_PHASE_SYM g_phase_cycles_ecl
#include "si_kernels.cuh"

namespace snop_si {
SNOP_INST_PI(SNOP_K, 32, true)
SNOP_INST_PI(SNOP_K, 64, true)
SNOP_INST_PI(SNOP_K, 128, true)
SNOP_INST_PI(SNOP_K, 256, true)
}  // namespace snop_si

#ifdef SNOP_PHASE_TIMING
extern "C" int snop_internal_phase_cycles_ecl(unsigned long long* out /* [2][10] */, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out, snop_dev::g_phase_cycles_ecl, sizeof(unsigned long long) * 20);
  if (reset) {
    unsigned long long z[20] = {};
    cudaMemcpyToSymbol(snop_dev::g_phase_cycles_ecl, z, sizeof(z));
  }
  return (int)e;
}
#endif

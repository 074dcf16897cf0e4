// Explicit instantiations: K2 power-iteration kernels, K = 16.
#include "si_kernels.cuh"

namespace snop_si {
template snop_status launch_pi_t<16, 32>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, const EigenParams&, int, const double*, const double*, const double*, const double*, const double*, const double*, const double*, double*, double*, double*, int32_t*, int64_t*, uint8_t*);
template snop_status launch_pi_t<16, 64>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, const EigenParams&, int, const double*, const double*, const double*, const double*, const double*, const double*, const double*, double*, double*, double*, int32_t*, int64_t*, uint8_t*);
template snop_status launch_pi_t<16, 128>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, const EigenParams&, int, const double*, const double*, const double*, const double*, const double*, const double*, const double*, double*, double*, double*, int32_t*, int64_t*, uint8_t*);
template snop_status launch_pi_t<16, 256>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, const EigenParams&, int, const double*, const double*, const double*, const double*, const double*, const double*, const double*, double*, double*, double*, int32_t*, int64_t*, uint8_t*);
}  // namespace snop_si

// Explicit instantiations: K1 fixed-source kernels, K = 8.
#include "si_kernels.cuh"

namespace snop_si {
template snop_status launch_si_t<8, 32>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int, const double*, const double*, const double*, const double*, const double*, double*, double*, int32_t*, uint8_t*);
template snop_status launch_si_t<8, 64>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int, const double*, const double*, const double*, const double*, const double*, double*, double*, int32_t*, uint8_t*);
template snop_status launch_si_t<8, 128>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int, const double*, const double*, const double*, const double*, const double*, double*, double*, int32_t*, uint8_t*);
template snop_status launch_si_t<8, 256>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int, const double*, const double*, const double*, const double*, const double*, double*, double*, int32_t*, uint8_t*);
template snop_status launch_si_t<8, 512>(snop_impl::Ctx&, const SweepConsts&, const SolveConfig&, int, const double*, const double*, const double*, const double*, const double*, double*, double*, int32_t*, uint8_t*);
}  // namespace snop_si

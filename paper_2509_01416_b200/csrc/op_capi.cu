// op_capi.cu — SolutionOperator entry points (DeepONet / FNO / exact operator). Placeholder
// until the operator kernels land: every call reports that the operator is unavailable.
#include "snop_internal.h"

using namespace snop_impl;

extern "C" {

static snop_status not_built() {
  set_error("neural-operator kernels are not built in this revision");
  return SNOP_INVALID_ARGUMENT;
}

snop_status snop_deeponet_create(snop_ctx*, const snop_grid*, double, double, int32_t, int32_t, const int32_t*,
                                 const float*, int32_t, const int32_t*, const float*, int32_t, float, snop_op** out) {
  if (out) *out = nullptr;
  return not_built();
}
snop_status snop_fno_create(snop_ctx*, const snop_grid*, double, double, int32_t, int32_t, int32_t, int32_t, int32_t,
                            const float*, snop_op** out) {
  if (out) *out = nullptr;
  return not_built();
}
snop_status snop_exact_operator_create(snop_ctx*, const snop_grid*, int32_t, double, double,
                                       const snop_solver_config*, snop_op** out) {
  if (out) *out = nullptr;
  return not_built();
}
snop_status snop_op_destroy(snop_op*) { return SNOP_OK; }
snop_status snop_op_predict(snop_ctx*, snop_op*, int32_t, int32_t, const double*, double*) { return not_built(); }
snop_status snop_recast_fixed_point(snop_ctx*, snop_op*, int32_t, int32_t, const double*, const double*, const double*,
                                    double, int32_t, int32_t, const double*, double*, int32_t*, int32_t*) {
  return not_built();
}
snop_status snop_precondition_fixed_source(snop_ctx*, snop_op*, int32_t, int32_t, int32_t, const double*,
                                           const double*, const double*, const double*, double, int32_t,
                                           const snop_solver_config*, double*, int32_t*, int32_t*, int32_t*,
                                           uint8_t*) {
  return not_built();
}

}  // extern "C"

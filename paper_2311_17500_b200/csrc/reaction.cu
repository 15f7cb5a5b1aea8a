// Reaction correction M_R x (placeholder until the fused quadrature sweep lands).
#include "common.cuh"

namespace mi {
int reaction_apply(mi_ctx* c, const double* x, double* y) {
  (void)c; (void)x; (void)y;
  set_error("reaction correction not available");
  return MI_ERR_STATE;
}
}  // namespace mi

extern "C" {
int mi_op_set_reaction(mi_ctx* c, const double*, const double*, double, double, double, int, const int*, int,
                       const double*, const int*, const double*, const double*, const int*, const double*) {
  (void)c;
  mi::set_error("reaction correction not available");
  return MI_ERR_STATE;
}
int mi_op_clear_reaction(mi_ctx* c) {
  if (c) c->reaction_on = false;
  return MI_OK;
}
}

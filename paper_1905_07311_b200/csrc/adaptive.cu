// Adaptive R-STHOSVD (Alg 5) — implemented in a later milestone.
#include "orchestrate.h"

namespace rt {

rtucker_result *run_adaptive(Ctx &c, const rtucker_dense_desc *X, double tol, int block, const double *mode_tol,
                             const int32_t *order, uint64_t seed, uint32_t flags) {
  (void)c; (void)X; (void)tol; (void)block; (void)mode_tol; (void)order; (void)seed; (void)flags;
  throw Error(RTUCKER_EUNSUPPORTED, "rtucker_adaptive: not built yet");
}

}  // namespace rt

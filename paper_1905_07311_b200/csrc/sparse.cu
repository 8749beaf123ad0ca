// SP-STHOSVD (Alg 6) — implemented in a later milestone.
#include "orchestrate.h"

namespace rt {

void sketch_coo(Ctx &, const CooDev &, int, int, uint64_t, double *) {
  throw Error(RTUCKER_EUNSUPPORTED, "sparse sketch: not built yet");
}
void srrqr(Ctx &, const double *, int64_t, int, double, int64_t *, double *, int *) {
  throw Error(RTUCKER_EUNSUPPORTED, "srrqr: not built yet");
}
int64_t coo_select(Ctx &, const CooDev &, int, const int64_t *, int, int32_t *const *, void *) {
  throw Error(RTUCKER_EUNSUPPORTED, "coo_select: not built yet");
}
rtucker_result *run_sparse_sthosvd(Ctx &, const rtucker_coo_desc *, const int64_t *, int, uint64_t,
                                   const int32_t *, double, uint32_t) {
  throw Error(RTUCKER_EUNSUPPORTED, "rtucker_sparse_sthosvd: not built yet");
}

}  // namespace rt

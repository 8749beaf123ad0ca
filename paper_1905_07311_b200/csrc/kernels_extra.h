#pragma once
#include "kernels.h"

namespace rt {
// out (L x J x R, fp64) = X (L x I x R) x_n M, M: J x I column-major with leading dim ldm.
void ttm_expand(Ctx &c, const void *X, DT in, ModeView v, const double *M, int64_t ldm, int64_t J,
                double *out);
// y (ext x ell) -> rows off.. of Y (I x ell, zeroed); cov[off .. off+ext) = 1 (coverage column)
void place_rows(Ctx &c, const double *y, int64_t ext, int ell, int64_t off, int64_t I, double *Y, double *cov);
// sets ST_SHARD_LAYOUT in the status word unless every cov[i] == 1
void check_cover(Ctx &c, const double *cov, int64_t I);
// out = *normsq - sum_{i<r} w[i]
// out = sum_{i<r} w_i (||U_B(:, :r)^T B||^2 = ||G||^2 after the shrink, without forming G)
void sum_top_eigs(Ctx &c, const double *w, int r, double *out);
void residual_from_eigs(Ctx &c, const double *w, int r, const double *normsq, double *out);
}  // namespace rt

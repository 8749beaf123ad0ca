#pragma once
#include "kernels.h"

namespace rt {
// out (L x J x R, fp64) = X (L x I x R) x_n M, M: J x I column-major with leading dim ldm.
void ttm_expand(Ctx &c, const void *X, DT in, ModeView v, const double *M, int64_t ldm, int64_t J,
                double *out);
void rows_scatter(Ctx &c, const double *g, int nranks, int64_t ext, int ell, const int64_t *offs,
                  const int64_t *exts, int64_t I, double *Y);
// out = *normsq - sum_{i<r} w[i]
void residual_from_eigs(Ctx &c, const double *w, int r, const double *normsq, double *out);
}  // namespace rt

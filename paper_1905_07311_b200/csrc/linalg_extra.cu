// Auxiliary device kernels for the orchestrator (layout moves and expansion products).
#include "kernels_extra.h"

namespace rt {

namespace {

// out(l, j, r) = sum_{i<I} M[j + ldm*i] * X(l, i, r), M is J x I column-major (fp64).
// Used to expand a Tucker core (measurement helper rtucker_rel_error) where J is large
// and I (a rank) is small.
template <typename Tin>
__global__ void ttm_expand_kernel(const Tin *__restrict__ X, int64_t L, int64_t I, int64_t R,
                                  const double *__restrict__ M, int64_t ldm, int64_t J,
                                  double *__restrict__ out) {
  const int64_t n = L * J * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e % L;
    const int64_t t = e / L;
    const int64_t j = t % J, r = t / J;
    double s = 0.0;
    for (int64_t i = 0; i < I; ++i) s += M[j + ldm * i] * (double)X[l + L * (i + I * r)];
    out[e] = s;
  }
}

// Local rows y (ext x ell, column-major) into the zeroed global buffer Y (I x ell) at row
// offset off, and the coverage column cov[off .. off + ext) = 1.
__global__ void place_rows_kernel(const double *__restrict__ y, int64_t ext, int ell, int64_t off, int64_t I,
                                  double *__restrict__ Y, double *__restrict__ cov) {
  const int64_t n = ext * (ell + 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % ext, k = e / ext;
    if (k < ell) Y[off + i + I * k] = y[i + ext * k];
    else cov[off + i] = 1.0;
  }
}

// After the sum over ranks every row must be covered exactly once.
__global__ void check_cover_kernel(const double *__restrict__ cov, int64_t I, unsigned *__restrict__ status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < I; i += (int64_t)gridDim.x * blockDim.x)
    if (cov[i] != 1.0) atomicOr(status, (unsigned)ST_SHARD_LAYOUT);
}

__global__ void sum_first_kernel(const double *__restrict__ w, int r, const double *__restrict__ nsq,
                                 double *__restrict__ out) {
  double s = 0.0;
  for (int i = 0; i < r; ++i) s += w[i];
  *out = *nsq - s;
}

__global__ void sum_top_kernel(const double *__restrict__ w, int r, double *__restrict__ out) {
  double s = 0.0;
  for (int i = 0; i < r; ++i) s += w[i];  // the order of factor_sign_kernel's sum
  *out = s;
}

}  // namespace

void ttm_expand(Ctx &c, const void *X, DT in, ModeView v, const double *M, int64_t ldm, int64_t J,
                double *out) {
  const int64_t n = v.L * J * v.R;
  const int g = std::max(1, std::min(8192, ceil_div(n, 256)));
  if (in == DT::F64)
    RT_LAUNCH(c, ttm_expand_kernel<double>, g, 256, 0, (const double *)X, v.L, v.I, v.R, M, ldm, J, out);
  else
    RT_LAUNCH(c, ttm_expand_kernel<float>, g, 256, 0, (const float *)X, v.L, v.I, v.R, M, ldm, J, out);
}

void place_rows(Ctx &c, const double *y, int64_t ext, int ell, int64_t off, int64_t I, double *Y, double *cov) {
  const int64_t n = ext * (ell + 1);
  const int gr = std::max(1, std::min(4096, ceil_div(n, 256)));
  RT_LAUNCH(c, place_rows_kernel, gr, 256, 0, y, ext, ell, off, I, Y, cov);
}

void check_cover(Ctx &c, const double *cov, int64_t I) {
  RT_LAUNCH(c, check_cover_kernel, std::max(1, std::min(64, ceil_div(I, 256))), 256, 0, cov, I, c.status);
}

void sum_top_eigs(Ctx &c, const double *w, int r, double *out) {
  RT_LAUNCH(c, sum_top_kernel, 1, 1, 0, w, r, out);
}

void residual_from_eigs(Ctx &c, const double *w, int r, const double *normsq, double *out) {
  RT_LAUNCH(c, sum_first_kernel, 1, 1, 0, w, r, normsq, out);
}

}  // namespace rt

// Host-side launchers of the librtucker kernels (one translation unit per family).
#pragma once
#include "common.cuh"

namespace rt {

enum class DT { F32 = 0, F64 = 1 };
inline size_t dt_size(DT t) { return t == DT::F32 ? 4 : 8; }

// (L, I, R) view of mode n of a first-mode-fastest tensor: element (l, i, r) at
// l + L*(i + I*r); unfolding column c = l + L*r.
struct ModeView {
  int64_t L, I, R;
};
inline ModeView mode_view(const int64_t *dims, int d, int n) {
  ModeView v{1, dims[n], 1};
  for (int k = 0; k < n; ++k) v.L *= dims[k];
  for (int k = n + 1; k < d; ++k) v.R *= dims[k];
  return v;
}

// ---- sketch.cu ---------------------------------------------------------------------
// Y (I x ell, fp64 col-major) = X_(n) Omega_n(:, k0:k0+ell) with Omega rows indexed by
// c + col_offset (global column).  normsq (optional, device scalar) <- ||X||_F^2.
// mul_f64: multiply in fp64 (else fp32 products with fp64 accumulation every 32 terms).
// Normals (reading R3): products in fp32 (FAST) draw fp32 normals; products in fp64 draw fp64
// normals unless normals_f32 (fp32 input under the HYBRID policy, whose later passes run in
// fp64 on fp64 intermediates but keep the fp32 data's Omega).
// colmax (optional, mode-1 fp32 tcgen05 path only): gets max_i |X(i, c)| (fp32 bits, atomic
// max into a zeroed buffer) for every unfolding column c - the Ozaki B-pass's column scales.
void sketch_dense(Ctx &c, const void *X, DT in, ModeView v, int mode, int ell, int64_t k0,
                  uint64_t seed, int64_t col_offset, bool mul_f64, double *Y, double *normsq,
                  bool normals_f32 = false, uint32_t *colmax = nullptr);

// sketch_tc.cu: tcgen05 3xTF32 variant for fp32 data with L == 1 (MN-major rows); returns
// false when the shape is outside its envelope.
bool sketch_tc_mn(Ctx &c, const float *X, ModeView v, int mode, int ell, int64_t k0, uint64_t seed,
                  int64_t col_offset, double *Y, double *normsq, uint32_t *colmax = nullptr);
bool sketch_tc_enabled();
// bpass_tc.cu: B = Q^T X_(n) (B[k + ell c]) for fp32 X with L == 1 on tcgen05 (3xTF32).
bool bpass_tc_mn(Ctx &c, const float *X, ModeView v, const double *Q, int64_t ldq, int ell, void *B, bool out_f64);

// Y (I x ell) = X_(n) Om_(n)^T with an explicit fp64 (L, ell, R) tensor Om in place of Omega
// (subspace iteration: Y = X_(n) Z with Z = B'^T), fp64 products, ell <= 64.
void sketch_explicit(Ctx &c, const void *X, DT in, ModeView v, const double *Om, int ell, double *Y);
// Deferred shrink (R-STHOSVD): the explicit sketch tensor Om (L', ell, R') of the
// mode-m unfolding of B (G's dims gdims except mode n, which B holds at ell_n) such that
// B_(m) Om = G_(m) Omega_m for G = B x_n V(:, :gdims[n])^T, V (ell_n x ell_n, col-major),
// Omega_m the on-the-fly Gaussian of mode m (columns 0..ell-1, unsharded).
void omega_fold(Ctx &c, const int64_t *gdims, int d, int n, int m, int ell_n, const double *V, int ell, uint64_t seed,
                bool normals_f32, double *Om);
// Rinv (n x n, column-major upper) = R^{-1} of the Cholesky factor G = R^T R of an SPD Gram
// (subspace iteration's re-orthonormalisation); *bad = 1 on a non-positive pivot.
void chol_rinv(Ctx &c, const double *G, int n, double *Rinv, int *bad);
// Generates Omega rows for given columns (debug / parity).
void omega_rows(Ctx &c, DT out, uint64_t seed, int mode, const int64_t *cols, int64_t n,
                int ell, int64_t k0, void *dst);
void philox_raw(Ctx &c, const uint32_t *ctr, int64_t n, uint32_t k0, uint32_t k1, uint32_t *out);

// ---- ttm.cu ------------------------------------------------------------------------
// out = X x_n A^T with A (I x J, fp64 col-major, leading dim lda): out(l, j, r) = sum_i A[i,j] X(l,i,r).
// out may be null (Gram-only pass).  gram (optional, J x J fp64) <- B_(n) B_(n)^T of the
// (stored-precision) output.
// Ozaki-style mode-1 B-pass on the int8 tensor cores (bpass_ozaki.cu); false if not applicable.
// colmax: column maxima from the mode-1 sketch (sketch_dense), or null (computed here).
bool ttm_ozaki(Ctx &c, const float *X, ModeView v, const double *A, int64_t lda, int J, double *out, double *gram,
               const uint32_t *colmax = nullptr);
bool ozaki_bpass_enabled();
// cm[p] = fp32 bits of max_i |X(i, p)| for X (I x P, column-major) - the Ozaki column scales.
void column_maxima(Ctx &c, const float *X, ModeView v, uint32_t *cm);  // max_i |X(l, i, r)| per l + L r
void ttm_dense(Ctx &c, const void *X, DT in, ModeView v, const double *A, int64_t lda, int J,
               void *out, DT outT, bool mul_f64, double *gram, const uint32_t *colmax = nullptr);

// Gram of the mode-n unfolding of B (mode size v.I): gram (v.I x v.I, fp64).
void mode_gram(Ctx &c, const void *B, DT t, ModeView v, double *gram);
// Same for fp64 B with v.L, v.I <= 64, slab by slab (B(:, :, r) contiguous).
void slab_gram(Ctx &c, const double *B, ModeView v, double *gram);

// ---- linalg.cu ---------------------------------------------------------------------
// gate (device int, optional): the kernels return immediately when *gate == 0.
void householder_qr(Ctx &c, const double *Y, int64_t m, int n, double *Q, const int *gate = nullptr);
// Hot-path thin QR: CholeskyQR2, with Householder recomputation when ill-conditioned.
// orth_tol > 0 (fp32 data): the one-cluster CholeskyQR2 stops after its first pass when the
// second pass's Gram shows ||Q^T Q - I||_max <= orth_tol (DESIGN reading R22).
void thin_qr(Ctx &c, const double *Y, int64_t m, int n, double *Q, double orth_tol = 0.0);
// w descending; sweeps (optional, device int) <- Jacobi sweeps used
// gate (device int, optional): the kernel returns immediately when *gate == 0.
void sym_eig(Ctx &c, const double *A, int n, double *w, double *V, int *sweeps = nullptr, const int *gate = nullptr);
// PSD Gram: pivoted Cholesky + one-sided Jacobi on the factor; eigenvectors accurate to
// ~eps sqrt(w_0 / w_k).  When the r_need-th eigenvalue is below 1e-8 w_0 the unpreconditioned
// sym_eig recomputes the result (device-side gate, no host sync).  n > 64 uses sym_eig.
// rel_acc: fp64 data (preconditioned Jacobi, relative accuracy); else the tridiagonal solver.
// A = Q U(:, 1:r) (m x r), canonical signs on A and U (reading R4b), and, when w is given,
// residual = normsq - sum_{i<r} w_i: one launch for ell <= 64.
void factor_epilogue(Ctx &c, const double *Q, int64_t m, int ell, double *U, int r, double *A, const double *w,
                     const double *normsq, double *residual);
void gram_eig(Ctx &c, const double *A, int n, double *w, double *V, int *sweeps = nullptr, int r_need = 1 << 30,
              bool rel_acc = false);
// Symmetric eigensolver for n <= 64 (trideig.cu): Householder tridiagonalisation, multisection,
// twisted-factorisation eigenvectors, one CTA; eigenvalues descending.  Returns false if n > 64.
bool trid_eig(Ctx &c, const double *A, int n, double *w, double *V, int *info = nullptr);
// Sign convention of reading R4b: for each column k < r of A (m x r) make the entry of
// largest magnitude positive (first on ties); the same sign is applied to column k of U
// (ell x r, leading dim ldu) so that the shrink U^T B stays consistent.
void canonical_signs(Ctx &c, double *A, int64_t m, int r, double *U, int64_t ldu, int ell);
// C (m x n) = op(A) (m x k) * B (k x n), fp64 col-major with leading dims.
void gemm_small(Ctx &c, bool transA, const double *A, int64_t lda, const double *B, int64_t ldb,
                double *C, int64_t ldc, int64_t m, int64_t n, int64_t k);
// C (m x n) = beta C + alpha op(A) B on the fp64 tensor cores (tiled, deterministic), column-major.
void gemm_f64(Ctx &c, bool transA, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
              int64_t ldc, int64_t m, int64_t n, int64_t k, double beta = 0.0, double alpha = 1.0);
// Batched variant (blockIdx.z = batch, element strides sA, sB, sC), op(B) = B^T with transB.
void gemm_f64_batched(Ctx &c, bool transA, bool transB, const double *A, int64_t lda, int64_t sA, const double *B,
                      int64_t ldb, int64_t sB, double *C, int64_t ldc, int64_t sC, int64_t m, int64_t n, int64_t k,
                      int64_t batch, double beta = 0.0, double alpha = 1.0);
// Gram C (K x K) = B_(n) B_(n)^T of an fp64 tensor stored (L, K, R), tensor cores, deterministic.
void gram_f64(Ctx &c, const double *B, int64_t L, int64_t K, int64_t R, double *C);
void convert(Ctx &c, const void *src, DT s, void *dst, DT d, int64_t n);
void sumsq(Ctx &c, const void *X, DT t, int64_t n, double *out);             // deterministic
void diff_sumsq(Ctx &c, const void *X, DT t, const double *Y, int64_t n, double *out);
void sum_vec(Ctx &c, const double *x, int64_t n, double *out);             // out = sum x
void sub_scalar(Ctx &c, const double *a, const double *b, double *out);   // out = a - b

// ---- sparse.cu ---------------------------------------------------------------------
struct CooDev {
  int d;
  int64_t dims[kMaxModes];
  int64_t nnz;
  const int32_t *idx[kMaxModes];
  const void *vals;
  DT vt;
};
// Y (I_n x ell, fp64) = G_(n) Omega_n for a COO tensor, summed in fixed point (deterministic)
// and over the ranks.  nnz_dev (optional): live nnz on the device (g.nnz is then an upper
// bound).  fs_dev (optional): the call's fixed-point scale (computed from g when null).
// normals_f64: fp64 Box-Muller normals (else fp32 normals; products in fp64).
void sketch_coo(Ctx &c, const CooDev &g, int mode, int ell, uint64_t seed, bool normals_f64, double *Y,
                const int64_t *nnz_dev = nullptr, const void *fs_dev = nullptr);
// Strong-RRQR (CPQR + maxvol, eta) on Q (m x l) in one cooperative kernel: sel sorted (device
// int64), A (m x l), swaps (device int); singular P^T Q sets the status word.
void srrqr(Ctx &c, const double *Q, int64_t m, int l, double eta, int64_t *sel, double *A, int *swaps_dev);
// Keep entries whose mode-n index is in sel (sorted, length l) and renumber it; the live input
// nnz is read from nnz_dev, the new nnz written to nnz_out (device).
void coo_select(Ctx &c, const CooDev &in, const int64_t *nnz_dev, int mode, const int64_t *sel, int l,
                int32_t *const *out_idx, void *out_vals, int64_t *nnz_out);

}  // namespace rt

// Dense fixed-rank algorithms: R-STHOSVD (Alg 3) and R-HOSVD (Alg 2,
// P:158-171), single GPU or sharded along the last mode, plus the
// measurement helper rel_error.  No host synchronisation on the fixed-rank path.
#include <algorithm>
#include <cstring>

#include "comm.h"
#include "kernels_extra.h"
#include "orchestrate.h"

namespace rt {

namespace {

// Precision policy for the passes (include/rtucker.h flags).  Passes over fp64
// data always multiply in fp64.  For fp32 data:
//   FP64    fp64 products, fp64 B and intermediates
//   FAST    fp32 products (flushed into fp64 accumulators), fp32 B and intermediates
//   HYBRID  fp32 products on the fp32 input X, fp64 B and intermediates (so every later
//           pass runs in fp64)
//   AUTO    FP64 while max l <= 12 (2l/4 flop/B under the DFMA ridge), else HYBRID
struct Policy {
  bool mul_f64;  // fp64 products when reading fp32 data
  DT store;      // precision of B and of the shrunk intermediates
};

Policy policy_for(DT in, uint32_t flags, int max_ell) {
  uint32_t acc = flags & RTUCKER_ACCUM_MASK;
  if (in == DT::F64) return Policy{true, DT::F64};
  if (acc == RTUCKER_ACCUM_AUTO) acc = max_ell <= 12 ? RTUCKER_ACCUM_FP64 : RTUCKER_ACCUM_HYBRID;
  if (acc == RTUCKER_ACCUM_FP64) return Policy{true, DT::F64};
  if (acc == RTUCKER_ACCUM_HYBRID) return Policy{false, DT::F64};
  return Policy{false, DT::F32};
}

int max_ell(const DenseIn &in, const int64_t *ranks, int p) {
  int64_t m = 1;
  for (int k = 0; k < in.d; ++k) m = std::max<int64_t>(m, std::min<int64_t>(ranks[k] + p, in.gdims[k]));
  return (int)m;
}

void check_ranks(const DenseIn &in, const int64_t *ranks, int p) {
  RT_REQUIRE(p >= 0, "p must be >= 0");
  for (int k = 0; k < in.d; ++k)
    RT_REQUIRE(ranks[k] >= 1 && ranks[k] <= in.gdims[k], "r_n must lie in [1, I_n]");
}

void fill_header(rtucker_result *r, const DenseIn &in, const int32_t *ord, uint64_t seed, uint32_t flags) {
  for (int k = 0; k < in.d; ++k) {
    r->dims[k] = in.gdims[k];
    r->order[k] = ord[k];
  }
  r->seed = seed;
  r->flags = flags;
}

// Sketch of the sharded last mode: local rows are complete.  Every rank writes its rows (and
// a coverage column of ones) into a zeroed global-size buffer at its own offset and the
// buffers are summed over the ranks: the rows come out bit-exact (x + 0 = x) with no host
// synchronisation or metadata exchange, and a device check flags shards that do not tile
// [0, I_d) (status word, reported as EINVAL at the next synchronising call).  normsq gets the
// global ||G||^2.
void sketch_last_sharded(Ctx &c, const DenseIn &in, const void *G, DT gt, const int64_t *cur, int ell,
                         uint64_t seed, bool mulf64, double *Y, double *normsq, bool n32) {
  const int d = in.d, n = d - 1;
  const ModeView v = mode_view(cur, d, n);  // v.I = local extent
  const int64_t ext = v.I, I = in.gdims[n];
  // [Y (I x ell) | ||G||^2 | coverage (I)]
  DevBuf<double> buf(c, (size_t)I * ell + 1 + (size_t)I);
  buf.zero();
  DevBuf<double> ytmp(c, (size_t)ext * ell);
  sketch_dense(c, G, gt, v, n, ell, 0, seed, 0, mulf64, ytmp.p, buf.p + (size_t)I * ell, n32);
  place_rows(c, ytmp.p, ext, ell, in.offset, I, buf.p, buf.p + (size_t)I * ell + 1);
  allreduce_sum_f64(c, buf.p, buf.n);
  check_cover(c, buf.p + (size_t)I * ell + 1, I);
  RT_CUDA(cudaMemcpyAsync(Y, buf.p, sizeof(double) * I * ell, cudaMemcpyDeviceToDevice, c.stream));
  RT_CUDA(cudaMemcpyAsync(normsq, buf.p + (size_t)I * ell, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
}

// q steps of randomized subspace iteration on the range basis Q (I x ell) of G_(n) (P:550-553,
// Halko et al.'s scheme as the paper cites it): B = Q^T G_(n) (the B-pass, with its Gram),
// Z = B^T re-orthonormalised by the Cholesky factor of that Gram (B' = R^{-T} B), Y = G_(n) Z
// (the sketch kernel with Z in place of Omega), Q = qr(Y).  fp64 throughout.
void power_iterate(Ctx &c, const void *G, DT gt, ModeView v, int ell, int q, bool mul_f64, double *Q,
                   const uint32_t *colmax) {
  const int64_t I = v.I;
  for (int it = 0; it < q; ++it) {
    DevBuf<double> B(c, (size_t)v.L * ell * v.R), B2(c, (size_t)v.L * ell * v.R), gram(c, (size_t)ell * ell),
        Rinv(c, (size_t)ell * ell), Y(c, (size_t)I * ell);
    DevBuf<int> bad(c, 1);
    bad.zero();
    ttm_dense(c, G, gt, v, Q, I, ell, B.p, DT::F64, mul_f64, gram.p, colmax);
    chol_rinv(c, gram.p, ell, Rinv.p, bad.p);
    ttm_dense(c, B.p, DT::F64, ModeView{v.L, ell, v.R}, Rinv.p, ell, ell, B2.p, DT::F64, true, nullptr);
    sketch_explicit(c, G, gt, v, B2.p, ell, Y.p);
    thin_qr(c, Y.p, I, ell, Q);
  }
}

// fp32 data: the sketch's range basis may stop at one CholeskyQR pass when Q^T Q is within 1e-10
// of I (reading R22: 1e-10 is far below the 1e-5 criteria and fp32's own 6e-8); fp64 data keeps
// both passes (orthonormal to working precision).
double qr_orth_tol(const DenseIn &in) { return in.dt == DT::F32 ? 1e-10 : 0.0; }

void copy_residuals(Ctx &c, rtucker_result *r, const double *scal, int d, int first_mode) {
  for (int k = 0; k < d; ++k)
    RT_CUDA(cudaMemcpyAsync(&r->mode_residual_sq[k], scal + 2 * k + 1, sizeof(double), cudaMemcpyDeviceToHost,
                            c.stream));
  RT_CUDA(cudaMemcpyAsync(&r->norm_sq, scal + 2 * first_mode, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
}

}  // namespace

// Deterministic comparators (RTUCKER_EXACT_SVD, NEXT-4): HOSVD and STHOSVD from
// the eigenpairs of the full unfolding's Gram G_(n) G_(n)^T (the Gram route of Alg 1 line 4 with
// Q = I): no sketch, fp64 products and intermediates, signs per R4b.
rtucker_result *run_exact(Ctx &c, const rtucker_dense_desc *X, const int64_t *ranks, const int32_t *order,
                          uint32_t flags, bool st) {
  DenseIn in;
  prepare_dense(c, X, in);
  RT_REQUIRE(!in.sharded, "RTUCKER_EXACT_SVD: unsharded inputs only");
  check_ranks(in, ranks, 0);
  const int d = in.d;
  int32_t ord[kMaxModes];
  if (st) check_order(order, d, ord, in.gdims, false);
  else for (int k = 0; k < d; ++k) ord[k] = k;
  ResultGuard rg{c, new_result(d)};
  rtucker_result *res = rg.r;
  fill_header(res, in, ord, 0, flags);
  DevBuf<double> scal(c, 2 * (size_t)d);
  scal.zero();
  int64_t cur[kMaxModes];
  memcpy(cur, in.gdims, sizeof cur);
  const void *G = in.ptr;
  DT gt = in.dt;
  DevBuf<unsigned char> gown;
  for (int jj = 0; jj < d; ++jj) {
    const int n = ord[jj];
    const int64_t *dims = st ? cur : in.gdims;
    const void *src = st ? G : in.ptr;
    const DT stt = st ? gt : in.dt;
    const ModeView v = mode_view(dims, d, n);
    const int I = (int)v.I, r = (int)std::min<int64_t>(ranks[n], v.I);
    DevBuf<double> gram(c, (size_t)I * I), w(c, I), V(c, (size_t)I * I);
    {
      PhaseScope ps(c, PH_BPASS, jj);
      sumsq(c, src, stt, v.L * v.I * v.R, scal.p + 2 * n);
      if (stt == DT::F64 && I > 64) gram_f64(c, (const double *)src, v.L, I, v.R, gram.p);
      else mode_gram(c, src, stt, v, gram.p);
    }
    double *A = (double *)dev_alloc(c, sizeof(double) * I * r);
    res->factors[n] = A;
    {
      PhaseScope ps(c, PH_EIG, jj);
      // relative-accuracy Jacobi for small fp64 Grams; the tridiagonal solver above 64 (the
      // unpreconditioned grid Jacobi can miss its sweep cap on these nearly singular Grams)
      gram_eig(c, gram.p, I, w.p, V.p, nullptr, r, in.dt == DT::F64 && I <= 64);
      RT_CUDA(cudaMemcpyAsync(A, V.p, sizeof(double) * I * r, cudaMemcpyDeviceToDevice, c.stream));
      canonical_signs(c, A, I, r, V.p, I, I);
      residual_from_eigs(c, w.p, r, scal.p + 2 * n, scal.p + 2 * n + 1);
    }
    res->ranks[n] = r;
    res->ell[n] = I;
    if (st) {  // G_(n) <- U(:, 1:r)^T G_(n)
      PhaseScope ps(c, PH_SHRINK, jj);
      DevBuf<unsigned char> Gn(c, (size_t)v.L * r * v.R * sizeof(double));
      ttm_dense(c, G, gt, v, V.p, I, r, Gn.p, DT::F64, true, nullptr);
      gown = std::move(Gn);
      G = gown.p;
      gt = DT::F64;
      cur[n] = r;
    }
  }
  if (!st) {  // G = X x_1 A_1^T ... x_d A_d^T
    PhaseScope ps(c, PH_SHRINK, 0);
    DevBuf<unsigned char> g0, g1;
    for (int n = 0; n < d; ++n) {
      const ModeView v = mode_view(cur, d, n);
      const int rr = (int)res->ranks[n];
      DevBuf<unsigned char> &dst = (G == g0.p) ? g1 : g0;
      dst.alloc(c, (size_t)v.L * rr * v.R * sizeof(double));
      ttm_dense(c, G, gt, v, (const double *)res->factors[n], in.gdims[n], rr, dst.p, DT::F64, true, nullptr);
      G = dst.p;
      gt = DT::F64;
      cur[n] = rr;
    }
    gown = std::move(G == g0.p ? g0 : g1);
    G = gown.p;
  }
  const int64_t ncore = prod(cur, d);
  res->core = dev_alloc(c, sizeof(double) * ncore);
  convert(c, G, gt, res->core, DT::F64, ncore);
  copy_residuals(c, res, scal.p, d, ord[0]);
  finish_result(c, res, flags);
  return rg.release();
}

rtucker_result *run_sthosvd(Ctx &c, const rtucker_dense_desc *X, const int64_t *ranks, int p, uint64_t seed,
                            const int32_t *order, uint32_t flags) {
  if (flags & RTUCKER_EXACT_SVD) return run_exact(c, X, ranks, order, flags, true);
  DenseIn in;
  prepare_dense(c, X, in);
  check_ranks(in, ranks, p);
  int32_t ord[kMaxModes];
  check_order(order, in.d, ord, in.gdims, in.sharded);
  const Policy pol = policy_for(in.dt, flags, max_ell(in, ranks, p));
  const int d = in.d;
  const int power = (int)((flags & RTUCKER_POWER_MASK) >> 12);
  if (power > 0 && in.sharded) throw Error(RTUCKER_EUNSUPPORTED, "subspace iteration: unsharded inputs only");
  ResultGuard rg{c, new_result(d)};
  rtucker_result *res = rg.r;
  fill_header(res, in, ord, seed, flags);

  int64_t cur[kMaxModes], gcur[kMaxModes];
  memcpy(cur, in.ldims, sizeof cur);
  memcpy(gcur, in.gdims, sizeof gcur);
  const void *G = in.ptr;
  DT gt = in.dt;
  DevBuf<unsigned char> gown;
  DevBuf<double> scal(c, 2 * (size_t)d);
  scal.zero();
  struct Deferred {  // the previous mode's unshrunk B and its eigenpairs (deferred shrink)
    bool on = false;
    int n = 0, ell = 0;
    DevBuf<unsigned char> B;
    DevBuf<double> V, w;
  } dfr;

  for (int jj = 0; jj < d; ++jj) {
    const int n = ord[jj];
    int ell, rr;
    rank_caps(gcur, d, n, ranks[n], p, flags & RTUCKER_STRICT, ell, rr);
    const ModeView v = mode_view(cur, d, n);
    const bool last_sharded = in.sharded && n == d - 1;
    const int64_t Ig = gcur[n];

    // ---- line 2 of Alg 3 / line 1 of Alg 1: Y = G_(n) Omega_n   (+ ||G||^2)
    DevBuf<double> Y(c, (size_t)Ig * ell + 1);
    // fp32 input, HYBRID, L == 1: the sketch also records the column maxima that scale the
    // Ozaki B-pass of the same pass over X (bpass_ozaki.cu)
    DevBuf<uint32_t> colmax;
    if (gt == DT::F32 && !pol.mul_f64 && v.L == 1 && !last_sharded && ozaki_bpass_enabled()) {
      colmax.alloc(c, (size_t)v.R);
      colmax.zero();
    }
    {
      PhaseScope ps(c, PH_SKETCH, jj);
      if (dfr.on) {
        // deferred shrink of the previous mode: Y = G_(n) Omega_n = B_(n) Om with Om = Omega_n
        // folded with U_B (omega_fold), ||G||^2 = the sum of its kept eigenvalues
        int64_t cb[kMaxModes];
        memcpy(cb, cur, sizeof cb);
        cb[dfr.n] = dfr.ell;
        const ModeView vB = mode_view(cb, d, n);
        DevBuf<double> Om(c, (size_t)vB.L * ell * vB.R);
        omega_fold(c, cur, d, dfr.n, n, dfr.ell, dfr.V.p, ell, seed, in.dt == DT::F32 && !pol.mul_f64, Om.p);
        sketch_explicit(c, dfr.B.p, DT::F64, vB, Om.p, ell, Y.p);
        sum_top_eigs(c, dfr.w.p, (int)cur[dfr.n], scal.p + 2 * n);
      } else if (!last_sharded) {
        sketch_dense(c, G, gt, v, n, ell, 0, seed, col_offset_for(in, cur, n), pol.mul_f64, Y.p, Y.p + Ig * ell,
                     in.dt == DT::F32 && !pol.mul_f64, colmax.p);
        allreduce_sum_f64(c, Y.p, (size_t)Ig * ell + 1);
        RT_CUDA(cudaMemcpyAsync(scal.p + 2 * n, Y.p + Ig * ell, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
      } else {
        sketch_last_sharded(c, in, G, gt, cur, ell, seed, pol.mul_f64, Y.p, scal.p + 2 * n,
                            in.dt == DT::F32 && !pol.mul_f64);
      }
    }
    // ---- Alg 1 line 2: thin QR
    DevBuf<double> Q(c, (size_t)Ig * ell);
    {
      PhaseScope ps(c, PH_QR, jj);
      thin_qr(c, Y.p, Ig, ell, Q.p, qr_orth_tol(in));
    }
    Y.release();
    if (power > 0) {  // subspace iteration (NEXT-3)
      PhaseScope ps(c, PH_OTHER, jj);
      power_iterate(c, G, gt, v, ell, power, pol.mul_f64 || gt == DT::F64, Q.p, colmax.p);
    }
    // ---- Alg 1 line 3: B = Q^T G_(n)   (+ Gram B B^T)
    DevBuf<unsigned char> B(c, (size_t)v.L * ell * v.R * dt_size(pol.store));
    DevBuf<double> gram(c, (size_t)ell * ell);
    PhaseScope ps_b(c, PH_BPASS, jj);
    if (dfr.on) {
      // B = Q^T G_(n) = (B_prev x_n Q^T) x_prev U_B^T: the long product on B_prev, then the short
      // ell_prev -> r_prev one; the Gram of the result separately
      int64_t cb[kMaxModes];
      memcpy(cb, cur, sizeof cb);
      cb[dfr.n] = dfr.ell;
      const ModeView vB = mode_view(cb, d, n);
      DevBuf<double> Cq(c, (size_t)vB.L * ell * vB.R);
      ttm_dense(c, dfr.B.p, DT::F64, vB, Q.p, Ig, ell, Cq.p, DT::F64, pol.mul_f64, nullptr);
      cb[n] = ell;
      ttm_dense(c, Cq.p, DT::F64, mode_view(cb, d, dfr.n), dfr.V.p, dfr.ell, (int)cur[dfr.n], B.p, DT::F64,
                pol.mul_f64, nullptr);
      if (v.L <= 64) slab_gram(c, (const double *)B.p, ModeView{v.L, ell, v.R}, gram.p);
      else mode_gram(c, B.p, DT::F64, ModeView{v.L, ell, v.R}, gram.p);
      dfr = Deferred{};
    } else if (!last_sharded) {
      ttm_dense(c, G, gt, v, Q.p, Ig, ell, B.p, pol.store, pol.mul_f64, gram.p, colmax.p);
      allreduce_sum_f64(c, gram.p, (size_t)ell * ell);
    } else {
      ttm_dense(c, G, gt, v, Q.p + in.offset, Ig, ell, B.p, pol.store, pol.mul_f64, nullptr);
      allreduce_sum(c, B.p, (size_t)v.L * ell, pol.store == DT::F64);
      DevBuf<double> b64;
      const double *bp = (const double *)B.p;
      if (pol.store != DT::F64) {
        b64.alloc(c, (size_t)v.L * ell);
        convert(c, B.p, pol.store, b64.p, DT::F64, v.L * ell);
        bp = b64.p;
      }
      gemm_small(c, true, bp, v.L, bp, v.L, gram.p, ell, ell, ell, v.L);
    }
    ps_b.next(PH_EIG);
    // ---- Alg 1 line 4: thin SVD of B through the eigenpairs of its Gram
    DevBuf<double> w(c, ell), V(c, (size_t)ell * ell);
    gram_eig(c, gram.p, ell, w.p, V.p, nullptr, rr, in.dt == DT::F64);
    // ---- Alg 1 line 5: A_n = Q U_B(:, 1:r)
    double *A = nullptr;
    A = (double *)dev_alloc(c, sizeof(double) * Ig * rr);
    res->factors[n] = A;
    // A_n = Q U_B(:, 1:r), signs (reading R4b; the shrink uses the signed U_B), residual
    factor_epilogue(c, Q.p, Ig, ell, V.p, rr, A, w.p, scal.p + 2 * n, scal.p + 2 * n + 1);
    ps_b.next(PH_SHRINK);
    // ---- Alg 3 line 6: G_(n) <- Sigma_hat V_hat^T = U_B(:, 1:r)^T B
    // Deferred: when the next mode's sketch and B-pass are cheaper on B than the
    // shrink itself, G is not formed; the next mode works on B with U_B folded into its
    // Omega and applied to its (small) B-pass output.  Mathematically the same products.
    const ModeView vb{v.L, ell, v.R};
    bool defer = false;
    if (!in.sharded && power == 0 && pol.store == DT::F64 && jj + 1 < d && v.L * ell * v.R >= (1 << 22)) {
      int64_t g2[kMaxModes];
      memcpy(g2, gcur, sizeof g2);
      g2[n] = rr;
      int ell2, rr2;
      rank_caps(g2, d, ord[jj + 1], ranks[ord[jj + 1]], p, false, ell2, rr2);
      defer = ell2 <= 64 && (int64_t)ell * rr > 2 * (int64_t)(ell - rr) * ell2;
    }
    if (defer) {
      dfr.on = true;
      dfr.n = n;
      dfr.ell = ell;
      dfr.B = std::move(B);
      dfr.V = std::move(V);
      dfr.w = std::move(w);
      gown.release();
      G = nullptr;
      gt = pol.store;
    } else {
      DevBuf<unsigned char> Gn(c, (size_t)v.L * rr * v.R * dt_size(pol.store));
      ttm_dense(c, B.p, pol.store, vb, V.p, ell, rr, Gn.p, pol.store, pol.mul_f64, nullptr);
      gown = std::move(Gn);
      G = gown.p;
      gt = pol.store;
    }
    cur[n] = rr;
    gcur[n] = rr;
    if (last_sharded) cur[n] = rr;  // core is replicated from here on
    res->ranks[n] = rr;
    res->ell[n] = ell;
  }
  const int64_t ncore = prod(cur, d);
  res->core = dev_alloc(c, sizeof(double) * ncore);
  convert(c, G, gt, res->core, DT::F64, ncore);
  copy_residuals(c, res, scal.p, d, ord[0]);
  if (c.capturing) res->internal = scal.p;  // graph template: the residual block lives in the arena
  finish_result(c, res, flags);
  return rg.release();
}

rtucker_result *run_hosvd(Ctx &c, const rtucker_dense_desc *X, const int64_t *ranks, int p, uint64_t seed,
                          uint32_t flags) {
  if (flags & RTUCKER_EXACT_SVD) return run_exact(c, X, ranks, nullptr, flags, false);
  DenseIn in;
  prepare_dense(c, X, in);
  check_ranks(in, ranks, p);
  const Policy pol = policy_for(in.dt, flags, max_ell(in, ranks, p));
  const int d = in.d;
  int32_t ord[kMaxModes];
  for (int k = 0; k < d; ++k) ord[k] = k;
  ResultGuard rg{c, new_result(d)};
  rtucker_result *res = rg.r;
  fill_header(res, in, ord, seed, flags);
  const bool want_core = !(flags & RTUCKER_NO_CORE);
  DevBuf<double> scal(c, 2 * (size_t)d);
  scal.zero();
  // B_1 = Q_1^T X_(1) is kept so that the core chain starts from U_B1^T B_1 (unsharded).
  const bool keep_b1 = want_core && !in.sharded && d > 1;
  DevBuf<unsigned char> B1;
  DevBuf<double> U1;
  int ell1 = 0;

  // Unsharded: the d modes are independent (Alg 2), so the small solves of mode n (QR after its
  // sketch, eigensolve after its B-pass: one CTA / cluster each) run on the context's side
  // stream while the main stream streams the next mode's sketch / B-pass over X.  Only the last
  // mode's QR and eigensolve stay exposed.  Event edges order the two streams (and become graph
  // edges under RTUCKER_GRAPH).
  const int power = (int)((flags & RTUCKER_POWER_MASK) >> 12);
  if (power > 0 && in.sharded) throw Error(RTUCKER_EUNSUPPORTED, "subspace iteration: unsharded inputs only");
  const bool overlap = !in.sharded && d > 1 && c.aux && power == 0;
  if (overlap) {
    // the persistent streaming kernels size their grids by c.num_sms: leave 4 SMs to the side
    // stream (a QR cluster of <= 4 CTAs, or one eigensolver CTA), restored at the join
    struct SmReserve {
      Ctx &c;
      int saved;
      explicit SmReserve(Ctx &cc) : c(cc), saved(cc.num_sms) { c.num_sms = std::max(8, c.num_sms - 4); }
      ~SmReserve() { c.num_sms = saved; }
    } reserve(c);
    DevBuf<double> Ys[kMaxModes], Qs[kMaxModes], grams[kMaxModes], ws[kMaxModes], Vs[kMaxModes];
    DevBuf<uint32_t> cms[kMaxModes];
    int ells[kMaxModes], rrs[kMaxModes];
    cudaEvent_t qdone[kMaxModes];  // Q_n ready on the side stream
    for (int n = 0; n < d; ++n) RT_CUDA(cudaEventCreateWithFlags(&qdone[n], cudaEventDisableTiming));
    for (int n = 0; n < d; ++n) {  // sketches on the main stream, QRs on the side stream
      rank_caps(in.gdims, d, n, ranks[n], p, flags & RTUCKER_STRICT, ells[n], rrs[n]);
      const int ell = ells[n];
      const ModeView v = mode_view(in.ldims, d, n);
      const int64_t Ig = in.gdims[n];
      Ys[n].alloc(c, (size_t)Ig * ell + 1);
      if (in.dt == DT::F32 && !pol.mul_f64 && (v.L == 1 || (v.L % 4) == 0) && ozaki_bpass_enabled()) {
        cms[n].alloc(c, (size_t)(v.L * v.R));
        cms[n].zero();
      }
      Qs[n].alloc(c, (size_t)Ig * ell);
      grams[n].alloc(c, (size_t)ell * ell);
      ws[n].alloc(c, ell);
      Vs[n].alloc(c, (size_t)ell * ell);
      {
        PhaseScope ps(c, PH_SKETCH, n);
        sketch_dense(c, in.ptr, in.dt, v, n, ell, 0, seed, 0, pol.mul_f64, Ys[n].p, Ys[n].p + Ig * ell,
                     in.dt == DT::F32 && !pol.mul_f64, cms[n].p);
        RT_CUDA(cudaMemcpyAsync(scal.p + 2 * n, Ys[n].p + Ig * ell, sizeof(double), cudaMemcpyDeviceToDevice,
                                c.stream));
      }
      stream_dep(c.stream, c.aux);
      OnStream os(c, c.aux);
      PhaseScope ps(c, PH_QR, n);
      thin_qr(c, Ys[n].p, Ig, ell, Qs[n].p, qr_orth_tol(in));
      RT_CUDA(cudaEventRecord(qdone[n], c.stream));
    }
    for (int n = 0; n < d; ++n) {  // B-passes on the main stream, eigensolves on the side stream
      const int ell = ells[n], rr = rrs[n];
      const ModeView v = mode_view(in.ldims, d, n);
      const int64_t Ig = in.gdims[n];
      RT_CUDA(cudaStreamWaitEvent(c.stream, qdone[n], 0));  // Q_n ready (not the earlier eigensolves)
      {
        PhaseScope ps(c, PH_BPASS, n);
        if (n == 0 && keep_b1) {
          B1.alloc(c, (size_t)v.L * ell * v.R * dt_size(pol.store));
          ttm_dense(c, in.ptr, in.dt, v, Qs[n].p, Ig, ell, B1.p, pol.store, pol.mul_f64, grams[n].p, cms[n].p);
        } else {
          ttm_dense(c, in.ptr, in.dt, v, Qs[n].p, Ig, ell, nullptr, pol.store, pol.mul_f64, grams[n].p, cms[n].p);
        }
      }
      double *A = (double *)dev_alloc(c, sizeof(double) * Ig * rr);
      res->factors[n] = A;
      if (n == 0 && keep_b1) U1.alloc(c, (size_t)ell * rr);
      stream_dep(c.stream, c.aux);
      OnStream os(c, c.aux);
      PhaseScope ps(c, PH_EIG, n);
      gram_eig(c, grams[n].p, ell, ws[n].p, Vs[n].p, nullptr, rr, in.dt == DT::F64);
      factor_epilogue(c, Qs[n].p, Ig, ell, Vs[n].p, rr, A, ws[n].p, scal.p + 2 * n, scal.p + 2 * n + 1);
      if (n == 0 && keep_b1) {
        RT_CUDA(cudaMemcpyAsync(U1.p, Vs[n].p, sizeof(double) * ell * rr, cudaMemcpyDeviceToDevice, c.stream));
        ell1 = ell;
      }
      res->ranks[n] = rr;
      res->ell[n] = ell;
    }
    stream_dep(c.aux, c.stream);  // join: factors, U_B1 and residuals ready; buffers freed after
    for (int n = 0; n < d; ++n) RT_CUDA(cudaEventDestroy(qdone[n]));
  }
  for (int n = 0; n < d && !overlap; ++n) {
    int ell, rr;
    rank_caps(in.gdims, d, n, ranks[n], p, flags & RTUCKER_STRICT, ell, rr);
    const ModeView v = mode_view(in.ldims, d, n);
    const bool last_sharded = in.sharded && n == d - 1;
    const int64_t Ig = in.gdims[n];
    DevBuf<double> Y(c, (size_t)Ig * ell + 1);
    DevBuf<uint32_t> colmax;  // column maxima for the Ozaki B-pass (fp32, HYBRID), recorded by the sketch
    if (in.dt == DT::F32 && !pol.mul_f64 && (v.L == 1 || (v.L % 4) == 0) && !last_sharded && ozaki_bpass_enabled()) {
      colmax.alloc(c, (size_t)(v.L * v.R));
      colmax.zero();
    }
    PhaseScope ps(c, PH_SKETCH, n);
    if (!last_sharded) {
      sketch_dense(c, in.ptr, in.dt, v, n, ell, 0, seed, col_offset_for(in, in.ldims, n), pol.mul_f64, Y.p,
                   Y.p + Ig * ell, in.dt == DT::F32 && !pol.mul_f64, colmax.p);
      allreduce_sum_f64(c, Y.p, (size_t)Ig * ell + 1);
      RT_CUDA(cudaMemcpyAsync(scal.p + 2 * n, Y.p + Ig * ell, sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    } else {
      sketch_last_sharded(c, in, in.ptr, in.dt, in.ldims, ell, seed, pol.mul_f64, Y.p, scal.p + 2 * n,
                          in.dt == DT::F32 && !pol.mul_f64);
    }
    ps.next(PH_QR);
    DevBuf<double> Q(c, (size_t)Ig * ell);
    thin_qr(c, Y.p, Ig, ell, Q.p, qr_orth_tol(in));
    if (power > 0) power_iterate(c, in.ptr, in.dt, v, ell, power, pol.mul_f64 || in.dt == DT::F64, Q.p, colmax.p);
    DevBuf<double> gram(c, (size_t)ell * ell);
    ps.next(PH_BPASS);
    if (!last_sharded) {
      if (n == 0 && keep_b1) {
        B1.alloc(c, (size_t)v.L * ell * v.R * dt_size(pol.store));
        ttm_dense(c, in.ptr, in.dt, v, Q.p, Ig, ell, B1.p, pol.store, pol.mul_f64, gram.p, colmax.p);
      } else {
        ttm_dense(c, in.ptr, in.dt, v, Q.p, Ig, ell, nullptr, pol.store, pol.mul_f64, gram.p, colmax.p);  // Gram only
      }
      allreduce_sum_f64(c, gram.p, (size_t)ell * ell);
    } else {
      // B_d = Q_d^T X_(d) sums over the sharded index: partial B, then allreduce (fp64)
      DevBuf<double> Bd(c, (size_t)v.L * ell);
      ttm_dense(c, in.ptr, in.dt, v, Q.p + in.offset, Ig, ell, Bd.p, DT::F64, true, nullptr);
      allreduce_sum_f64(c, Bd.p, (size_t)v.L * ell);
      gemm_small(c, true, Bd.p, v.L, Bd.p, v.L, gram.p, ell, ell, ell, v.L);
    }
    ps.next(PH_EIG);
    DevBuf<double> w(c, ell), V(c, (size_t)ell * ell);
    gram_eig(c, gram.p, ell, w.p, V.p, nullptr, rr, in.dt == DT::F64);
    double *A = nullptr;
    A = (double *)dev_alloc(c, sizeof(double) * Ig * rr);
    res->factors[n] = A;
    // A_n = Q U_B(:, 1:r), signs (reading R4b; the shrink uses the signed U_B), residual
    factor_epilogue(c, Q.p, Ig, ell, V.p, rr, A, w.p, scal.p + 2 * n, scal.p + 2 * n + 1);
    if (n == 0 && keep_b1) {
      U1.alloc(c, (size_t)ell * rr);
      RT_CUDA(cudaMemcpyAsync(U1.p, V.p, sizeof(double) * ell * rr, cudaMemcpyDeviceToDevice, c.stream));
      ell1 = ell;
    }
    res->ranks[n] = rr;
    res->ell[n] = ell;
  }
  if (want_core) {
    PhaseScope ps(c, PH_SHRINK, 0);
    // G = X x_1 A_1^T ... x_d A_d^T (Alg 2 line 5)
    int64_t cur[kMaxModes];
    memcpy(cur, in.ldims, sizeof cur);
    DevBuf<unsigned char> g0, g1;
    const void *G = in.ptr;
    DT gt = in.dt;
    int start = 0;
    if (keep_b1) {
      // G = B_1 x_1 U_B1(:, 1:r1)^T x_2 A_2^T ... x_d A_d^T (A_1^T X_(1) = U_B1^T B_1).  The
      // mode products commute, so they run in the order of their shrink ratio r_n / I_n,
      // smallest first (each product costs 2 r_n flop per element of its input): on C4 the
      // 800 -> 50 products before the 60 -> 50 one, 4.1 instead of 7.2 GFLOP (fp64).
      cur[0] = ell1;
      int ordc[kMaxModes];
      for (int k = 0; k < d; ++k) ordc[k] = k;
      std::stable_sort(ordc, ordc + d, [&](int a, int b) {
        return (double)res->ranks[a] / (double)cur[a] < (double)res->ranks[b] / (double)cur[b];
      });
      G = B1.p;
      gt = pol.store;
      for (int k = 0; k < d; ++k) {
        const int n = ordc[k];
        const ModeView v = mode_view(cur, d, n);
        const int rr = (int)res->ranks[n];
        DevBuf<unsigned char> &dst = (G == g0.p) ? g1 : g0;
        dst.alloc(c, (size_t)v.L * rr * v.R * dt_size(pol.store));
        if (n == 0) ttm_dense(c, G, gt, v, U1.p, ell1, rr, dst.p, pol.store, pol.mul_f64, nullptr);
        else ttm_dense(c, G, gt, v, (const double *)res->factors[n], in.gdims[n], rr, dst.p, pol.store, pol.mul_f64,
                       nullptr);
        G = dst.p;
        cur[n] = rr;
      }
      start = d;
    }
    for (int n = start; n < d; ++n) {
      const ModeView v = mode_view(cur, d, n);
      const bool last_sharded = in.sharded && n == d - 1;
      const int rr = (int)res->ranks[n];
      DevBuf<unsigned char> &dst = (G == g0.p) ? g1 : g0;
      dst.alloc(c, (size_t)v.L * rr * v.R * dt_size(last_sharded ? DT::F64 : pol.store));
      if (!last_sharded) {
        ttm_dense(c, G, gt, v, (const double *)res->factors[n], in.gdims[n], rr, dst.p, pol.store, pol.mul_f64,
                  nullptr);
        gt = pol.store;
      } else {
        ttm_dense(c, G, gt, v, (const double *)res->factors[n] + in.offset, in.gdims[n], rr, dst.p, DT::F64, true,
                  nullptr);
        allreduce_sum_f64(c, (double *)dst.p, (size_t)v.L * rr);
        gt = DT::F64;
      }
      G = dst.p;
      cur[n] = rr;
    }
    const int64_t ncore = prod(cur, d);
    res->core = dev_alloc(c, sizeof(double) * ncore);
    convert(c, G, gt, res->core, DT::F64, ncore);
  }
  copy_residuals(c, res, scal.p, d, 0);
  if (c.capturing) res->internal = scal.p;
  finish_result(c, res, flags);
  return rg.release();
}

// ||X - [G; A_1..A_d]||_F / ||X||_F: expand the core mode by mode (fp64) and take
// the squared difference with X on the device.  Unsharded inputs only.
double run_rel_error(Ctx &c, const rtucker_dense_desc *X, const rtucker_result *res) {
  DenseIn in;
  prepare_dense(c, X, in);
  RT_REQUIRE(!in.sharded, "rel_error: unsharded inputs only");
  RT_REQUIRE(res->d == in.d, "rel_error: mode count mismatch");
  RT_REQUIRE(res->memory == RTUCKER_DEVICE && res->core, "rel_error: needs a device-resident dense result");
  const int d = in.d;
  int64_t cur[kMaxModes];
  for (int k = 0; k < d; ++k) cur[k] = res->ranks[k];
  DevBuf<double> a, b;
  const double *G = (const double *)res->core;
  for (int n = 0; n < d; ++n) {
    const ModeView v = mode_view(cur, d, n);
    DevBuf<double> &dst = (G == a.p) ? b : a;
    dst.alloc(c, (size_t)v.L * in.gdims[n] * v.R);
    ttm_expand(c, G, DT::F64, v, (const double *)res->factors[n], in.gdims[n], in.gdims[n], dst.p);
    G = dst.p;
    cur[n] = in.gdims[n];
  }
  const int64_t N = prod(in.gdims, d);
  DevBuf<double> s(c, 2);
  diff_sumsq(c, in.ptr, in.dt, G, N, s.p);
  sumsq(c, in.ptr, in.dt, N, s.p + 1);
  double h[2];
  RT_CUDA(cudaMemcpyAsync(h, s.p, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  RT_CUDA(cudaStreamSynchronize(c.stream));
  RT_REQUIRE(h[1] > 0.0, "rel_error: ||X|| = 0");
  if (!std::isfinite(h[0]) || !std::isfinite(h[1])) throw Error(RTUCKER_ENUMERIC, "rel_error: non-finite norm");
  return std::sqrt(h[0] / h[1]);
}

}  // namespace rt

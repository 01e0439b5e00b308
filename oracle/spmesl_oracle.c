/*
 * SPMESL CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 implementation of what the SPMESL hot
 * path computes, written from the paper (arXiv 2203.15031, /root/reference/
 * PAPER.md, cited as P:<line>).  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline leg / --impl reference) may load this library.  The
 * product path (paper_2203_15031_b200/) never links, imports or calls it, and
 * shares no code, header, table or constant with it.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared -o liboracle.so spmesl_oracle.c -lm
 * (-ffp-contract=off: every a*b+c below is a rounded multiply followed by a
 * rounded add, exactly as written.)
 *
 * What it computes (each function cites its passage):
 *   oracle_standardize     P:305-307 "centered and scaled to X_k^T X_k = n" (reading g14: divisor n)
 *   oracle_soft_threshold  P:595 Soft_lambda(a) = sign(a)(|a|-lambda)_+
 *   oracle_scaled_lasso    Algorithm 1 on an arbitrary response y
 *   oracle_spmesl_columns  Algorithm 2 first loop: Algorithm 1 with
 *                          (x_k, X_{-k}, lambda0) for a list of columns k
 *   oracle_assemble        Algorithm 2 lines P:698-708 + Proposition 1
 *   oracle_symmetrize      Algorithm 2 lines P:709-719 / Eq. (symm)
 *   oracle_spmesl_fit      the whole Algorithm 2 pipeline
 *
 * Readings of silent/garbled passages (listed in DESIGN.md §3):
 *   g1  inner stop is the per-column criterion of Alg. 1, not Alg. 3's joint one.
 *   g3  both tolerances absolute.
 *   g4  the residual is recomputed from scratch at every outer boundary (Alg. 3).
 *   g5  sigma floor (sigma_floor argument, default 1e-8) — parity unpinned (design decision).
 *   g6  b_kk stored as 0 and row k skipped in column k's sweep.
 *   g15 constant column: s_k <= 1e-13 * max_i |x_ik| -> error (parity unpinned).
 *   g16 max_inner ends that inner loop (column flagged), max_outer retires the column.
 *   g18 |a| == lambda maps to +0.0.
 *   g22 Alg. 1 line 623 writes e_j without the l = j term; together with the
 *       "+ beta_j^[cur]" of line 625 that would double count coordinate j.  We
 *       read e_j as the full current residual y - X beta (Prop. 2, P:805,
 *       a_j = x_j^T E / n + beta^(j),[cur]); pinned by the lasso/brute-force tests.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_WARN_NOT_CONVERGED 1
#define ORACLE_ERR_ARG -1
#define ORACLE_ERR_CONSTANT_COLUMN -2
#define ORACLE_ERR_NONFINITE -3
#define ORACLE_ERR_OOM -6

/* column-major n x p: element (i, j) at X[i + j*n] */
#define COL(X, j, n) ((X) + (size_t)(j) * (size_t)(n))

/* centre each column and scale it so that x_k^T x_k = n. */
int oracle_standardize(const double* X, int64_t n, int64_t p, double* Xs, double* mu,
                       double* s, int64_t* bad_col) {
  if (n < 2 || p < 1) return ORACLE_ERR_ARG;
  for (int64_t k = 0; k < p; ++k) {
    const double* x = COL(X, k, n);
    double sum = 0.0, maxabs = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      if (!isfinite(x[i])) { if (bad_col) *bad_col = k; return ORACLE_ERR_NONFINITE; }
      sum = sum + x[i];
      if (fabs(x[i]) > maxabs) maxabs = fabs(x[i]);
    }
    double m = sum / (double)n;
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double c = x[i] - m;
      ss = ss + c * c;
    }
    double sk = sqrt(ss / (double)n);
    if (!(sk > 1e-13 * maxabs)) { if (bad_col) *bad_col = k; return ORACLE_ERR_CONSTANT_COLUMN; }
    mu[k] = m;
    s[k] = sk;
    double* xs = COL(Xs, k, n);
    for (int64_t i = 0; i < n; ++i) xs[i] = (x[i] - m) / sk;
  }
  return ORACLE_OK;
}

/* Soft_lambda(a) = sign(a) (|a| - lambda)_+ ; reading g18: result +0.0 when |a| <= lambda. */
double oracle_soft_threshold(double a, double lambda) {
  double m = fabs(a) - lambda;
  if (m > 0.0) return a > 0.0 ? m : -m;
  return 0.0;
}

/*
 * Algorithm 1: CD with warm start for the scaled lasso
 *   min_{beta, sigma} ||y - X beta||^2 / (2 n sigma) + sigma/2 + lambda0 ||beta||_1   (Eq. sc)
 * on the n x q column-major design X, skipping predictor `skip` (-1: none; Alg. 2 passes
 * X_{-k} by skipping column k in place, reading g6).
 * Outputs: beta[q] (beta[skip] = 0), sigma, outer iterations r, total sweeps, flags
 * (bit0 = outer converged, bit1 = some inner loop hit max_inner), optional
 * sigma_trace[max_outer+1] (sigma^(0..r)), optional margin[q] = |a_j| - lambda at the last
 * visit of j, optional resid[n] = the fresh residual of the last outer boundary.
 */
static int scaled_lasso_core(const double* X, int64_t n, int64_t q, const double* y,
                             int64_t skip, double lambda0, double delta, int32_t max_outer,
                             int32_t max_inner, double sigma_floor, double* beta,
                             double* sigma_out, int32_t* outer_out, int32_t* sweeps_out,
                             int32_t* flags_out, double* sigma_trace, double* margin,
                             double* resid) {
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  if (!r) return ORACLE_ERR_OOM;
  /* Require line P:608-609: sigma^(0) = 1, beta^(0) = 0 */
  double sigma = 1.0;
  for (int64_t j = 0; j < q; ++j) beta[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) r[i] = y[i]; /* r = y - X*0 */
  if (sigma_trace) sigma_trace[0] = sigma;
  int32_t outer = 0, sweeps = 0, flags = 0;
  for (;;) {
    double lambda = sigma * lambda0;
    int32_t inner = 0;
    double maxd;
    do {                                         /* inner repeat */
      maxd = 0.0;
      for (int64_t j = 0; j < q; ++j) {          /* cyclic ascending order */
        if (j == skip) continue;                 /* beta_kk = 0 fixed (reading g6) */
        const double* xj = COL(X, j, n);
        double dot = 0.0;
        for (int64_t i = 0; i < n; ++i) dot = dot + xj[i] * r[i];
        double z = dot / (double)n;              /* x_j^T e / n (reading g22) */
        double a = z + beta[j];
        double bn = oracle_soft_threshold(a, lambda);
        double d = beta[j] - bn;
        if (d != 0.0)                            /* e <- e + x_j (beta_cur - beta_next), Prop. 2 */
          for (int64_t i = 0; i < n; ++i) r[i] = r[i] + xj[i] * d;
        beta[j] = bn;
        if (fabs(d) > maxd) maxd = fabs(d);      /* ||beta^[next] - beta^[cur]||_inf */
        if (margin) margin[j] = fabs(a) - lambda;
      }
      ++sweeps;
      ++inner;
    } while (!(maxd < delta) && inner < max_inner);
    if (!(maxd < delta)) flags |= 2;             /* reading g16 */
    /* P:634 sigma^(r+1) = ||y - X beta^(r+1)||_2 / sqrt(n), residual recomputed (reading g4) */
    for (int64_t i = 0; i < n; ++i) r[i] = y[i];
    for (int64_t j = 0; j < q; ++j) {
      if (j == skip || beta[j] == 0.0) continue;
      const double* xj = COL(X, j, n);
      for (int64_t i = 0; i < n; ++i) r[i] = r[i] - xj[i] * beta[j];
    }
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) ss = ss + r[i] * r[i];
    double sn = sqrt(ss) / sqrt((double)n);
    if (sn < sigma_floor) sn = sigma_floor;      /* reading g5 */
    ++outer;
    if (sigma_trace) sigma_trace[outer] = sn;
    int done = fabs(sn - sigma) < delta;
    sigma = sn;
    if (done) { flags |= 1; break; }
    if (outer >= max_outer) break;               /* reading g16 */
  }
  *sigma_out = sigma;
  *outer_out = outer;
  *sweeps_out = sweeps;
  *flags_out = flags;
  if (resid) memcpy(resid, r, sizeof(double) * (size_t)n);
  free(r);
  return ORACLE_OK;
}

static int check_args(int64_t n, int64_t q, double lambda0, double delta, int32_t max_outer,
                      int32_t max_inner) {
  if (n < 1 || q < 1 || !(lambda0 >= 0.0) || !isfinite(lambda0) || !(delta > 0.0) ||
      max_outer < 1 || max_inner < 1)
    return ORACLE_ERR_ARG;
  return ORACLE_OK;
}

/* Algorithm 1 on an arbitrary response y (used by the oracle's own pins). */
int oracle_scaled_lasso(const double* X, int64_t n, int64_t q, const double* y, double lambda0,
                        double delta, int32_t max_outer, int32_t max_inner, double sigma_floor,
                        double* beta, double* sigma, int32_t* outer, int32_t* sweeps,
                        int32_t* flags, double* sigma_trace, double* margin, double* resid) {
  int rc = check_args(n, q, lambda0, delta, max_outer, max_inner);
  if (rc) return rc;
  return scaled_lasso_core(X, n, q, y, -1, lambda0, delta, max_outer, max_inner, sigma_floor,
                           beta, sigma, outer, sweeps, flags, sigma_trace, margin, resid);
}

/* The inner lasso of Alg. 1 at a fixed lambda (Eq. lasso), warm start from beta. */
int oracle_lasso_cd(const double* X, int64_t n, int64_t q, const double* y, double lambda,
                    double delta, int32_t max_inner, double* beta, int32_t* sweeps) {
  if (n < 1 || q < 1 || !(lambda >= 0.0) || !(delta > 0.0) || max_inner < 1) return ORACLE_ERR_ARG;
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  if (!r) return ORACLE_ERR_OOM;
  for (int64_t i = 0; i < n; ++i) r[i] = y[i];
  for (int64_t j = 0; j < q; ++j) {
    if (beta[j] == 0.0) continue;
    const double* xj = COL(X, j, n);
    for (int64_t i = 0; i < n; ++i) r[i] = r[i] - xj[i] * beta[j];
  }
  int32_t sw = 0;
  double maxd;
  do {
    maxd = 0.0;
    for (int64_t j = 0; j < q; ++j) {
      const double* xj = COL(X, j, n);
      double dot = 0.0;
      for (int64_t i = 0; i < n; ++i) dot = dot + xj[i] * r[i];
      double a = dot / (double)n + beta[j];
      double bn = oracle_soft_threshold(a, lambda);
      double d = beta[j] - bn;
      if (d != 0.0)
        for (int64_t i = 0; i < n; ++i) r[i] = r[i] + xj[i] * d;
      beta[j] = bn;
      if (fabs(d) > maxd) maxd = fabs(d);
    }
    ++sw;
  } while (!(maxd < delta) && sw < max_inner);
  *sweeps = sw;
  free(r);
  return maxd < delta ? ORACLE_OK : ORACLE_WARN_NOT_CONVERGED;
}

/*
 * Algorithm 2 first loop for the columns cols[0..ncols-1] of the standardized
 * n x p matrix Xs: column k is Algorithm 1 with response x_k and predictors X_{-k}.
 * B is p x ncols column-major (column c holds beta_{-cols[c]}, with B[cols[c], c] = 0).
 * margin (nullable) is p x ncols.  Columns are independent; OpenMP over columns does not
 * change any column's arithmetic.
 */
int oracle_spmesl_columns(const double* Xs, int64_t n, int64_t p, const int64_t* cols,
                          int64_t ncols, double lambda0, double delta, int32_t max_outer,
                          int32_t max_inner, double sigma_floor, int32_t nthreads, double* B,
                          double* sigma, int32_t* outer, int32_t* sweeps, uint8_t* converged,
                          double* margin) {
  int rc = check_args(n, p, lambda0, delta, max_outer, max_inner);
  if (rc) return rc;
  for (int64_t c = 0; c < ncols; ++c)
    if (cols[c] < 0 || cols[c] >= p) return ORACLE_ERR_ARG;
  int any_bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : any_bad)
#endif
  for (int64_t c = 0; c < ncols; ++c) {
    int64_t k = cols[c];
    int32_t fl = 0;
    int e = scaled_lasso_core(Xs, n, p, COL(Xs, k, n), k, lambda0, delta, max_outer, max_inner,
                              sigma_floor, B + (size_t)c * (size_t)p, &sigma[c], &outer[c],
                              &sweeps[c], &fl, NULL, margin ? margin + (size_t)c * (size_t)p : NULL,
                              NULL);
    if (e) any_bad = 1;
    converged[c] = (uint8_t)((fl & 1) && !(fl & 2));
  }
  (void)nthreads;
  return any_bad ? ORACLE_ERR_OOM : ORACLE_OK;
}

/*
 * Algorithm 2 lines P:698-708: omega_kk = sigma_k^-2, omega_jk = -beta_jk * omega_kk,
 * then Proposition 1: omega^o_jk = omega^C_jk / (s_j s_k) when s != NULL.
 */
int oracle_assemble(const double* B, const double* sigma, const double* s, int64_t p,
                    double* Theta1) {
  for (int64_t k = 0; k < p; ++k) {
    double wkk = 1.0 / (sigma[k] * sigma[k]);
    for (int64_t j = 0; j < p; ++j) {
      double w = (j == k) ? wkk : -B[j + k * p] * wkk;
      if (s) w = w / (s[j] * s[k]);
      Theta1[j + k * p] = w;
    }
  }
  return ORACLE_OK;
}

/* Algorithm 2 lines P:709-719 (Eq. symm): keep the smaller-magnitude entry;
 * tie -> the (j,k), j<k entry wins (the "else" branch, reading g7). In place. */
int oracle_symmetrize(double* T, int64_t p) {
  for (int64_t j = 0; j + 1 < p; ++j)
    for (int64_t k = j + 1; k < p; ++k) {
      double wjk = T[j + k * p], wkj = T[k + j * p];
      if (fabs(wjk) > fabs(wkj)) T[j + k * p] = wkj;
      else T[k + j * p] = wjk;
    }
  return ORACLE_OK;
}

/*
 * The whole Algorithm 2 pipeline on raw X (n x p col-major):
 * standardize (if standardize != 0) -> p column scaled lassos -> assemble (+Prop. 1 rescale)
 * -> symmetrize.  Outputs Theta (p x p), sigma_out[p] (original scale when standardized,
 * sigma_k^o = s_k sigma_k^C), outer[p], sweeps[p], converged[p]; optional B (p x p),
 * Theta1 (p x p, before symmetrization), margin (p x p).
 * Returns ORACLE_OK, ORACLE_WARN_NOT_CONVERGED or a negative error; *bad_col on column errors.
 */
int oracle_spmesl_fit(const double* X, int64_t n, int64_t p, double lambda0, double delta,
                      int32_t max_outer, int32_t max_inner, double sigma_floor, int32_t standardize,
                      int32_t nthreads, double* Theta, double* sigma_out, int32_t* outer,
                      int32_t* sweeps, uint8_t* converged, double* B_out, double* Theta1_out,
                      double* margin, int64_t* bad_col) {
  int rc = check_args(n, p, lambda0, delta, max_outer, max_inner);
  if (rc) return rc;
  if (n < 2 || p < 2) return ORACLE_ERR_ARG;
  size_t np = (size_t)n * (size_t)p, pp = (size_t)p * (size_t)p;
  double* Xs = (double*)malloc(sizeof(double) * np);
  double* mu = (double*)malloc(sizeof(double) * (size_t)p);
  double* s = (double*)malloc(sizeof(double) * (size_t)p);
  double* B = B_out ? B_out : (double*)malloc(sizeof(double) * pp);
  int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  if (!Xs || !mu || !s || !B || !cols) { rc = ORACLE_ERR_OOM; goto done; }
  if (standardize) {
    rc = oracle_standardize(X, n, p, Xs, mu, s, bad_col);
    if (rc) goto done;
  } else {
    for (size_t t = 0; t < np; ++t) {
      if (!isfinite(X[t])) { if (bad_col) *bad_col = (int64_t)(t / (size_t)n); rc = ORACLE_ERR_NONFINITE; goto done; }
      Xs[t] = X[t];
    }
  }
  for (int64_t k = 0; k < p; ++k) cols[k] = k;
  rc = oracle_spmesl_columns(Xs, n, p, cols, p, lambda0, delta, max_outer, max_inner, sigma_floor,
                             nthreads, B, sigma_out, outer, sweeps, converged, margin);
  if (rc) goto done;
  oracle_assemble(B, sigma_out, standardize ? s : NULL, p, Theta);
  if (Theta1_out) memcpy(Theta1_out, Theta, sizeof(double) * pp);
  oracle_symmetrize(Theta, p);
  if (standardize)
    for (int64_t k = 0; k < p; ++k) sigma_out[k] = s[k] * sigma_out[k];
  rc = ORACLE_OK;
  for (int64_t k = 0; k < p; ++k)
    if (!converged[k]) rc = ORACLE_WARN_NOT_CONVERGED;
done:
  free(Xs); free(mu); free(s); free(cols);
  if (!B_out) free(B);
  return rc;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/*
 * Algorithm 3, the paper-literal joint ("PCD") mode, for the columns cols[0..m-1] of
 * the standardized Xs (reading g8: the compaction keeps I_l <- I_j; g9: the residual update uses
 * x_j).  Outer loop r: lambda_c = sigma_c lambda0; E = x_{I} - X B (fresh);
 * inner repeat: for j = 1..p: for every active column c: a = x_j^T e_c / n + b_jc,
 * a_cc <- 0, b_jc <- Soft(a), e_c += x_j (b_old - b_new); until
 * max_{active c, j} |db_jc| < delta (the joint criterion) or max_inner sweeps; then
 * sigma_c = ||e_c||/sqrt(n) from a fresh residual, F_c = |dsigma_c| >= delta
 * and the active set keeps the columns with F_c = 1 in order.  Stops when no column
 * is active or after max_outer outer iterations.  Outputs as oracle_spmesl_columns.
 */
int oracle_joint_columns(const double* Xs, int64_t n, int64_t p, const int64_t* cols, int64_t m,
                         double lambda0, double delta, int32_t max_outer, int32_t max_inner,
                         double sigma_floor, double* B, double* sigma, int32_t* outer,
                         int32_t* sweeps, uint8_t* converged) {
  int rc = check_args(n, p, lambda0, delta, max_outer, max_inner);
  if (rc) return rc;
  for (int64_t c = 0; c < m; ++c)
    if (cols[c] < 0 || cols[c] >= p) return ORACLE_ERR_ARG;
  double* E = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(m > 0 ? m : 1));
  double* lam = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  int64_t* I = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));   /* active set */
  uint8_t* capped = (uint8_t*)calloc((size_t)(m > 0 ? 2 * m : 1), 1);
  if (!E || !lam || !I || !capped) { free(E); free(lam); free(I); free(capped); return ORACLE_ERR_OOM; }
  for (int64_t c = 0; c < m; ++c) {                 /* Require line P:941-943 */
    for (int64_t j = 0; j < p; ++j) B[j + c * p] = 0.0;
    sigma[c] = 1.0;
    outer[c] = 0;
    sweeps[c] = 0;
    converged[c] = 0;
    I[c] = c;
  }
  int64_t nc = m;
  for (int32_t r = 0; nc > 0 && r < max_outer; ++r) {
    for (int64_t a = 0; a < nc; ++a) lam[a] = sigma[I[a]] * lambda0;
#pragma omp parallel for schedule(dynamic)
    for (int64_t a = 0; a < nc; ++a) {
      const int64_t c = I[a], k = cols[c];
      double* e = E + a * n;
      for (int64_t i = 0; i < n; ++i) e[i] = Xs[i + k * n];
      for (int64_t j = 0; j < p; ++j) {
        const double b = B[j + c * p];
        if (j == k || b == 0.0) continue;
        for (int64_t i = 0; i < n; ++i) e[i] = e[i] - Xs[i + j * n] * b;
      }
    }
    int32_t inner = 0;
    double maxd;
    do {
      maxd = 0.0;
      for (int64_t j = 0; j < p; ++j) {
        const double* xj = Xs + j * n;
        /* the active columns are independent: threads split them, each column's arithmetic
           is unchanged */
#pragma omp parallel for reduction(max : maxd) schedule(static) if (nc >= 64)
        for (int64_t a = 0; a < nc; ++a) {
          const int64_t c = I[a], k = cols[c];
          if (j == k) continue;                                                   /* a_jj <- 0 */
          double* e = E + a * n;
          double dot = 0.0;
          for (int64_t i = 0; i < n; ++i) dot = dot + xj[i] * e[i];
          const double av = dot / (double)n + B[j + c * p];
          const double bn = oracle_soft_threshold(av, lam[a]);
          const double d = B[j + c * p] - bn;
          if (d != 0.0)
            for (int64_t i = 0; i < n; ++i) e[i] = e[i] + xj[i] * d;
          B[j + c * p] = bn;
          if (fabs(d) > maxd) maxd = fabs(d);
        }
      }
      for (int64_t a = 0; a < nc; ++a) sweeps[I[a]] += 1;
      ++inner;
    } while (!(maxd < delta) && inner < max_inner);
    if (!(maxd < delta))
      for (int64_t a = 0; a < nc; ++a) capped[I[a]] = 1;
    uint8_t* F = capped + m;  /* scratch F_c flags */
#pragma omp parallel for schedule(dynamic)
    for (int64_t a = 0; a < nc; ++a) {
      const int64_t c = I[a], k = cols[c];
      double* e = E + a * n;                         /* fresh residual (reading g4) */
      for (int64_t i = 0; i < n; ++i) e[i] = Xs[i + k * n];
      for (int64_t j = 0; j < p; ++j) {
        const double b = B[j + c * p];
        if (j == k || b == 0.0) continue;
        for (int64_t i = 0; i < n; ++i) e[i] = e[i] - Xs[i + j * n] * b;
      }
      double ss = 0.0;
      for (int64_t i = 0; i < n; ++i) ss = ss + e[i] * e[i];
      double sn = sqrt(ss) / sqrt((double)n);
      if (sn < sigma_floor) sn = sigma_floor;
      F[a] = (uint8_t)!(fabs(sn - sigma[c]) < delta);                            /* F_c */
      sigma[c] = sn;
      outer[c] += 1;
    }
    int64_t l = 0;
    for (int64_t a = 0; a < nc; ++a) {
      if (F[a]) I[l++] = I[a];
      else converged[I[a]] = 1;
    }
    nc = l;
  }
  for (int64_t c = 0; c < m; ++c)
    if (capped[c]) converged[c] = 0;
  free(E); free(lam); free(I); free(capped);
  return ORACLE_OK;
}

/* Algorithm 3 end to end (standardize, joint CD, assemble + rescale, symmetrize). */
int oracle_spmesl_fit_joint(const double* X, int64_t n, int64_t p, double lambda0, double delta,
                            int32_t max_outer, int32_t max_inner, double sigma_floor,
                            int32_t standardize, double* Theta, double* sigma_out, int32_t* outer,
                            int32_t* sweeps, uint8_t* converged, double* B_out, int64_t* bad_col) {
  int rc = check_args(n, p, lambda0, delta, max_outer, max_inner);
  if (rc) return rc;
  if (n < 2 || p < 2) return ORACLE_ERR_ARG;
  size_t np = (size_t)n * (size_t)p, pp = (size_t)p * (size_t)p;
  double* Xs = (double*)malloc(sizeof(double) * np);
  double* mu = (double*)malloc(sizeof(double) * (size_t)p);
  double* s = (double*)malloc(sizeof(double) * (size_t)p);
  double* B = B_out ? B_out : (double*)malloc(sizeof(double) * pp);
  int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  if (!Xs || !mu || !s || !B || !cols) { rc = ORACLE_ERR_OOM; goto done; }
  if (standardize) {
    rc = oracle_standardize(X, n, p, Xs, mu, s, bad_col);
    if (rc) goto done;
  } else {
    for (size_t t = 0; t < np; ++t) Xs[t] = X[t];
  }
  for (int64_t k = 0; k < p; ++k) cols[k] = k;
  rc = oracle_joint_columns(Xs, n, p, cols, p, lambda0, delta, max_outer, max_inner, sigma_floor,
                            B, sigma_out, outer, sweeps, converged);
  if (rc) goto done;
  oracle_assemble(B, sigma_out, standardize ? s : NULL, p, Theta);
  oracle_symmetrize(Theta, p);
  if (standardize)
    for (int64_t k = 0; k < p; ++k) sigma_out[k] = s[k] * sigma_out[k];
  rc = ORACLE_OK;
  for (int64_t k = 0; k < p; ++k)
    if (!converged[k]) rc = ORACLE_WARN_NOT_CONVERGED;
done:
  free(Xs); free(mu); free(s); free(cols);
  if (!B_out) free(B);
  return rc;
}

/*
 * cqk_oracle.c -- TEST INFRASTRUCTURE ONLY (see cqk_oracle.h).
 *
 * A plain-C restatement of the reference `cqksolve` hot path, written from
 * the reference's documented behaviour (file:line cited per function).  It is
 * the checker for the CUDA product and the CPU baseline timed by bench.py.
 * Build: oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off: every product
 * and sum is rounded separately, exactly like numpy's element-wise ufuncs).
 */
#include "cqk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ sums */

/* numpy's pairwise summation of a contiguous double array: blocks of <= 128
 * summed with 8 interleaved accumulators, larger ranges split at a multiple
 * of 8 near the middle.  This is what `ndarray.sum()` does in the reference
 * (e.g. core.py:198-211), so reproducing it makes the oracle bit-faithful. */
double orc_pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i];
    return s;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) s += a[i];
    return s;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return orc_pairwise_sum(a, n2) + orc_pairwise_sum(a + n2, n - n2);
}

/* parallel.py:62-72 _tree_sum: adjacent pairs, odd tail carried. */
static double tree_sum(double *v, int64_t k) {
  if (k == 0) return 0.0;
  while (k > 1) {
    int64_t j = 0;
    for (int64_t i = 0; i + 1 < k; i += 2) v[j++] = v[i] + v[i + 1];
    if (k % 2) v[j++] = v[k - 1];
    k = j;
  }
  return v[0];
}

static void *xmalloc(size_t bytes) { return malloc(bytes ? bytes : 1); }

/* ------------------------------------------------------------- validate */

static int domain(orc_result *res, int field, int64_t index) {
  if (res) {
    res->status = ORC_E_DOMAIN;
    res->domain_field = field;
    res->domain_index = index;
  }
  return ORC_E_DOMAIN;
}

/* core.py:126-165: checks in the reference's order, first offending index. */
int orc_validate(const double *d, const double *a, const double *b,
                 const double *l, const double *u, int64_t n, double r,
                 orc_result *res) {
  if (n < 1) return domain(res, 0, -1);
  const double *fin[3] = {d, a, b};
  for (int f = 0; f < 3; ++f)
    for (int64_t i = 0; i < n; ++i)
      if (!isfinite(fin[f][i])) return domain(res, f, i);
  for (int64_t i = 0; i < n; ++i)
    if (isnan(l[i])) return domain(res, 3, i);
  for (int64_t i = 0; i < n; ++i)
    if (isnan(u[i])) return domain(res, 4, i);
  if (!isfinite(r)) return domain(res, 5, -1);
  for (int64_t i = 0; i < n; ++i)
    if (!(d[i] > 0)) return domain(res, 0, i);
  for (int64_t i = 0; i < n; ++i)
    if (!(b[i] > 0)) return domain(res, 2, i);
  for (int64_t i = 0; i < n; ++i)
    if (!(l[i] <= u[i])) return domain(res, 6, i);
  for (int64_t i = 0; i < n; ++i)
    if (l[i] == INFINITY) return domain(res, 3, i);
  for (int64_t i = 0; i < n; ++i)
    if (u[i] == -INFINITY) return domain(res, 4, i);
  return ORC_SOLVED;
}

/* ------------------------------------------------------ initial lambda */

/* s = sum b*(a/d), q = sum b*(b/d) over an index subset, pairwise ordered */
static void sq_sums(const double *d, const double *a, const double *b,
                    const int64_t *sel, int64_t m, double *s, double *q) {
  double *ts = xmalloc(sizeof(double) * m), *tq = xmalloc(sizeof(double) * m);
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = sel ? sel[k] : k;
    ts[k] = b[i] * (a[i] / d[i]);
    tq[k] = b[i] * (b[i] / d[i]);
  }
  *s = orc_pairwise_sum(ts, m);
  *q = orc_pairwise_sum(tq, m);
  free(ts);
  free(tq);
}

/* core.py:237-257: lambda0 = (r - s)/q over all indices, or over the strictly
 * interior components of xbar when there are any. */
double orc_initial_multiplier(const double *d, const double *a, const double *b,
                              const double *l, const double *u, int64_t n,
                              double r, const double *xbar) {
  double s, q;
  if (xbar) {
    int64_t *sel = xmalloc(sizeof(int64_t) * n), m = 0;
    for (int64_t i = 0; i < n; ++i)
      if (l[i] < xbar[i] && xbar[i] < u[i]) sel[m++] = i;
    if (m > 0) {
      sq_sums(d, a, b, sel, m, &s, &q);
      free(sel);
      return (r - s) / q;
    }
    free(sel);
  }
  sq_sums(d, a, b, NULL, n, &s, &q);
  return (r - s) / q;
}

/* ----------------------------------------------------------- phi scan */

typedef struct {
  double value, dminus, dplus, abs_bx;
} scan4;

/* core.py:182-212 _phi_scan: one pass over idx[0..m) (NULL = identity).
 * Temporaries mirror the numpy expression graph; masked sums sum the
 * compacted subsequence, as `w[mask].sum()` does. */
static scan4 phi_scan(const double *d, const double *a, const double *b,
                      const double *l, const double *u, const int64_t *idx,
                      int64_t m, double lam, uint8_t *at_lo, uint8_t *at_hi) {
  double *bx = xmalloc(sizeof(double) * m), *ab = xmalloc(sizeof(double) * m);
  double *wi = xmalloc(sizeof(double) * m), *wl = xmalloc(sizeof(double) * m);
  double *wh = xmalloc(sizeof(double) * m);
  int64_t ni = 0, nl = 0, nh = 0;
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = idx ? idx[k] : k;
    double t = (b[i] * lam + a[i]) / d[i];
    double x = t < l[i] ? l[i] : t; /* np.clip: min(max(t, l), u) */
    x = x > u[i] ? u[i] : x;
    bx[k] = b[i] * x;
    ab[k] = fabs(bx[k]);
    int lo = t <= l[i], hi = t >= u[i];
    if (at_lo) at_lo[k] = (uint8_t)lo;
    if (at_hi) at_hi[k] = (uint8_t)hi;
    double w = b[i] * b[i] / d[i];
    if (!(lo | hi)) wi[ni++] = w;
    if (lo && t == l[i] && l[i] < u[i]) wl[nl++] = w;
    if (hi && t == u[i] && l[i] < u[i]) wh[nh++] = w;
  }
  scan4 s;
  s.value = orc_pairwise_sum(bx, m);
  s.abs_bx = orc_pairwise_sum(ab, m);
  double core = orc_pairwise_sum(wi, ni);
  s.dplus = core + orc_pairwise_sum(wl, nl);
  s.dminus = core + orc_pairwise_sum(wh, nh);
  free(bx); free(ab); free(wi); free(wl); free(wh);
  return s;
}

int orc_phi_scan(const double *d, const double *a, const double *b,
                 const double *l, const double *u, const int64_t *idx,
                 int64_t m, double lam, double *out, uint8_t *at_lower,
                 uint8_t *at_upper) {
  scan4 s = phi_scan(d, a, b, l, u, idx, m, lam, at_lower, at_upper);
  out[0] = s.value;
  out[1] = s.dminus;
  out[2] = s.dplus;
  out[3] = s.abs_bx;
  return 0;
}

/* core.py:168-179 eval_x */
void orc_eval_x(const double *d, const double *a, const double *b,
                const double *l, const double *u, const int64_t *idx,
                int64_t m, double lam, double *x) {
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = idx ? idx[k] : k;
    double t = (b[i] * lam + a[i]) / d[i];
    double v = t < l[i] ? l[i] : t;
    x[k] = v > u[i] ? u[i] : v;
  }
}

/* ------------------------------------------------ scalar Newton helpers */

/* newton.py:106-121 */
int orc_secant_step(double lo, double phi_lo, double hi, double phi_hi,
                    double r, double *out) {
  if (!(lo < hi) || !(phi_lo < r && r < phi_hi)) return ORC_E_CONTRACT;
  double lam = lo + (r - phi_lo) * (hi - lo) / (phi_hi - phi_lo);
  if (!(lo < lam && lam < hi)) lam = lo + 0.5 * (hi - lo);
  *out = lam;
  return 0;
}

/* newton.py:129-162 (and parallel.py:130-145 per chunk): dir 0 = RIGHT
 * (min bp > edge), 1 = LEFT (max bp < edge); lower bounds, then upper. */
int orc_nearest_breakpoint(const double *d, const double *a, const double *b,
                           const double *l, const double *u, const int64_t *idx,
                           int64_t m, double edge, int dir, double *out) {
  int found = 0;
  double best = 0.0;
  const double *bounds[2] = {l, u};
  for (int s = 0; s < 2; ++s) {
    const double *bd = bounds[s];
    for (int64_t k = 0; k < m; ++k) {
      int64_t i = idx ? idx[k] : k;
      if (!isfinite(bd[i])) continue;
      double bp = (d[i] * bd[i] - a[i]) / b[i];
      if (dir == 0 ? bp > edge : bp < edge) {
        if (!found || (dir == 0 ? bp < best : bp > best)) best = bp;
        found = 1;
      }
    }
  }
  if (found) *out = best;
  return found;
}

/* ------------------------------------------------------------ solve_cqk */

typedef struct {
  double lo, hi, phi_lo, phi_hi;
  int has_plo, has_phi;
} bracket;

/* The branch body shared by every CQK driver (newton.py:266-333,
 * parallel.py:252-310, parallel.py:443-493).  `bp_fn` evaluates the nearest
 * breakpoint for the driver's active set.  Returns: 0 continue with *next,
 * 1 finish at *next, 2 infeasible, <0 error. */
typedef int (*bp_fn_t)(void *ctx, double edge, int dir, double *out);

static int newton_branch(double lam, double diff, double dminus, double dplus,
                         double tau, double r_res, const bracket *br,
                         bp_fn_t bp_fn, void *ctx, double *next) {
  double next_lam;
  if (diff < 0) {
    if (dplus > 0) {
      double step = -diff / dplus;
      if (step < tau) { *next = lam + step; return 1; }
      double tilde = lam + step;
      if (tilde < br->hi) next_lam = tilde;
      else if (orc_secant_step(br->lo, br->phi_lo, br->hi, br->phi_hi, r_res, &next_lam))
        return ORC_E_CONTRACT;
    } else {
      double bp;
      int found = bp_fn(ctx, br->lo, 0, &bp);
      if (found && bp < br->hi) next_lam = bp;
      else if (br->has_phi) {
        if (orc_secant_step(br->lo, br->phi_lo, br->hi, br->phi_hi, r_res, &next_lam))
          return ORC_E_CONTRACT;
      } else return 2;
    }
  } else {
    if (dminus > 0) {
      double step = -diff / dminus;
      if (-step < tau) { *next = lam + step; return 1; }
      double tilde = lam + step;
      if (tilde > br->lo) next_lam = tilde;
      else if (orc_secant_step(br->lo, br->phi_lo, br->hi, br->phi_hi, r_res, &next_lam))
        return ORC_E_CONTRACT;
    } else {
      double bp;
      int found = bp_fn(ctx, br->hi, 1, &bp);
      if (found && bp > br->lo) next_lam = bp;
      else if (br->has_plo) {
        if (orc_secant_step(br->lo, br->phi_lo, br->hi, br->phi_hi, r_res, &next_lam))
          return ORC_E_CONTRACT;
      } else return 2;
    }
  }
  if (next_lam == lam) { *next = lam; return 1; }
  if (isfinite(br->lo) && isfinite(br->hi)) {
    double w = br->hi - br->lo;
    double m = fabs(br->hi) > fabs(br->lo) ? fabs(br->hi) : fabs(br->lo);
    if (w < tau * m) { *next = next_lam; return 1; }
  }
  *next = next_lam;
  return 0;
}

typedef struct {
  const double *d, *a, *b, *l, *u;
  const int64_t *idx;
  int64_t m;
} seq_ctx;

static int seq_bp(void *c, double edge, int dir, double *out) {
  seq_ctx *s = (seq_ctx *)c;
  return orc_nearest_breakpoint(s->d, s->a, s->b, s->l, s->u, s->idx, s->m,
                                edge, dir, out);
}

static void fill_result(orc_result *res, int status, double lam, double lam0,
                        int64_t it, int64_t ev, int64_t fc, const bracket *br) {
  if (!res) return;
  res->status = status;
  res->lam = lam;
  res->lam0 = lam0;
  res->iterations = it;
  res->phi_evals = ev;
  res->fixed_count = fc;
  res->bracket_lo = br ? br->lo : -INFINITY;
  res->bracket_hi = br ? br->hi : INFINITY;
}

/* newton.py:209-342 */
int orc_solve_cqk(const double *d, const double *a, const double *b,
                  const double *l, const double *u, int64_t n, double r,
                  int fixing, int64_t max_iter, double tau, const double *xbar,
                  double lam0, int check, double *x, orc_result *res) {
  if (check) {
    int st = orc_validate(d, a, b, l, u, n, r, res);
    if (st) return st;
  }
  double lam = isnan(lam0) ? orc_initial_multiplier(d, a, b, l, u, n, r, xbar) : lam0;
  double lam_init = lam;
  int64_t *idx = xmalloc(sizeof(int64_t) * n), m = n;
  uint8_t *alo = xmalloc(n), *ahi = xmalloc(n);
  double *tmp = xmalloc(sizeof(double) * n), *tabs = xmalloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  double r_res = r, fixed_abs = 0.0;
  int64_t fixed_count = 0, iterations = 0, phi_evals = 0;
  bracket br = {-INFINITY, INFINITY, 0.0, 0.0, 0, 0};
  int status = ORC_E_MAXITER;
  double out_lam = lam;

  while (iterations <= max_iter) {
    scan4 s = phi_scan(d, a, b, l, u, idx, m, lam, alo, ahi);
    phi_evals++;
    double diff = s.value - r_res;
    double scale = s.abs_bx + fixed_abs + fabs(r);
    if (fabs(diff) < tau * scale) { status = ORC_SOLVED; out_lam = lam; break; }
    if (diff < 0) { br.lo = lam; br.phi_lo = s.value; br.has_plo = 1; }
    else { br.hi = lam; br.phi_hi = s.value; br.has_phi = 1; }
    if (fixing) { /* newton.py:165-206 fix_variables */
      double rr = s.value - diff;
      const uint8_t *mask = NULL;
      const double *bound = NULL;
      if (s.value > rr) { mask = alo; bound = l; }
      else if (s.value < rr) { mask = ahi; bound = u; }
      if (mask) {
        int64_t k = 0, keep = 0;
        for (int64_t j = 0; j < m; ++j) {
          int64_t i = idx[j];
          if (mask[j] && isfinite(bound[i])) {
            tmp[k] = b[i] * bound[i];
            tabs[k] = fabs(tmp[k]);
            ++k;
            if (x) x[i] = bound[i];
          } else {
            idx[keep++] = i;
          }
        }
        if (k > 0) {
          double total = orc_pairwise_sum(tmp, k);
          r_res -= total;
          fixed_abs += orc_pairwise_sum(tabs, k);
          fixed_count += k;
          if (br.has_plo) br.phi_lo -= total;
          if (br.has_phi) br.phi_hi -= total;
          m = keep;
        }
      }
    }
    seq_ctx ctx = {d, a, b, l, u, idx, m};
    double next;
    int rc = newton_branch(lam, diff, s.dminus, s.dplus, tau, r_res, &br, seq_bp, &ctx, &next);
    if (rc == 1) { status = ORC_SOLVED; out_lam = next; break; }
    if (rc == 2) { status = ORC_INFEASIBLE; break; }
    if (rc < 0) { status = rc; out_lam = lam; break; }
    lam = next;
    iterations++;
    out_lam = lam;
  }
  if (status == ORC_SOLVED && x) {
    double *xa = tmp; /* reuse: m <= n */
    orc_eval_x(d, a, b, l, u, idx, m, out_lam, xa);
    for (int64_t j = 0; j < m; ++j) x[idx[j]] = xa[j];
  }
  fill_result(res, status, out_lam, lam_init, iterations, phi_evals, fixed_count, &br);
  free(idx); free(alo); free(ahi); free(tmp); free(tabs);
  return status;
}

/* ------------------------------------------------------- chunked drivers */

/* parallel.py:82-85: np.linspace(0, n, w + 1).astype(int64), empty dropped */
static int chunk_ranges(int64_t n, int workers, int64_t *lo, int64_t *hi) {
  double step = (double)n / (double)workers;
  int k = 0;
  for (int c = 0; c < workers; ++c) {
    int64_t e0 = (int64_t)((double)c * step);
    int64_t e1 = c + 1 == workers ? n : (int64_t)((double)(c + 1) * step);
    if (e1 > e0) { lo[k] = e0; hi[k] = e1; ++k; }
  }
  return k;
}

typedef struct {
  const double *d, *a, *b, *l, *u;
  int64_t *lo, *hi;
  int nch;
} jac_ctx;

static int jac_bp(void *c, double edge, int dir, double *out) {
  jac_ctx *j = (jac_ctx *)c;
  int found = 0;
  double best = 0;
  for (int k = 0; k < j->nch; ++k) {
    double v;
    if (orc_nearest_breakpoint(j->d + j->lo[k], j->a + j->lo[k], j->b + j->lo[k],
                               j->l + j->lo[k], j->u + j->lo[k], NULL,
                               j->hi[k] - j->lo[k], edge, dir, &v)) {
      if (!found || (dir == 0 ? v < best : v > best)) best = v;
      found = 1;
    }
  }
  if (found) *out = best;
  return found;
}

/* parallel.py:371-500 */
int orc_jacobi_solve(const double *d, const double *a, const double *b,
                     const double *l, const double *u, int64_t n, double r,
                     int64_t max_iter, double tau, int workers, double lam0,
                     int check, double *x, orc_result *res) {
  if (check) {
    int st = orc_validate(d, a, b, l, u, n, r, res);
    if (st) return st;
  }
  if (workers < 1) workers = 1;
  int64_t *clo = xmalloc(sizeof(int64_t) * workers), *chi = xmalloc(sizeof(int64_t) * workers);
  int nch = chunk_ranges(n, workers, clo, chi);
  double *parts = xmalloc(sizeof(double) * 4 * nch), *col = xmalloc(sizeof(double) * nch);
  double lam = isnan(lam0) ? orc_initial_multiplier(d, a, b, l, u, n, r, NULL) : lam0;
  double lam_init = lam, out_lam = lam;
  bracket br = {-INFINITY, INFINITY, 0.0, 0.0, 0, 0};
  int64_t iterations = 0, phi_evals = 0;
  int status = ORC_E_MAXITER;
  jac_ctx ctx = {d, a, b, l, u, clo, chi, nch};
  while (iterations <= max_iter) {
#pragma omp parallel for schedule(static, 1) num_threads(workers)
    for (int k = 0; k < nch; ++k) {
      int64_t o = clo[k];
      scan4 s = phi_scan(d + o, a + o, b + o, l + o, u + o, NULL, chi[k] - o, lam, NULL, NULL);
      parts[4 * k + 0] = s.value;
      parts[4 * k + 1] = s.dminus;
      parts[4 * k + 2] = s.dplus;
      parts[4 * k + 3] = s.abs_bx;
    }
    phi_evals++;
    double tot[4];
    for (int c = 0; c < 4; ++c) {
      for (int k = 0; k < nch; ++k) col[k] = parts[4 * k + c];
      tot[c] = tree_sum(col, nch);
    }
    double diff = tot[0] - r;
    if (fabs(diff) < tau * (tot[3] + fabs(r))) { status = ORC_SOLVED; out_lam = lam; break; }
    if (diff < 0) { br.lo = lam; br.phi_lo = tot[0]; br.has_plo = 1; }
    else { br.hi = lam; br.phi_hi = tot[0]; br.has_phi = 1; }
    double next;
    int rc = newton_branch(lam, diff, tot[1], tot[2], tau, r, &br, jac_bp, &ctx, &next);
    if (rc == 1) { status = ORC_SOLVED; out_lam = next; break; }
    if (rc == 2) { status = ORC_INFEASIBLE; break; }
    if (rc < 0) { status = rc; out_lam = lam; break; }
    lam = next;
    iterations++;
    out_lam = lam;
  }
  if (status == ORC_SOLVED && x) {
#pragma omp parallel for schedule(static, 1) num_threads(workers)
    for (int k = 0; k < nch; ++k) {
      int64_t o = clo[k];
      orc_eval_x(d + o, a + o, b + o, l + o, u + o, NULL, chi[k] - o, out_lam, x + o);
    }
  }
  fill_result(res, status, out_lam, lam_init, iterations, phi_evals, 0, &br);
  free(clo); free(chi); free(parts); free(col);
  return status;
}

/* parallel.py:174-327 par_solve_cqk: per-chunk active lists, per-chunk
 * fixing, fixed-order tree reduction, merging of depleted chunks. */
typedef struct {
  int64_t *idx;
  int64_t m;
} chunk_t;

typedef struct {
  const double *d, *a, *b, *l, *u;
  chunk_t *ch;
  int nch;
} par_ctx;

static int par_bp(void *c, double edge, int dir, double *out) {
  par_ctx *p = (par_ctx *)c;
  int found = 0;
  double best = 0;
  for (int k = 0; k < p->nch; ++k) {
    double v;
    if (orc_nearest_breakpoint(p->d, p->a, p->b, p->l, p->u, p->ch[k].idx,
                               p->ch[k].m, edge, dir, &v)) {
      if (!found || (dir == 0 ? v < best : v > best)) best = v;
      found = 1;
    }
  }
  if (found) *out = best;
  return found;
}

int orc_par_solve_cqk(const double *d, const double *a, const double *b,
                      const double *l, const double *u, int64_t n, double r,
                      int fixing, int64_t max_iter, double tau, int workers,
                      const double *xbar, int64_t merge_threshold, double lam0,
                      int check, double *x, orc_result *res) {
  if (check) {
    int st = orc_validate(d, a, b, l, u, n, r, res);
    if (st) return st;
  }
  if (workers < 1) workers = 1;
  int64_t *clo = xmalloc(sizeof(int64_t) * workers), *chi = xmalloc(sizeof(int64_t) * workers);
  int nch = chunk_ranges(n, workers, clo, chi);
  chunk_t *ch = xmalloc(sizeof(chunk_t) * nch);
  for (int k = 0; k < nch; ++k) {
    ch[k].m = chi[k] - clo[k];
    ch[k].idx = xmalloc(sizeof(int64_t) * ch[k].m);
    for (int64_t j = 0; j < ch[k].m; ++j) ch[k].idx[j] = clo[k] + j;
  }
  double *parts = xmalloc(sizeof(double) * 8 * nch), *col = xmalloc(sizeof(double) * nch);
  uint8_t **alo = xmalloc(sizeof(uint8_t *) * nch), **ahi = xmalloc(sizeof(uint8_t *) * nch);
  for (int k = 0; k < nch; ++k) { alo[k] = xmalloc(ch[k].m); ahi[k] = xmalloc(ch[k].m); }
  int64_t *fcnt = xmalloc(sizeof(int64_t) * nch);

  double lam;
  if (!isnan(lam0)) {
    lam = lam0;
  } else { /* parallel.py:148-171 _parallel_lambda0 */
    double *ps = xmalloc(sizeof(double) * 4 * nch);
    int64_t *pc = xmalloc(sizeof(int64_t) * nch);
#pragma omp parallel for schedule(static, 1) num_threads(workers)
    for (int k = 0; k < nch; ++k) {
      sq_sums(d, a, b, ch[k].idx, ch[k].m, &ps[4 * k], &ps[4 * k + 1]);
      ps[4 * k + 2] = ps[4 * k];
      ps[4 * k + 3] = ps[4 * k + 1];
      pc[k] = ch[k].m;
      if (xbar) {
        int64_t *sel = xmalloc(sizeof(int64_t) * ch[k].m), mm = 0;
        for (int64_t j = 0; j < ch[k].m; ++j) {
          int64_t i = ch[k].idx[j];
          if (l[i] < xbar[i] && xbar[i] < u[i]) sel[mm++] = i;
        }
        if (mm) sq_sums(d, a, b, sel, mm, &ps[4 * k + 2], &ps[4 * k + 3]);
        else ps[4 * k + 2] = ps[4 * k + 3] = 0.0;
        pc[k] = mm;
        free(sel);
      }
    }
    int64_t cj = 0;
    for (int k = 0; k < nch; ++k) cj += pc[k];
    int use = (xbar && cj > 0) ? 2 : 0;
    for (int k = 0; k < nch; ++k) col[k] = ps[4 * k + use];
    double s = tree_sum(col, nch);
    for (int k = 0; k < nch; ++k) col[k] = ps[4 * k + use + 1];
    double q = tree_sum(col, nch);
    lam = (r - s) / q;
    free(ps); free(pc);
  }
  double lam_init = lam, out_lam = lam, r_res = r, fixed_abs = 0.0;
  int64_t fixed_count = 0, iterations = 0, phi_evals = 0;
  bracket br = {-INFINITY, INFINITY, 0.0, 0.0, 0, 0};
  int status = ORC_E_MAXITER;

  while (iterations <= max_iter) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(workers)
    for (int k = 0; k < nch; ++k) {
      scan4 s = phi_scan(d, a, b, l, u, ch[k].idx, ch[k].m, lam, alo[k], ahi[k]);
      parts[8 * k + 0] = s.value;
      parts[8 * k + 1] = s.dminus;
      parts[8 * k + 2] = s.dplus;
      parts[8 * k + 3] = s.abs_bx;
    }
    phi_evals++;
    double tot[4];
    for (int c = 0; c < 4; ++c) {
      for (int k = 0; k < nch; ++k) col[k] = parts[8 * k + c];
      tot[c] = tree_sum(col, nch);
    }
    double diff = tot[0] - r_res;
    if (fabs(diff) < tau * (tot[3] + fixed_abs + fabs(r))) { status = ORC_SOLVED; out_lam = lam; break; }
    if (diff < 0) { br.lo = lam; br.phi_lo = tot[0]; br.has_plo = 1; }
    else { br.hi = lam; br.phi_hi = tot[0]; br.has_phi = 1; }
    if (fixing) { /* parallel.py:111-127 _fix_chunk, 234-250 */
      int lower = diff > 0;
      const double *bound = lower ? l : u;
#pragma omp parallel for schedule(dynamic, 1) num_threads(workers)
      for (int k = 0; k < nch; ++k) {
        uint8_t *mask = lower ? alo[k] : ahi[k];
        double *c = xmalloc(sizeof(double) * ch[k].m), *ca = xmalloc(sizeof(double) * ch[k].m);
        int64_t cnt = 0, keep = 0;
        for (int64_t j = 0; j < ch[k].m; ++j) {
          int64_t i = ch[k].idx[j];
          if (mask[j] && isfinite(bound[i])) {
            c[cnt] = b[i] * bound[i];
            ca[cnt] = fabs(c[cnt]);
            ++cnt;
            if (x) x[i] = bound[i];
          } else {
            ch[k].idx[keep++] = i;
          }
        }
        parts[8 * k + 4] = cnt ? orc_pairwise_sum(c, cnt) : 0.0;
        parts[8 * k + 5] = cnt ? orc_pairwise_sum(ca, cnt) : 0.0;
        fcnt[k] = cnt;
        if (cnt) ch[k].m = keep;
        free(c); free(ca);
      }
      for (int k = 0; k < nch; ++k) col[k] = parts[8 * k + 4];
      double total = tree_sum(col, nch);
      int64_t nfix = 0;
      for (int k = 0; k < nch; ++k) nfix += fcnt[k];
      if (total != 0.0 || nfix) {
        r_res -= total;
        for (int k = 0; k < nch; ++k) col[k] = parts[8 * k + 5];
        fixed_abs += tree_sum(col, nch);
        fixed_count += nfix;
        if (br.has_plo) br.phi_lo -= total;
        if (br.has_phi) br.phi_hi -= total;
      }
    }
    par_ctx ctx = {d, a, b, l, u, ch, nch};
    double next;
    int rc = newton_branch(lam, diff, tot[1], tot[2], tau, r_res, &br, par_bp, &ctx, &next);
    if (rc == 1) { status = ORC_SOLVED; out_lam = next; break; }
    if (rc == 2) { status = ORC_INFEASIBLE; break; }
    if (rc < 0) { status = rc; out_lam = lam; break; }
    lam = next;
    iterations++;
    out_lam = lam;
    if (nch > 1) { /* parallel.py:314-322 coalesce depleted chunks */
      int nsmall = 0;
      for (int k = 0; k < nch; ++k) nsmall += ch[k].m < merge_threshold;
      if (nsmall > 1) {
        int64_t tot_m = 0;
        for (int k = 0; k < nch; ++k) if (ch[k].m < merge_threshold) tot_m += ch[k].m;
        int64_t *mi = xmalloc(sizeof(int64_t) * tot_m), pos = 0;
        chunk_t *nc = xmalloc(sizeof(chunk_t) * nch);
        uint8_t **nlo = xmalloc(sizeof(uint8_t *) * nch), **nhi = xmalloc(sizeof(uint8_t *) * nch);
        int q = 0;
        for (int k = 0; k < nch; ++k) {
          if (ch[k].m >= merge_threshold) { nc[q] = ch[k]; nlo[q] = alo[k]; nhi[q] = ahi[k]; ++q; }
          else {
            memcpy(mi + pos, ch[k].idx, sizeof(int64_t) * ch[k].m);
            pos += ch[k].m;
            free(ch[k].idx); free(alo[k]); free(ahi[k]);
          }
        }
        nc[q].idx = mi; nc[q].m = tot_m; nlo[q] = xmalloc(tot_m); nhi[q] = xmalloc(tot_m); ++q;
        free(ch); free(alo); free(ahi);
        ch = nc; alo = nlo; ahi = nhi; nch = q;
      }
    }
  }
  if (status == ORC_SOLVED && x) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(workers)
    for (int k = 0; k < nch; ++k) {
      double *xa = xmalloc(sizeof(double) * ch[k].m);
      orc_eval_x(d, a, b, l, u, ch[k].idx, ch[k].m, out_lam, xa);
      for (int64_t j = 0; j < ch[k].m; ++j) x[ch[k].idx[j]] = xa[j];
      free(xa);
    }
  }
  fill_result(res, status, out_lam, lam_init, iterations, phi_evals, fixed_count, &br);
  for (int k = 0; k < nch; ++k) { free(ch[k].idx); free(alo[k]); free(ahi[k]); }
  free(ch); free(alo); free(ahi); free(clo); free(chi); free(parts); free(col); free(fcnt);
  return status;
}

/* ------------------------------------------------------------- simplex */

/* simplex.py:47-111 _init_lambda_kernel (Algorithm 2, Gauss-Seidel) */
static double init_kernel(const double *y, double r, const int64_t *idx,
                          int64_t p, const double *xbar, int sharpened,
                          int64_t *J, uint8_t *fixed, int64_t *Jt,
                          int64_t *nJ_out, double *sumJ_out, int64_t *jplus_out) {
  int64_t i1 = idx ? idx[0] : 0;
  int64_t nJ = 1, nJt = 0, jplus = 0;
  J[0] = i1;
  double sumJ = y[i1], lam = r - y[i1];
  if (!xbar || xbar[i1] > 0.0) jplus = 1;
  for (int64_t jj = 1; jj < p; ++jj) {
    int64_t i = idx ? idx[jj] : jj;
    if (xbar && xbar[i] <= 0.0) continue;
    double yi = y[i];
    int ok = yi + lam > 0.0;
    if (sharpened && yi <= 0.0) ok = 0;
    if (!ok) { fixed[i] = 1; continue; }
    double cand = (r - sumJ - yi) / (double)(nJ + 1);
    if (cand < r - yi) {
      J[nJ++] = i;
      sumJ += yi;
      lam = cand;
    } else {
      for (int64_t q = 0; q < nJ; ++q) Jt[nJt++] = J[q];
      J[0] = i;
      nJ = 1;
      sumJ = yi;
      lam = r - yi;
      jplus = 0;
    }
    if (!xbar || xbar[i] > 0.0) jplus++;
  }
  for (int64_t q = 0; q < nJt; ++q) {
    int64_t i = Jt[q];
    double yi = y[i];
    int ok = yi + lam > 0.0;
    if (sharpened && yi <= 0.0) ok = 0;
    if (!ok) { fixed[i] = 1; continue; }
    lam = (r - sumJ - yi) / (double)(nJ + 1);
    J[nJ++] = i;
    sumJ += yi;
    if (!xbar || xbar[i] > 0.0) jplus++;
  }
  *nJ_out = nJ;
  *sumJ_out = sumJ;
  *jplus_out = jplus;
  return lam;
}

/* simplex.py:114-154 */
int orc_simplex_init_lambda(const double *y, int64_t n, double r,
                            const int64_t *idx, int64_t p, const double *xbar,
                            int sharpened, double *lam, int64_t *free_out,
                            int64_t *nfree, uint8_t *fixed_mask, double *sumJ) {
  if (p < 1) return ORC_E_DOMAIN;
  int64_t *Jt = xmalloc(sizeof(int64_t) * p), jplus;
  memset(fixed_mask, 0, n);
  double lm = init_kernel(y, r, idx, p, xbar, sharpened, free_out, fixed_mask, Jt,
                          nfree, sumJ, &jplus);
  if (xbar && jplus == 0) {
    double c1 = r / (double)n, c2 = -y[0];
    lm = c1 >= c2 ? c1 : c2; /* Python max keeps the first on ties */
  }
  *lam = lm;
  free(Jt);
  return 0;
}

/* parallel.py:330-368 par_simplex_init: Algorithm 2 per contiguous chunk
 * (chunks as _chunk_ranges), merged with _tree_sum; free = concatenated J. */
int orc_par_simplex_init(const double *y, int64_t n, double r, int workers, double *lam,
                         int64_t *free_out, int64_t *nfree, uint8_t *fixed_mask, double *sumJ) {
  if (workers < 1) workers = 1;
  int64_t *clo = xmalloc(sizeof(int64_t) * workers), *chi = xmalloc(sizeof(int64_t) * workers);
  int nch = chunk_ranges(n, workers, clo, chi);
  double *sums = xmalloc(sizeof(double) * nch);
  int64_t *cnt = xmalloc(sizeof(int64_t) * nch);
  memset(fixed_mask, 0, n);
  int64_t *J = xmalloc(sizeof(int64_t) * n), *Jt = xmalloc(sizeof(int64_t) * n);
#pragma omp parallel for schedule(dynamic, 1)
  for (int k = 0; k < nch; ++k) {
    int64_t p = chi[k] - clo[k], *idx = xmalloc(sizeof(int64_t) * p), jp;
    for (int64_t j = 0; j < p; ++j) idx[j] = clo[k] + j;
    init_kernel(y, r, idx, p, NULL, 0, J + clo[k], fixed_mask, Jt + clo[k], &cnt[k], &sums[k], &jp);
    free(idx);
  }
  int64_t tot = 0;
  for (int k = 0; k < nch; ++k) {
    memmove(free_out + tot, J + clo[k], sizeof(int64_t) * cnt[k]);
    tot += cnt[k];
  }
  double s = tree_sum(sums, nch);
  *sumJ = s;
  *nfree = tot;
  *lam = (r - s) / (double)tot;
  free(clo); free(chi); free(sums); free(cnt); free(J); free(Jt);
  return 0;
}

static int newton_simplex_loop(const double *y, int64_t n, double r, int fixing,
                               int64_t max_iter, double tau, double lam, int64_t *free_,
                               int64_t m, double *x, double *trace, int64_t trace_cap,
                               orc_result *res);

/* Algorithm 4 from a given start and free set (the loop of simplex.py:252-308) */
int orc_newton_simplex_from(const double *y, int64_t n, double r, int fixing, int64_t max_iter,
                            double tau, double lam0, const int64_t *free_idx, int64_t m,
                            double *x, orc_result *res) {
  int64_t *f = xmalloc(sizeof(int64_t) * n);
  memcpy(f, free_idx, sizeof(int64_t) * m);
  return newton_simplex_loop(y, n, r, fixing, max_iter, tau, lam0, f, m, x, NULL, 0, res);
}

/* simplex.py:218-308, dense output. */
int orc_newton_project_simplex(const double *y, int64_t n, double r,
                               int fixing, int64_t max_iter, double tau,
                               const double *xbar, int sharpened, double lam0,
                               double *x, double *trace, int64_t trace_cap,
                               orc_result *res) {
  if (!(r > 0)) { domain(res, 5, -1); return ORC_E_DOMAIN; }
  int64_t *free_ = xmalloc(sizeof(int64_t) * n), m = 0;
  double lam;
  if (isnan(lam0)) {
    uint8_t *fixed = xmalloc(n);
    int64_t *J = xmalloc(sizeof(int64_t) * n), nJ;
    double sJ;
    orc_simplex_init_lambda(y, n, r, NULL, n, xbar, sharpened, &lam, J, &nJ, fixed, &sJ);
    for (int64_t i = 0; i < n; ++i) if (!fixed[i]) free_[m++] = i;
    free(fixed); free(J);
  } else {
    double mn = -y[0];
    for (int64_t i = 1; i < n; ++i) if (-y[i] < mn) mn = -y[i];
    lam = lam0 >= mn ? lam0 : mn;
    for (int64_t i = 0; i < n; ++i) free_[i] = i;
    m = n;
  }
  return newton_simplex_loop(y, n, r, fixing, max_iter, tau, lam, free_, m, x, trace, trace_cap,
                             res);
}

/* takes ownership of free_ */
static int newton_simplex_loop(const double *y, int64_t n, double r, int fixing,
                               int64_t max_iter, double tau, double lam, int64_t *free_,
                               int64_t m, double *x, double *trace, int64_t trace_cap,
                               orc_result *res) {
  double lam_init = lam;
  int64_t fixed_count = n - m, iterations = 0, phi_evals = 0;
  double lo = -INFINITY, hi = INFINITY;
  double *t = xmalloc(sizeof(double) * n), *pv = xmalloc(sizeof(double) * n);
  uint8_t *zero = xmalloc(n);
  for (;;) { /* simplex.py:207-215 _phi_free */
    int64_t np_ = 0, nz = 0;
    for (int64_t k = 0; k < m; ++k) {
      t[k] = y[free_[k]] + lam;
      int pos = t[k] > 0;
      zero[k] = !pos;
      if (pos) pv[np_++] = t[k];
      if (t[k] == 0) nz++;
    }
    double value = orc_pairwise_sum(pv, np_);
    double dminus = (double)np_, dplus = dminus + (double)nz;
    if (trace && phi_evals < trace_cap) {
      trace[4 * phi_evals + 0] = lam;
      trace[4 * phi_evals + 1] = value;
      trace[4 * phi_evals + 2] = dminus;
      trace[4 * phi_evals + 3] = dplus;
    }
    phi_evals++;
    double deriv;
    if (iterations == 0) {
      if (value == r) break;
      deriv = value < r ? dplus : dminus;
    } else {
      if (value <= r) break;
      deriv = dminus;
    }
    if (value < r) lo = lam;
    else {
      hi = lam;
      if (fixing && np_ < m) {
        int64_t keep = 0;
        for (int64_t k = 0; k < m; ++k) if (!zero[k]) free_[keep++] = free_[k];
        fixed_count += m - keep;
        m = keep;
      }
    }
    if (deriv <= 0) {
      double mx = -y[free_[0]];
      for (int64_t k = 1; k < m; ++k) if (-y[free_[k]] > mx) mx = -y[free_[k]];
      lam = mx;
      iterations++;
      continue;
    }
    double step = -(value - r) / deriv;
    double next = lam + step;
    if (fabs(step) < tau || next == lam) { lam = next; break; }
    if (isfinite(lo) && isfinite(hi)) {
      double mm = fabs(hi) > fabs(lo) ? fabs(hi) : fabs(lo);
      if (hi - lo < tau * mm) { lam = next; break; }
    }
    lam = next;
    iterations++;
    if (iterations > max_iter) break;
  }
  if (x)
    for (int64_t i = 0; i < n; ++i) {
      double v = y[i] + lam;
      x[i] = v > 0.0 ? v : 0.0;
    }
  bracket br = {lo, hi, 0, 0, 0, 0};
  fill_result(res, ORC_SOLVED, lam, lam_init, iterations, phi_evals, fixed_count, &br);
  free(free_); free(t); free(pv); free(zero);
  return ORC_SOLVED;
}

/* simplex.py:311-333 */
int orc_project_l1(const double *y, int64_t n, double r, int fixing,
                   int64_t max_iter, double tau, const double *xbar, double *x,
                   orc_result *res) {
  if (!(r > 0)) { domain(res, 5, -1); return ORC_E_DOMAIN; }
  double *ay = xmalloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) ay[i] = fabs(y[i]);
  if (orc_pairwise_sum(ay, n) <= r) {
    if (x) memcpy(x, y, sizeof(double) * n);
    fill_result(res, ORC_SOLVED, NAN, NAN, -1, 0, 0, NULL);
    free(ay);
    return ORC_SOLVED;
  }
  int st = orc_newton_project_simplex(ay, n, r, fixing, max_iter, tau, xbar, 1, NAN,
                                      NULL, NULL, 0, res);
  if (st == ORC_SOLVED && x) {
    double lam = res->lam;
    for (int64_t i = 0; i < n; ++i) {
      double v = ay[i] + lam;
      v = v > 0.0 ? v : 0.0;
      double sg = y[i] > 0 ? 1.0 : (y[i] < 0 ? -1.0 : 0.0);
      x[i] = sg * v;
    }
  }
  free(ay);
  return st;
}

/* oracle.py:88-97: sort descending, cumulative sums, largest feasible k */
static int cmp_desc(const void *p, const void *q) {
  double a = *(const double *)p, b = *(const double *)q;
  return (a < b) - (a > b);
}

double orc_exact_simplex_lambda(const double *y, int64_t n, double r) {
  double *ys = xmalloc(sizeof(double) * n);
  memcpy(ys, y, sizeof(double) * n);
  qsort(ys, n, sizeof(double), cmp_desc);
  double c = 0.0, lam = 0.0;
  int64_t kk = 0;
  double *cs = xmalloc(sizeof(double) * n);
  for (int64_t k = 0; k < n; ++k) {
    c += ys[k];
    cs[k] = c;
    if (ys[k] + (r - c) / (double)(k + 1) > 0) kk = k + 1;
  }
  lam = (r - cs[kk - 1]) / (double)kk;
  free(ys); free(cs);
  return lam;
}

/* Batched rows (C5; no reference function): newton_project_simplex(Y[i], r)
 * (simplex.py:218-308, default Algorithm-2 start) per row, rows spread over
 * `threads` OpenMP threads.  Returns the number of rows that did not solve. */
int64_t orc_project_simplex_rows(const double *Y, int64_t rows, int64_t cols, double r,
                                 int threads, double *X, double *lam, int64_t *iters) {
  int64_t bad = 0;
  const double tau = pow(2.220446049250313e-16, 0.75); /* newton.py:64-67 */
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads > 0 ? threads : 1) reduction(+ : bad)
  for (int64_t i = 0; i < rows; ++i) {
    orc_result res;
    const int st = orc_newton_project_simplex(Y + i * cols, cols, r, 1, 100, tau, NULL, 0, NAN,
                                              X ? X + i * cols : NULL, NULL, 0, &res);
    if (lam) lam[i] = res.lam;
    if (iters) iters[i] = res.iterations;
    bad += st != ORC_SOLVED;
  }
  return bad;
}

/*
 * cqk_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, fp64) of the reference package `cqksolve`
 * (/root/reference/pkg/src/cqksolve) for the Newton-on-lambda hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library, and only as the checker or
 * as the timed CPU baseline.  The product (paper_2603_15910_b200) never links
 * or calls it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every entry point against
 * golden vectors produced by the real reference (tests/golden/make_golden.py).
 * Sums emulate numpy's pairwise summation (the reference's `ndarray.sum`), so
 * with the reference's own lambda0 injected (`lam0` argument, NaN = compute it)
 * the iterate sequence is reproduced bit for bit.  lambda0 itself is a BLAS
 * ddot in the reference (core.py:255-256) whose order is OpenBLAS-kernel
 * specific; the oracle uses the pairwise sum there (agreement ~1e-16).
 */
#ifndef CQK_ORACLE_H
#define CQK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_SOLVED = 0,
  ORC_INFEASIBLE = 1,
  ORC_E_DOMAIN = -1,
  ORC_E_MAXITER = -2,
  ORC_E_CONTRACT = -3,
  ORC_E_ALLOC = -4,
};

typedef struct {
  int32_t status;
  int32_t domain_field;   /* 0 d,1 a,2 b,3 l,4 u,5 r,6 bounds,7 y,8 xbar */
  int64_t domain_index;   /* -1 when not element specific */
  double lam;
  double lam0;
  int64_t iterations;
  int64_t phi_evals;
  int64_t fixed_count;
  double bracket_lo, bracket_hi;
} orc_result;

/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src) */
double orc_pairwise_sum(const double *a, int64_t n);

/* core.py:126-165 validate; returns ORC_SOLVED or ORC_E_DOMAIN (+field/index) */
int orc_validate(const double *d, const double *a, const double *b,
                 const double *l, const double *u, int64_t n, double r,
                 orc_result *res);

/* core.py:237-257 initial_multiplier (xbar may be NULL) */
double orc_initial_multiplier(const double *d, const double *a, const double *b,
                              const double *l, const double *u, int64_t n,
                              double r, const double *xbar);

/* core.py:182-212 _phi_scan over idx (NULL = all).  out[4] = value, dminus,
   dplus, abs_bx.  at_lower/at_upper may be NULL. */
int orc_phi_scan(const double *d, const double *a, const double *b,
                 const double *l, const double *u, const int64_t *idx,
                 int64_t m, double lam, double *out, uint8_t *at_lower,
                 uint8_t *at_upper);

/* core.py:168-179 eval_x over idx (NULL = all) into x[m] */
void orc_eval_x(const double *d, const double *a, const double *b,
                const double *l, const double *u, const int64_t *idx,
                int64_t m, double lam, double *x);

/* newton.py:106-121 secant_step; returns 0 or ORC_E_CONTRACT */
int orc_secant_step(double lo, double phi_lo, double hi, double phi_hi,
                    double r, double *out);

/* newton.py:129-162 nearest_breakpoint over idx; dir 0 RIGHT (edge = lo),
   1 LEFT (edge = hi).  Returns 1 when found (value in *out), 0 otherwise. */
int orc_nearest_breakpoint(const double *d, const double *a, const double *b,
                           const double *l, const double *u, const int64_t *idx,
                           int64_t m, double edge, int dir, double *out);

/* newton.py:209-342 solve_cqk.  x may be NULL.  lam0 NaN => initial_multiplier */
int orc_solve_cqk(const double *d, const double *a, const double *b,
                  const double *l, const double *u, int64_t n, double r,
                  int fixing, int64_t max_iter, double tau, const double *xbar,
                  double lam0, int check, double *x, orc_result *res);

/* parallel.py:371-500 jacobi_solve with `workers` contiguous chunks
   (OpenMP threads), per-chunk pairwise partials and _tree_sum. */
int orc_jacobi_solve(const double *d, const double *a, const double *b,
                     const double *l, const double *u, int64_t n, double r,
                     int64_t max_iter, double tau, int workers, double lam0,
                     int check, double *x, orc_result *res);

/* parallel.py:174-327 par_solve_cqk (chunked fixing + merge threshold) */
int orc_par_solve_cqk(const double *d, const double *a, const double *b,
                      const double *l, const double *u, int64_t n, double r,
                      int fixing, int64_t max_iter, double tau, int workers,
                      const double *xbar, int64_t merge_threshold, double lam0,
                      int check, double *x, orc_result *res);

/* simplex.py:47-154 simplex_init_lambda.  free_out[n] receives J (size *nfree),
   fixed_mask[n] the proven zeros.  xbar may be NULL.  idx NULL = all. */
int orc_simplex_init_lambda(const double *y, int64_t n, double r,
                            const int64_t *idx, int64_t p, const double *xbar,
                            int sharpened, double *lam, int64_t *free_out,
                            int64_t *nfree, uint8_t *fixed_mask, double *sumJ);

/* simplex.py:218-308 newton_project_simplex.  lam0 NaN => Algorithm-2 init.
   x (dense) may be NULL.  trace (4 doubles per phi eval) may be NULL,
   trace_cap = max rows. */
int orc_newton_project_simplex(const double *y, int64_t n, double r,
                               int fixing, int64_t max_iter, double tau,
                               const double *xbar, int sharpened, double lam0,
                               double *x, double *trace, int64_t trace_cap,
                               orc_result *res);

/* parallel.py:330-368 par_simplex_init (chunked Algorithm 2 + merge). */
int orc_par_simplex_init(const double *y, int64_t n, double r, int workers, double *lam,
                         int64_t *free_out, int64_t *nfree, uint8_t *fixed_mask, double *sumJ);

/* The Newton loop of simplex.py:252-308 from a given start lam0 (no clamp)
   and free index set (the route newton_project_simplex takes after its
   initializer). */
int orc_newton_simplex_from(const double *y, int64_t n, double r, int fixing, int64_t max_iter,
                            double tau, double lam0, const int64_t *free_idx, int64_t m,
                            double *x, orc_result *res);

/* simplex.py:311-333 project_l1 (dense).  Returns status; res->iterations = -1
   when y is inside the ball (copy). */
int orc_project_l1(const double *y, int64_t n, double r, int fixing,
                   int64_t max_iter, double tau, const double *xbar, double *x,
                   orc_result *res);

/* oracle.py:88-97 oracle_simplex: lam of the sort-based exact projection */
double orc_exact_simplex_lambda(const double *y, int64_t n, double r);

/* C5 batched rows: orc_newton_project_simplex per row, OpenMP over rows;
   returns the count of rows that did not solve */
int64_t orc_project_simplex_rows(const double *Y, int64_t rows, int64_t cols, double r,
                                 int threads, double *X, double *lam, int64_t *iters);

/* cqk_gen.c: instances.py:43-86 generators, sequential (r from pairwise dots) */
int orc_gen_cqk(int family, int64_t n, uint64_t seed, double *d, double *a, double *b,
                double *l, double *u, double *r);
int orc_gen_simplex_y(int family, int64_t n, uint64_t seed, double *y);

#ifdef __cplusplus
}
#endif
#endif

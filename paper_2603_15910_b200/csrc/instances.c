/*
 * instances.c -- seeded benchmark instance generators (host, OpenMP).
 *
 * Bit-compatible with the reference generators: Xoshiro256++ seeded by four
 * SplitMix64 outputs (rng.py:29-62), uniform01 = (x >> 11) * 2^-53
 * (rng.py:66-69), Box-Muller normals consuming two draws each
 * (rng.py:73-79), and the normative per-family draw orders of
 * instances.py:43-86.  Unlike the reference's sequential stream, every
 * OpenMP thread jumps straight to its first draw with a GF(2) matrix power of
 * the xoshiro transition, so generation of n = 1e8..1e9 runs on all cores.
 *
 * The one value that is not bit-compatible is r for the CQK families: the
 * reference forms it from BLAS ddot sums (instances.py:64-66) whose order is
 * OpenBLAS-kernel specific; here the two dots are pairwise sums.  Golden
 * fixtures carry the reference's r.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/cqk_instances.h"

#include "xoshiro_jump.h"

static int nthreads_for(int64_t count) {
#ifdef _OPENMP
  int t = omp_get_max_threads();
  int64_t cap = count / 65536 + 1;
  return (int)(t < cap ? t : cap);
#else
  (void)count;
  return 1;
#endif
}

/* Fill out[k*stride] for k in [0, count) with uniform01 draws starting at
 * draw `offset` of the seed's stream, scaled as lo + u*(hi-lo) when scale. */
typedef enum { K_U01, K_AFFINE, K_NORMAL } draw_kind;

static void fill_draws(uint64_t seed, uint64_t offset, int64_t count, double *out,
                       int64_t stride, draw_kind kind, double p, double q) {
  xo_state s0 = xo_seed(seed);
  int nt = nthreads_for(count);
  const double scale = 1.0 / 9007199254740992.0; /* 2^-53 */
  const double twopi = 2.0 * M_PI;
  int per = kind == K_NORMAL ? 2 : 1;
#pragma omp parallel num_threads(nt)
  {
#ifdef _OPENMP
    int tid = omp_get_thread_num(), T = omp_get_num_threads();
#else
    int tid = 0, T = 1;
#endif
    int64_t k0 = count * tid / T, k1 = count * (tid + 1) / T;
    xo_state st = xo_jump(s0, offset + (uint64_t)k0 * per);
    for (int64_t k = k0; k < k1; ++k) {
      double v;
      if (kind == K_NORMAL) {
        double u1 = (double)((xo_next(&st) >> 11) + 1) * scale;
        double u2 = (double)(xo_next(&st) >> 11) * scale;
        v = sqrt(-2.0 * log(u1)) * cos(twopi * u2);
      } else {
        v = (double)(xo_next(&st) >> 11) * scale;
        if (kind == K_AFFINE) v = p + v * (q - p);
      }
      out[k * stride] = v;
    }
  }
}

int cqk_gen_uniform01(uint64_t seed, uint64_t offset, int64_t count, double *out) {
  fill_draws(seed, offset, count, out, 1, K_U01, 0, 0);
  return 0;
}

int cqk_gen_normal(uint64_t seed, uint64_t offset, int64_t count, double *out) {
  fill_draws(seed, offset, count, out, 1, K_NORMAL, 0, 0);
  return 0;
}

static double pairwise(const double *a, int64_t n) {
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
  return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

/* pairwise sum of b*v computed blockwise so no n-sized temporary is needed
 * (the block boundaries follow the pairwise split, so the result equals the
 * pairwise sum of the materialised products). */
static double dot_pairwise(const double *b, const double *v, int64_t n) {
  if (n <= 131072) {
    double *t = malloc(sizeof(double) * (n ? n : 1));
    for (int64_t i = 0; i < n; ++i) t[i] = b[i] * v[i];
    double s = pairwise(t, n);
    free(t);
    return s;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return dot_pairwise(b, v, n2) + dot_pairwise(b + n2, v + n2, n - n2);
}

/* Each OpenMP thread owns elements [k0, k1) of a tuple stream in which
 * element k consumes draws [off + per*k, off + per*(k+1)). */
#define TUPLE_LOOP(seed, off, count, per, ...)                                \
  do {                                                                         \
    xo_state s0_ = xo_seed(seed);                                              \
    int nt_ = nthreads_for(count);                                             \
    _Pragma("omp parallel num_threads(nt_)") {                                 \
      int tid_ = 0, T_ = 1;                                                    \
      TUPLE_TID(tid_, T_);                                                     \
      int64_t k0 = (count) * tid_ / T_, k1 = (count) * (tid_ + 1) / T_;        \
      xo_state st = xo_jump(s0_, (off) + (uint64_t)k0 * (per));                \
      for (int64_t k = k0; k < k1; ++k) { __VA_ARGS__ }                               \
    }                                                                          \
  } while (0)
#ifdef _OPENMP
#define TUPLE_TID(t, T) (t = omp_get_thread_num(), T = omp_get_num_threads())
#else
#define TUPLE_TID(t, T) ((void)0)
#endif
#define U01() ((double)(xo_next(&st) >> 11) * (1.0 / 9007199254740992.0))

/* Elements [lo, hi) of gen_cqk(family, n, seed) (instances.py:43-70) into
 * arrays of length hi - lo, plus the shard's pairwise b.l and b.u sums.  The
 * draw offsets follow the reference's order: the (d, a, b) tuple of element
 * i at draws per*i.., the (lo, hi) bound pair at 3n (n for correlated) + 2i,
 * and the r draw at that offset + 2n. */
int cqk_gen_cqk_range(int family, int64_t n, uint64_t seed, int64_t lo, int64_t hi, double *d,
                      double *a, double *b, double *l, double *u, double *bl, double *bu) {
  if (n < 1 || family < 0 || family > 2 || lo < 0 || hi > n || lo > hi) return -1;
  const int64_t m = hi - lo;
  const uint64_t per = family == CQK_FAMILY_CORRELATED ? 1 : 3;
  const uint64_t off = per * (uint64_t)n;
  if (m > 0) {
    if (family == CQK_FAMILY_UNCORRELATED) {
      /* flat = uniform(10, 25, 3n); d, a, b = flat[0::3], flat[1::3], flat[2::3] */
      TUPLE_LOOP(seed, 3 * (uint64_t)lo, m, 3, {
        d[k] = 10.0 + U01() * (25.0 - 10.0);
        a[k] = 10.0 + U01() * (25.0 - 10.0);
        b[k] = 10.0 + U01() * (25.0 - 10.0);
      });
    } else if (family == CQK_FAMILY_WEAKLY) {
      TUPLE_LOOP(seed, 3 * (uint64_t)lo, m, 3, {
        double f0 = U01(), f1 = U01(), f2 = U01();
        double bk = 10.0 + 15.0 * f0;
        b[k] = bk;
        d[k] = (bk - 5.0) + 10.0 * f1;
        a[k] = (bk - 5.0) + 10.0 * f2;
      });
    } else {
      TUPLE_LOOP(seed, (uint64_t)lo, m, 1, {
        double bk = 10.0 + U01() * (25.0 - 10.0);
        b[k] = bk;
        d[k] = bk + 5.0;
        a[k] = bk + 5.0;
      });
    }
    /* pair = uniform(10, 25, 2n); l = min(pair[0::2], pair[1::2]), u = max */
    TUPLE_LOOP(seed, off + 2 * (uint64_t)lo, m, 2, {
      double p0 = 10.0 + U01() * (25.0 - 10.0);
      double p1 = 10.0 + U01() * (25.0 - 10.0);
      l[k] = p0 < p1 ? p0 : p1;
      u[k] = p0 > p1 ? p0 : p1;
    });
  }
  if (bl) *bl = dot_pairwise(b, l, m);
  if (bu) *bu = dot_pairwise(b, u, m);
  return 0;
}

/* r = b.l + U * (b.u - b.l) with the reference's final draw (instances.py:64-66) */
double cqk_gen_cqk_r(int family, int64_t n, uint64_t seed, double bl, double bu) {
  const uint64_t per = family == CQK_FAMILY_CORRELATED ? 1 : 3;
  double ur;
  fill_draws(seed, per * (uint64_t)n + 2 * (uint64_t)n, 1, &ur, 1, K_U01, 0, 0);
  return bl + ur * (bu - bl);
}

int cqk_gen_cqk(int family, int64_t n, uint64_t seed, double *d, double *a, double *b,
                double *l, double *u, double *r_out) {
  double bl, bu;
  int rc = cqk_gen_cqk_range(family, n, seed, 0, n, d, a, b, l, u, &bl, &bu);
  if (rc) return rc;
  *r_out = cqk_gen_cqk_r(family, n, seed, bl, bu);
  return 0;
}

/* instances.py:73-86: redraw the whole vector (continuing stream) while any
 * entry is exactly zero. */
int cqk_gen_simplex_y(int family, int64_t n, uint64_t seed, double *y) {
  if (n < 1 || family < 0 || family > 2) return -1;
  uint64_t per = family == SIMPLEX_FAMILY_U01 ? 1 : 2;
  for (uint64_t attempt = 0;; ++attempt) {
    uint64_t off = attempt * per * (uint64_t)n;
    if (family == SIMPLEX_FAMILY_U01) fill_draws(seed, off, n, y, 1, K_U01, 0, 0);
    else fill_draws(seed, off, n, y, 1, K_NORMAL, 0, 0);
    if (family == SIMPLEX_FAMILY_N0M3) {
      const double sd = sqrt(1e-3);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) y[i] *= sd;
    }
    int64_t zeros = 0;
#pragma omp parallel for reduction(+ : zeros) schedule(static)
    for (int64_t i = 0; i < n; ++i) zeros += y[i] == 0.0;
    if (!zeros) return 0;
  }
}

/*
 * cqk_gen.c -- TEST INFRASTRUCTURE ONLY (see cqk_oracle.h).
 *
 * Plain sequential restatement of the reference's seeded instance generators,
 * so that the checker and bench.py's `--impl reference` arm build their inputs
 * without loading any product library:
 *
 *   rng.py:29-62     Xoshiro256++ seeded by four SplitMix64 outputs
 *   rng.py:66-69     uniform01 = (x >> 11) * 2^-53
 *   rng.py:73-79     Box-Muller normal, two raw draws per value (cosine kept)
 *   instances.py:43-70  gen_cqk draw order (per family), bounds pair, r draw
 *   instances.py:73-86  gen_simplex_y (whole-vector redraw on an exact zero)
 *
 * One stream, one thread, no skip-ahead: the draws are consumed in exactly the
 * order the reference's numba loops consume them.  The only value that is not
 * the reference's bit for bit is r: the reference forms b.l and b.u with a
 * BLAS ddot (instances.py:64-65); here they are numpy-pairwise sums of the
 * materialised products (np.sum(b * l)), the same convention the product's
 * generator documents, so both arms of the benchmark see one identical r.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "cqk_oracle.h"

typedef struct { uint64_t s[4]; } orc_xo;

static uint64_t splitmix(uint64_t *z) { /* rng.py:32-38 */
  *z += 0x9E3779B97F4A7C15ull;
  uint64_t o = *z;
  o = (o ^ (o >> 30)) * 0xBF58476D1CE4E5B9ull;
  o = (o ^ (o >> 27)) * 0x94D049BB133111EBull;
  return o ^ (o >> 31);
}

static orc_xo xo_seeded(uint64_t seed) { /* rng.py:41-47 */
  orc_xo x;
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) x.s[i] = splitmix(&z);
  return x;
}

static inline uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static inline uint64_t xo_u64(orc_xo *x) { /* rng.py:55-64 */
  uint64_t *s = x->s;
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

static inline double u01(orc_xo *x) { return (double)(xo_u64(x) >> 11) * (1.0 / 9007199254740992.0); }

static inline double normal(orc_xo *x) { /* rng.py:73-79 */
  const double scale = 1.0 / 9007199254740992.0;
  const double u1 = (double)((xo_u64(x) >> 11) + 1) * scale;
  const double u2 = (double)(xo_u64(x) >> 11) * scale;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* np.sum(b * v): the products materialised blockwise along the pairwise
 * split, so the result equals orc_pairwise_sum of the full product array. */
static double dot_pairwise(const double *b, const double *v, int64_t n, double *t) {
  if (n <= 65536) {
    for (int64_t i = 0; i < n; ++i) t[i] = b[i] * v[i];
    return orc_pairwise_sum(t, n);
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return dot_pairwise(b, v, n2, t) + dot_pairwise(b + n2, v + n2, n - n2, t);
}

/* family: 0 cqk-uncorrelated, 1 cqk-weakly-correlated, 2 cqk-correlated */
int orc_gen_cqk(int family, int64_t n, uint64_t seed, double *d, double *a, double *b,
                double *l, double *u, double *r) {
  if (n < 1 || family < 0 || family > 2) return -1;
  orc_xo x = xo_seeded(seed);
  if (family == 0) { /* flat = uniform(10, 25, 3n); d, a, b = flat[0::3], [1::3], [2::3] */
    for (int64_t i = 0; i < n; ++i) {
      d[i] = 10.0 + u01(&x) * (25.0 - 10.0);
      a[i] = 10.0 + u01(&x) * (25.0 - 10.0);
      b[i] = 10.0 + u01(&x) * (25.0 - 10.0);
    }
  } else if (family == 1) { /* flat = uniform01(3n); b, d, a from flat[0::3], [1::3], [2::3] */
    for (int64_t i = 0; i < n; ++i) {
      const double f0 = u01(&x), f1 = u01(&x), f2 = u01(&x);
      b[i] = 10.0 + 15.0 * f0;
      d[i] = (b[i] - 5.0) + 10.0 * f1;
      a[i] = (b[i] - 5.0) + 10.0 * f2;
    }
  } else { /* b = uniform(10, 25, n); d = a = b + 5 */
    for (int64_t i = 0; i < n; ++i) {
      b[i] = 10.0 + u01(&x) * (25.0 - 10.0);
      d[i] = b[i] + 5.0;
      a[i] = b[i] + 5.0;
    }
  }
  for (int64_t i = 0; i < n; ++i) { /* pair = uniform(10, 25, 2n); l = min, u = max */
    const double p0 = 10.0 + u01(&x) * (25.0 - 10.0);
    const double p1 = 10.0 + u01(&x) * (25.0 - 10.0);
    l[i] = p0 < p1 ? p0 : p1;
    u[i] = p0 > p1 ? p0 : p1;
  }
  double *t = malloc(sizeof(double) * 65536);
  if (!t) return ORC_E_ALLOC;
  const double bl = dot_pairwise(b, l, n, t), bu = dot_pairwise(b, u, n, t);
  free(t);
  *r = bl + u01(&x) * (bu - bl); /* instances.py:66 */
  return 0;
}

/* family: 0 simplex-u01, 1 simplex-n01, 2 simplex-n0m3 (N(0, 1e-3) as variance) */
int orc_gen_simplex_y(int family, int64_t n, uint64_t seed, double *y) {
  if (n < 1 || family < 0 || family > 2) return -1;
  orc_xo x = xo_seeded(seed);
  const double sd = sqrt(1e-3);
  for (;;) {
    int64_t zeros = 0;
    for (int64_t i = 0; i < n; ++i) {
      double v = family == 0 ? u01(&x) : normal(&x);
      if (family == 2) v *= sd;
      y[i] = v;
      zeros += v == 0.0;
    }
    if (!zeros) return 0;
  }
}

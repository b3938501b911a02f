/*
 * cqk_instances.h -- seeded instance generators (host, OpenMP), bit-compatible
 * with the reference's Xoshiro256++ stream and draw order.
 *
 * Replaces (reference): cqksolve.rng.Xoshiro256pp (rng.py:82-106),
 * cqksolve.instances.gen_cqk (instances.py:43-70) and gen_simplex_y
 * (instances.py:73-86).  Inputs only -- not on the solver hot path.
 */
#ifndef CQK_INSTANCES_H
#define CQK_INSTANCES_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { CQK_FAMILY_UNCORRELATED = 0, CQK_FAMILY_WEAKLY = 1, CQK_FAMILY_CORRELATED = 2 };
enum { SIMPLEX_FAMILY_U01 = 0, SIMPLEX_FAMILY_N01 = 1, SIMPLEX_FAMILY_N0M3 = 2 };

/* uniform01 draws [offset, offset+count) of the stream seeded with `seed` */
int cqk_gen_uniform01(uint64_t seed, uint64_t offset, int64_t count, double *out);
/* Box-Muller normals; normal k consumes draws offset+2k, offset+2k+1 */
int cqk_gen_normal(uint64_t seed, uint64_t offset, int64_t count, double *out);
/* gen_cqk(family, n, seed): fills d, a, b, l, u (length n) and *r */
int cqk_gen_cqk(int family, int64_t n, uint64_t seed, double *d, double *a, double *b,
                double *l, double *u, double *r);
/* elements [lo, hi) of gen_cqk(family, n, seed) (arrays of length hi - lo),
   with the shard's b.l and b.u sums (for r on a sharded instance) */
int cqk_gen_cqk_range(int family, int64_t n, uint64_t seed, int64_t lo, int64_t hi, double *d,
                      double *a, double *b, double *l, double *u, double *bl, double *bu);
/* r from the full b.l and b.u sums and the stream's final draw */
double cqk_gen_cqk_r(int family, int64_t n, uint64_t seed, double bl, double bu);
/* gen_simplex_y(family, n, seed) */
int cqk_gen_simplex_y(int family, int64_t n, uint64_t seed, double *y);

#ifdef __cplusplus
}
#endif
#endif

/* xoshiro_jump.h -- Xoshiro256++ (rng.py:29-62) and GF(2) skip-ahead, shared
 * by the host generators (instances.c) and the device generator's host-side
 * set-up (cqk_abi.cu). */
#pragma once
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s[4]; } xo_state;

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static inline uint64_t xo_next(xo_state *st) {
  uint64_t *s = st->s;
  uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

static inline xo_state xo_seed(uint64_t seed) {
  xo_state st;
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) {
    z += 0x9E3779B97F4A7C15ULL;
    uint64_t o = z;
    o = (o ^ (o >> 30)) * 0xBF58476D1CE4E5B9ULL;
    o = (o ^ (o >> 27)) * 0x94D049BB133111EBULL;
    st.s[i] = o ^ (o >> 31);
  }
  return st;
}

/* ---- GF(2) skip-ahead: the state transition is linear on 256 bits. ---- */
typedef struct { uint64_t col[256][4]; } gf2mat; /* column j = image of e_j */

static inline void mat_apply(const gf2mat *m, const uint64_t v[4], uint64_t out[4]) {
  uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  for (int w = 0; w < 4; ++w) {
    uint64_t bits = v[w];
    while (bits) {
      int b = __builtin_ctzll(bits);
      bits &= bits - 1;
      const uint64_t *c = m->col[w * 64 + b];
      r0 ^= c[0]; r1 ^= c[1]; r2 ^= c[2]; r3 ^= c[3];
    }
  }
  out[0] = r0; out[1] = r1; out[2] = r2; out[3] = r3;
}

static inline void mat_mul(const gf2mat *a, const gf2mat *b, gf2mat *out) {
  for (int j = 0; j < 256; ++j) mat_apply(a, b->col[j], out->col[j]);
}

static inline void transition_matrix(gf2mat *m) {
  for (int j = 0; j < 256; ++j) {
    xo_state st = {{0, 0, 0, 0}};
    st.s[j / 64] = 1ULL << (j % 64);
    xo_next(&st);
    memcpy(m->col[j], st.s, sizeof st.s);
  }
}

/* state advanced by k draws */
static inline xo_state xo_jump(xo_state st, uint64_t k) {
  if (k == 0) return st;
  gf2mat *base = (gf2mat *)malloc(sizeof(gf2mat)), *tmp = (gf2mat *)malloc(sizeof(gf2mat));
  transition_matrix(base);
  uint64_t v[4];
  memcpy(v, st.s, sizeof v);
  while (k) {
    if (k & 1) {
      uint64_t o[4];
      mat_apply(base, v, o);
      memcpy(v, o, sizeof v);
    }
    k >>= 1;
    if (k) {
      mat_mul(base, base, tmp);
      gf2mat *sw = base; base = tmp; tmp = sw;
    }
  }
  memcpy(st.s, v, sizeof v);
  free(base);
  free(tmp);
  return st;
}


/* states[k] = state after base + k * stride draws, k < count (one matrix
 * power, then one matrix-vector product per state). */
static inline void xo_jump_states(uint64_t seed, uint64_t base, uint64_t stride, int64_t count,
                                  xo_state *states) {
  xo_state s = xo_jump(xo_seed(seed), base);
  if (count <= 0) return;
  states[0] = s;
  if (count == 1) return;
  /* M = T^stride by square-and-multiply on matrices */
  gf2mat *acc = (gf2mat *)malloc(sizeof(gf2mat)), *sq = (gf2mat *)malloc(sizeof(gf2mat)),
         *tmp = (gf2mat *)malloc(sizeof(gf2mat));
  for (int j = 0; j < 256; ++j) {
    memset(acc->col[j], 0, sizeof acc->col[j]);
    acc->col[j][j / 64] = 1ULL << (j % 64);
  }
  transition_matrix(sq);
  uint64_t k = stride;
  while (k) {
    if (k & 1) {
      mat_mul(sq, acc, tmp);
      gf2mat *t = acc; acc = tmp; tmp = t;
    }
    k >>= 1;
    if (k) {
      mat_mul(sq, sq, tmp);
      gf2mat *t = sq; sq = tmp; tmp = t;
    }
  }
  for (int64_t i = 1; i < count; ++i) {
    uint64_t o[4];
    mat_apply(acc, states[i - 1].s, o);
    memcpy(states[i].s, o, sizeof o);
  }
  free(acc); free(sq); free(tmp);
}

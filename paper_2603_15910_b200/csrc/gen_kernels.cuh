// gen_kernels.cuh -- on-device benchmark instances.
//
// Bit-identical to the reference generators for the uniform families
// (instances.py:43-86, rng.py:53-69): every thread continues the Xoshiro256++
// stream from a host-computed GF(2) jump state and produces a contiguous range
// of elements in the reference's draw order.  Uniform draws are integer ops
// plus one exact scaling, so no libm enters.  The CQK level r is formed from
// device sums of b.l and b.u (not the reference's BLAS order).
#pragma once
#include <stdint.h>

namespace cqk {

struct XoState {
  unsigned long long s[4];
};

DEVI unsigned long long xo_rotl(unsigned long long x, int k) { return (x << k) | (x >> (64 - k)); }
DEVI double xo_u01(XoState& st) {
  unsigned long long* s = st.s;
  const unsigned long long result = xo_rotl(s[0] + s[3], 23) + s[0];
  const unsigned long long t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = xo_rotl(s[3], 45);
  return (double)(result >> 11) * 0x1p-53;
}

// family 0 uncorrelated, 1 weakly, 2 correlated; thread k owns elements
// [k*per, min(n, (k+1)*per)); st_tuple[k] / st_pair[k] are its stream states.
// (n here = elements to produce; element i of the output is element lo + i
// of the instance -- the states already point at element lo.)
__global__ void __launch_bounds__(256) gen_cqk_kernel(int family, int64_t n, int64_t per,
                                                      const XoState* __restrict__ st_tuple,
                                                      const XoState* __restrict__ st_pair,
                                                      double* d, double* a, double* b, double* l,
                                                      double* u) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i0 = k * per;
  if (i0 >= n) return;
  const int64_t i1 = i0 + per < n ? i0 + per : n;
  XoState s1 = st_tuple[k], s2 = st_pair[k];
  for (int64_t i = i0; i < i1; ++i) {
    double bi;
    if (family == 0) {
      d[i] = __dadd_rn(10.0, __dmul_rn(xo_u01(s1), 15.0));
      a[i] = __dadd_rn(10.0, __dmul_rn(xo_u01(s1), 15.0));
      bi = __dadd_rn(10.0, __dmul_rn(xo_u01(s1), 15.0));
      b[i] = bi;
    } else if (family == 1) {
      const double f0 = xo_u01(s1), f1 = xo_u01(s1), f2 = xo_u01(s1);
      bi = __dadd_rn(10.0, __dmul_rn(15.0, f0));
      b[i] = bi;
      d[i] = __dadd_rn(__dsub_rn(bi, 5.0), __dmul_rn(10.0, f1));
      a[i] = __dadd_rn(__dsub_rn(bi, 5.0), __dmul_rn(10.0, f2));
    } else {
      bi = __dadd_rn(10.0, __dmul_rn(xo_u01(s1), 15.0));
      b[i] = bi;
      d[i] = __dadd_rn(bi, 5.0);
      a[i] = __dadd_rn(bi, 5.0);
    }
    const double p0 = __dadd_rn(10.0, __dmul_rn(xo_u01(s2), 15.0));
    const double p1 = __dadd_rn(10.0, __dmul_rn(xo_u01(s2), 15.0));
    l[i] = p0 < p1 ? p0 : p1;
    u[i] = p0 > p1 ? p0 : p1;
  }
}

// simplex-u01: y[i] = uniform01 draw i (of the given attempt's block)
__global__ void __launch_bounds__(256) gen_u01_kernel(int64_t n, int64_t per,
                                                      const XoState* __restrict__ st, double* y,
                                                      unsigned long long* zeros) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i0 = k * per;
  if (i0 >= n) return;
  const int64_t i1 = i0 + per < n ? i0 + per : n;
  XoState s = st[k];
  unsigned long long z = 0;
  for (int64_t i = i0; i < i1; ++i) {
    const double v = xo_u01(s);
    y[i] = v;
    z += v == 0.0;
  }
  if (z) atomicAdd(zeros, z);
}

// block partials of (sum b*l, sum b*u) for r
__global__ void __launch_bounds__(256) dot_bl_bu_kernel(const double* b, const double* l,
                                                        const double* u, int64_t n,
                                                        double* partials) {
  __shared__ double s_red[8][kMaxK];
  __shared__ double s_tot[kMaxK];
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    acc[0] += __dmul_rn(b[i], l[i]);
    acc[1] += __dmul_rn(b[i], u[i]);
  }
  const int ops[2] = {OP_SUM, OP_SUM};
  block_reduce<2>(acc, ops, s_red, s_tot);
  if (threadIdx.x < 2) partials[blockIdx.x * kMaxK + threadIdx.x] = s_tot[threadIdx.x];
}

}  // namespace cqk

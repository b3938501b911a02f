// cqk_rows.cuh -- C5: batched row-wise simplex projection, one warp per row,
// one pass over the row (sm_100a, fp64).
//
// Per row the reference semantics are newton_project_simplex(Y[i], r,
// lambda0=min((r - sum y)/n, r - max y)) (simplex.py:218-308, the lambda0=
// route: clamp to -max y, Algorithm 4 with at-zero dropping).  That start is
// an upper bound of the root, the iterates only decrease from it, so every
// variable that is ever positive (or at zero) satisfies
//     y_i + lam_k >= 0  with  lam_k <= lam_0 <= fl(r - max y)
// hence y_i >= -fl(r - max y).  A warp streams its row ONCE: it sums y,
// tracks the running (warp) max m and captures every y_i >= -fl(r - m) --
// m never exceeds the row's max, so the captured set is a superset of every
// iterate's support -- and writes the row's zeros to x as it goes.  The
// Newton iterations then run on the captured candidates held in registers
// (typically ~1-2% of the row), and x leaves as the zero fill plus a scatter
// of the positive candidates.  No row ever sits in shared memory, so the SM
// keeps dozens of rows in flight (the previous CTA-per-row design held six
// 32 KB rows per SM and was per-row latency bound, 0.75 of the copy peak).
//
// Rows reach the warps through per-warp rings of 1-D bulk copies (chunks of
// 2 KB, four in flight per warp, issued across row boundaries) and rows are
// handed out by a grid counter, so slow-streaming SMs simply take fewer rows.
//
// A row whose candidates overflow the warp's slots (e.g. u01 rows, where
// max y - r is below every y) or whose start is not below fl(r - max y) (the
// formula start, an explicit lambda0) gets a second capture against its
// actual start: every iterate stays at or below lambda0, so y >= -lambda0
// covers them (one more read of the row, from L2).  If that overflows too, or
// an iterate leaves the captured range (an explicit lambda0 below the root),
// or the deriv <= 0 snap is reached (simplex.py:276-281), the row takes the
// general warp path: the same Algorithm 4 over the whole row, re-read per phi
// evaluation.  Every path is deterministic per row.
#pragma once
#include "cqk_kernels.cuh"

namespace cqk {

constexpr int kRsWarps = 8;                // warps per CTA
constexpr int kRsCap = 256;                // candidate slots per warp
constexpr int kRsPer = kRsCap / 32;        // candidates per lane in registers
constexpr int kRsU = 4;                    // 16-byte pairs per lane per chunk (2 KB chunks)
constexpr int kRsStages = 4;               // chunks in flight per warp

DEVI int rs_warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Algorithm 4's state machine (simplex.py:256-294), shared by both paths:
// given phi at lam (value, #t>0, #t==0 over the free set) advance the state.
// Returns 0 continue, 1 done (lam final), 2 the deriv <= 0 snap is needed.
struct RsState {
  double lam, lo, hi, fix_hi;
  int iterations;
};
DEVI int rs_step(RsState& s, double value, int tpos, int tz, double r, double tau, int max_iter,
                 int fixing) {
  const double dminus = (double)tpos, dplus = (double)(tpos + tz);
  double deriv;
  if (s.iterations == 0) {
    if (value == r) return 1;
    deriv = value < r ? dplus : dminus;
  } else {
    if (value <= r) return 1;
    deriv = dminus;
  }
  if (value < r) s.lo = s.lam;
  else {
    s.hi = s.lam;
    if (fixing) s.fix_hi = s.lam;  // drops y + fix_hi <= 0 from now on
  }
  if (deriv <= 0) return 2;
  const double step = -(value - r) / deriv;
  const double next = s.lam + step;
  if (fabs(step) < tau || next == s.lam) { s.lam = next; return 1; }
  if (isfinite(s.lo) && isfinite(s.hi) && s.hi - s.lo < tau * fmax(fabs(s.hi), fabs(s.lo))) {
    s.lam = next;
    return 1;
  }
  s.lam = next;
  ++s.iterations;
  return s.iterations > max_iter ? 1 : 0;
}

// The general path: Algorithm 4 over the whole row (global memory), x dense.
DEVI void rs_general(const double* __restrict__ y, double* __restrict__ x, int cols, double lam0,
                     double r, double tau, int max_iter, int fixing, int lane, double& lam_out,
                     int& it_out) {
  RsState s{lam0, -HUGE_VAL, HUGE_VAL, HUGE_VAL, 0};
  const double2* y2 = reinterpret_cast<const double2*>(y);
  const int P = cols >> 1;
  for (;;) {
    double v0 = 0.0, v1 = 0.0;
    int p = 0, z = 0;
    const bool drop = fixing && isfinite(s.fix_hi);
    for (int q = lane; q < P; q += 32) {
      const double2 v = y2[q];
      const bool a0 = !drop || __dadd_rn(v.x, s.fix_hi) > 0, a1 = !drop || __dadd_rn(v.y, s.fix_hi) > 0;
      const double t0 = __dadd_rn(v.x, s.lam), t1 = __dadd_rn(v.y, s.lam);
      v0 += a0 && t0 > 0 ? t0 : 0.0;
      v1 += a1 && t1 > 0 ? t1 : 0.0;
      p += (a0 && t0 > 0) + (a1 && t1 > 0);
      z += (a0 && t0 == 0) + (a1 && t1 == 0);
    }
    const double value = warp_sum(v0 + v1);
    const int tpos = rs_warp_sum_i(p), tz = rs_warp_sum_i(z);
    const int st = rs_step(s, value, tpos, tz, r, tau, max_iter, fixing);
    if (st == 1) break;
    if (st == 2) {  // lam fell below every remaining breakpoint: snap to the largest
      double mneg = -HUGE_VAL;
      const bool drop2 = fixing && isfinite(s.fix_hi);
      for (int q = lane; q < P; q += 32) {
        const double2 v = y2[q];
        if (!drop2 || __dadd_rn(v.x, s.fix_hi) > 0) mneg = fmax(mneg, -v.x);
        if (!drop2 || __dadd_rn(v.y, s.fix_hi) > 0) mneg = fmax(mneg, -v.y);
      }
      s.lam = warp_max(mneg);
      ++s.iterations;
    }
  }
  __syncwarp();  // the streamed zeros of every lane land before these stores
  double2* x2 = reinterpret_cast<double2*>(x);
  for (int q = lane; q < P; q += 32) {
    const double2 v = y2[q];
    const double t0 = __dadd_rn(v.x, s.lam), t1 = __dadd_rn(v.y, s.lam);
    __stcs(x2 + q, make_double2(t0 > 0 ? t0 : 0.0, t1 > 0 ? t1 : 0.0));
  }
  lam_out = s.lam;
  it_out = s.iterations;
}

// One streamed step of a row: U pairs per lane (pair index q0 + 32u, valid
// below P), already in registers.  Writes the zeros of x, accumulates the
// sum, the running warp max m and captures y >= -fl(r - m) into the warp's
// candidate slots (count cnt, warp-uniform; may exceed kRsCap = overflow).
template <int U>
DEVI void rs_consume(const double2 (&v)[U], int q0, int P, double2* __restrict__ x2, double r,
                     int lane, double& s0, double& s1, double& m, int& cnt, double* cv,
                     uint16_t* ci) {
  double lm = -HUGE_VAL;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int q = q0 + 32 * u;
    if (q < P) {
      __stcs(x2 + q, make_double2(0.0, 0.0));
      s0 += v[u].x;
      s1 += v[u].y;
      lm = fmax(lm, fmax(v[u].x, v[u].y));
    }
  }
  m = fmax(m, warp_max(lm));
  const double nthr = -__dadd_rn(r, -m);  // y >= nthr  <=>  y + fl(r - m) >= 0
  int c = 0;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (q0 + 32 * u < P) c += (v[u].x >= nthr) + (v[u].y >= nthr);
  if (__any_sync(0xffffffffu, c)) {
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    int pos = cnt + inc - c;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + 32 * u;
      if (q >= P) continue;
      if (v[u].x >= nthr) {
        if (pos < kRsCap) { cv[pos] = v[u].x; ci[pos] = (uint16_t)(2 * q); }
        ++pos;
      }
      if (v[u].y >= nthr) {
        if (pos < kRsCap) { cv[pos] = v[u].y; ci[pos] = (uint16_t)(2 * q + 1); }
        ++pos;
      }
    }
    cnt += __shfl_sync(0xffffffffu, inc, 31);
  }
}

// Capture every y >= -lam of a row (global memory) into the candidate slots;
// returns the count (warp-uniform), stopping early once it overflows.
DEVI int rs_capture(const double2* __restrict__ y2, int P, double lam, int lane, double* cv,
                    uint16_t* ci) {
  const double nthr = -lam;
  int cnt = 0;
  for (int q0 = 0; q0 < P && cnt <= kRsCap; q0 += 32) {
    const int q = q0 + lane;
    const double2 v = q < P ? __ldcg(y2 + q) : make_double2(-HUGE_VAL, -HUGE_VAL);
    const int c = (v.x >= nthr) + (v.y >= nthr);
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    int pos = cnt + inc - c;
    if (v.x >= nthr) {
      if (pos < kRsCap) { cv[pos] = v.x; ci[pos] = (uint16_t)(2 * q); }
      ++pos;
    }
    if (v.y >= nthr && pos < kRsCap) { cv[pos] = v.y; ci[pos] = (uint16_t)(2 * q + 1); }
    cnt += __shfl_sync(0xffffffffu, inc, 31);
  }
  return cnt;
}

// After the row's last step: lambda0, Algorithm 4 on the candidates (or the
// general path), the scatter of the positive candidates, lam / iterations.
DEVI void rs_row_end(const double* __restrict__ Y, double* __restrict__ X, double* __restrict__ lam_out,
                     int32_t* __restrict__ it_out, int64_t row, int cols, double r, double tau,
                     int max_iter, int fixing, double lam0_given, int start, int lane, double s0,
                     double s1, double m, int cnt, double* cv, uint16_t* ci) {
  const double sum = warp_sum(s0 + s1);
  const double formula = (r - sum) / (double)cols, tight = r - m;
  double lam = !isnan(lam0_given) ? lam0_given : (start && tight < formula ? tight : formula);
  lam = lam >= -m ? lam : -m;
  double lam_fin;
  int it_fin;
  // the captured set holds every y with y + cap_lam >= 0
  double cap_lam = tight;
  bool fast = cnt <= kRsCap && lam <= tight;
  if (!fast) {
    // second chance: the iterates never exceed lam0 when it bounds the root
    // (both reference starts do), so capture y >= -lam0 in one more read of
    // the row (L2-resident: just streamed); fits unless the start is far out
    __syncwarp();
    cnt = rs_capture(reinterpret_cast<const double2*>(Y + row * (int64_t)cols), cols >> 1, lam,
                     lane, cv, ci);
    cap_lam = lam;
    fast = cnt <= kRsCap;
  }
  if (fast) {
    __syncwarp();
    double c[kRsPer];
#pragma unroll
    for (int k = 0; k < kRsPer; ++k) {
      const int j = lane + 32 * k;
      c[k] = j < cnt ? cv[j] : -HUGE_VAL;  // -inf: never positive, never at zero
    }
    RsState s{lam, -HUGE_VAL, HUGE_VAL, HUGE_VAL, 0};
    for (;;) {
      if (!(s.lam <= cap_lam)) { fast = false; break; }  // left the captured range
      double val = 0.0;
      int p = 0, z = 0;
#pragma unroll
      for (int k = 0; k < kRsPer; ++k) {
        const bool a = !fixing || __dadd_rn(c[k], s.fix_hi) > 0;  // fix_hi = +inf: all active
        const double t = __dadd_rn(c[k], s.lam);
        val += a && t > 0 ? t : 0.0;
        p += a && t > 0;
        z += a && t == 0;
      }
      const double value = warp_sum(val);
      const int tpos = rs_warp_sum_i(p), tz = rs_warp_sum_i(z);
      const int stp = rs_step(s, value, tpos, tz, r, tau, max_iter, fixing);
      if (stp == 1) break;
      if (stp == 2) { fast = false; break; }  // the snap needs the whole row
    }
    if (fast) {
      __syncwarp();  // every lane's zeros are issued before the scatter
      double* xr = X + row * (int64_t)cols;
#pragma unroll
      for (int k = 0; k < kRsPer; ++k) {
        const int j = lane + 32 * k;
        const double t = __dadd_rn(c[k], s.lam);
        if (j < cnt && t > 0) xr[ci[j]] = t;
      }
      lam_fin = s.lam;
      it_fin = s.iterations;
    }
  }
  if (!fast)
    rs_general(Y + row * (int64_t)cols, X + row * (int64_t)cols, cols, lam, r, tau, max_iter,
               fixing, lane, lam_fin, it_fin);
  if (lane == 0) {
    if (lam_out) lam_out[row] = lam_fin;
    if (it_out) it_out[row] = it_fin;
  }
  __syncwarp();  // the candidate slots are reused by the next row
}

// The same per-row work fed by 1-D bulk copies (TMA engine): each warp owns a
// ring of NS chunk stages (32 * U pairs each) with one mbarrier per stage;
// lane 0 issues the chunk NS ahead -- across row boundaries -- as soon as the
// warp has read a stage, so a warp keeps NS chunks in flight through its
// row-end work, without holding them in registers.  Rows: the warp's static
// first row, then (dyn != nullptr) rows handed out by a grid counter, or every
// GW-th row.
template <int U, int NS>
__host__ __device__ constexpr size_t rs_tma_warp_bytes() {
  return ((size_t)NS * 32 * U * 16 + (size_t)kRsCap * 8 + (size_t)kRsCap * 2 + (size_t)NS * 16 +
          127) / 128 * 128;
}

template <int U, int NS, int NW>
__global__ void __launch_bounds__(32 * NW) spx_rows_tma_kernel(
    const double* __restrict__ Y, double* __restrict__ X, double* __restrict__ lam_out,
    int32_t* __restrict__ it_out, int64_t rows, int cols, double r, double tau, int max_iter,
    int fixing, double lam0_given, int start, unsigned* dyn, unsigned* dyn_next) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int CH = 32 * U;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char* base = smem_raw + rs_tma_warp_bytes<U, NS>() * w;
  double2* stage = reinterpret_cast<double2*>(base);
  double* cv = reinterpret_cast<double*>(base + (size_t)NS * CH * 16);
  uint16_t* ci = reinterpret_cast<uint16_t*>(cv + kRsCap);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(ci + kRsCap) + 7) & ~(uintptr_t)7);
  long long* rowid = reinterpret_cast<long long*>(bar + NS);
  const int P = cols >> 1;
  const int S = (P + CH - 1) / CH;
  const int64_t GW = (int64_t)gridDim.x * NW;
  const int64_t gw = (int64_t)blockIdx.x * NW + w;
  // issuer state (lane 0 only)
  int64_t i_row = gw;
  int i_c = 0;
  auto issue = [&](int s) {
    if (i_row >= rows) {
      rowid[s] = -1;
      return;
    }
    const int q = i_c * CH;
    const unsigned bytes = (unsigned)((P - q < CH ? P - q : CH) * 16);
    rowid[s] = i_row;
    mbar_expect_tx(&bar[s], bytes);
    tma_load_1d(stage + (size_t)s * CH, Y + i_row * (int64_t)cols + 2 * (int64_t)q, bytes, &bar[s]);
    if (++i_c == S) {
      i_c = 0;
      i_row = dyn ? (int64_t)atomicAdd(dyn, 1u) + GW : i_row + GW;
    }
  };
  if (dyn_next && blockIdx.x == 0 && threadIdx.x == 0) *dyn_next = 0;  // the next launch's
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NS; ++s) issue(s);
  }
  __syncwarp();
  unsigned q = 0;  // chunks consumed
  for (;;) {
    int s = (int)(q % NS);
    const long long row = rowid[s];
    if (row < 0) break;
    double2* x2 = reinterpret_cast<double2*>(X + row * (int64_t)cols);
    double s0 = 0.0, s1 = 0.0, m = -HUGE_VAL;
    int cnt = 0;
    for (int c = 0; c < S; ++c, ++q) {
      s = (int)(q % NS);
      mbar_wait(&bar[s], (q / NS) & 1u);
      double2 v[U];
      const int q0 = c * CH + lane;
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = q0 + 32 * u < P ? stage[(size_t)s * CH + 32 * u + lane] : make_double2(-HUGE_VAL, -HUGE_VAL);
      __syncwarp();  // every lane has read the stage
      if (lane == 0) issue(s);
      rs_consume<U>(v, q0, P, x2, r, lane, s0, s1, m, cnt, cv, ci);
    }
    rs_row_end(Y, X, lam_out, it_out, row, cols, r, tau, max_iter, fixing, lam0_given, start, lane,
               s0, s1, m, cnt, cv, ci);
  }
}

}  // namespace cqk

// cqk_solver.cuh -- persistent single-launch CQK solve (sm_100a).
//
// One cooperative launch performs the whole of newton.solve_cqk
// (newton.py:209-342) / parallel.jacobi_solve (parallel.py:371-500) /
// parallel.par_solve_cqk (parallel.py:174-327):
//
//   pass 0   validate (core.py:126-165) fused with the lambda0 sums
//            (core.py:237-257)                                  24..48 B/elem
//   pass k   phi scan at lambda_k (core.py:182-212) over the warp-owned
//            physical working set, K = 5 (Jacobi) or 11 (fixing) partials;
//            optional in-place compaction of the survivors        40 B/elem
//            (+40 B per survivor written)
//   (rare)   nearest-breakpoint pass (newton.py:129-162)          40 B/elem
//   final    x = clip(t(lambda*), l, u) with fixed variables at their bound
//            (newton.py:232-242, fix_variables x[newly] = bound)  48 B/elem
//
// Between passes the last CTA to arrive reduces the per-CTA partials in a
// fixed order and runs the Newton state machine below on one thread; the
// other CTAs wait on a generation counter.  Variable fixing is *logical*
// and stateless: an element is fixed at its lower bound iff
// t(fix_hi) <= l, where fix_hi is the multiplier of the latest lower-fixing
// iteration (the bracket only shrinks and rounded t is monotone in lambda,
// so this reproduces fix_variables' accumulated sets exactly); compaction
// is a purely physical byte saving decided by the master from counts.
#pragma once
#include "cqk_device.cuh"

namespace cqk {

enum Phase : int32_t {
  PH_LAMBDA0 = 0,
  PH_SCAN = 1,
  PH_BP = 2,
  PH_FINAL = 3,
  PH_DONE = 4,
  PH_COPY = 5,   // simplex/l1: x = y (inside the l1 ball)
  PH_SNAP = 6,   // simplex: max(-y[free]) snap (simplex.py:276-281)
  PH_SAMPLE = 7, // fused start: lambda0 estimated from sample tiles
  PH_FUSED = 8,  // fused start: lambda0 sums + validate + the first scan's aggregates
  PH_GUESS = 9,  // fused start: phi at the estimate over the kept sample tiles (direction guess)
};

enum Status : int32_t {
  ST_RUNNING = 100,
  ST_SOLVED = 0,
  ST_INFEASIBLE = 1,
  ST_DOMAIN = -1,
  ST_MAXITER = -2,
  ST_CONTRACT = -3,
  ST_TIMEOUT = -7,
};

enum Variant : int32_t { V_SOLVE = 0, V_JACOBI = 1, V_PAR = 2 };

// What every CTA needs to run the next pass (written by the master only).
struct Cmd {
  double lam;     // scan point; final multiplier in PH_FINAL
  double fix_hi;  // lower-fixed iff t(fix_hi) <= l   (+inf: none yet)
  double fix_lo;  // upper-fixed iff t(fix_lo) >= u   (-inf: none yet)
  double edge;    // breakpoint-search edge (PH_BP)
  int32_t phase;
  int32_t compact;  // this scan writes the survivors into scratch
  int32_t right;    // PH_BP direction
  int32_t check_lu; // this (first) scan also validates l and u
  int32_t live_lo;  // a lower-fixed element may still be physically present
  int32_t live_hi;  // ... an upper-fixed one
  int32_t hist;     // simplex: this scan also histograms t > 0 (start "auto")
  int32_t side;     // this scan runs over the fused pass's side list (plus its aggregates)
  int32_t guess;    // fused start: the fixing direction (+1 lower, -1 upper) expected at
                    // lambda0 -- the fused pass then also writes the elements it would keep
  int32_t adopt;    // after the side scan: the direction taken at lambda0 when it is the
                    // guessed one -- the survivors become the working set; 0 none
  int32_t sparse;   // simplex capture start adopted: the final pass writes signed zeros and
                    // scatters the captured elements' x (cqk_tma_spx.cuh spx_sparse_final)
  int32_t capture;  // simplex, first scan from an upper-bound start: keep (compact) only
                    // w > -fix_hi, the possible support; the kept count comes back in slot 3
};

// Master-side solver state (SolveState, newton.py:70-90, plus counters).
struct CqkState {
  Cmd cmd;
  double lo, hi, phi_lo, phi_hi;
  double r_res, r_orig, fixed_abs, tau;
  double lam0, compact_ratio;
  double fhi_phys, flo_phys;  // fixing multipliers the working set was last compacted at
  int64_t fixed_count, fixed_removed, iterations, phi_evals, max_iter;
  int64_t n, phys_count, pending_phys;  // n: global size; phys_count: this rank
  int64_t fixed_local;                  // logically fixed elements of this rank
  int64_t elems_scan, elems_written, elems_bp;  // byte-model counters (this rank)
  int64_t domain_index;
  double vidx[10];  // first offending index per validate() check (pass 0 / first scan)
  int32_t has_plo, has_phi, fixing, variant, status, has_xbar, check, domain_field;
  int32_t trace_len, trace_cap, lam0_given, err;  // err: barrier-timeout flag at the final write
  // fused start (PH_SAMPLE -> PH_FUSED -> side scan): the first scan's
  // contributions of every element whose status is fixed on the interval
  // [cmd.lam - cmd.edge, cmd.lam + cmd.edge] around the estimated lambda0
  int32_t fused, fused_guess;  // fused start; with the direction guess (fixing solves)
  double fused_width;       // relative half-width of the classification interval
  double agg[11];           // scan slots 0..10 of those elements at lambda0 (all ranks)
  double agg_lo_loc, agg_hi_loc;  // their lower / upper at-bound counts on this rank
  int64_t side_local;       // elements in this rank's side list
  int64_t elems_sample;     // sample elements read (24 B each)
  int64_t surv_local;       // elements the fused pass wrote as guessed survivors (this rank)
  double rem_plus, rem_minus;          // elements the +1 / -1 guessing CTAs left out (all ranks)
  double rem_plus_loc, rem_minus_loc;  // ... of this rank
  double compact_ratio_adopt;          // compact_ratio once the survivors are adopted
};

template <typename T>
struct CqkParams {
  const T *d, *a, *b, *l, *u, *xbar;
  T *sd, *sa, *sb, *sl, *su;  // compaction scratch (n each) or null
  T *vd, *va, *vb, *vl, *vu;  // fused start: the side-list scratch (n each) or null
  T* x;                       // output or null
  double* trace;              // 4 doubles per phi evaluation
  int64_t n;                  // elements of this rank's shard
  int64_t offset;             // global index of the shard's first element
  double r;
  CqkState* st;               // device: the master's command broadcast (st->cmd)
  double* partials;           // [gridDim.x][kMaxK]
  GridSync sync;
  Exchange ex;                // cross-GPU partial exchange (world 1: none)
  CqkState* out;              // mapped host memory: the final state for the host
  CqkState init;              // the host-initialised state, by value (no H2D copy)
  GridAR ar;                  // single-GPU masterless grid step (rows null: master + release)
};

// ------------------------------------------------------------ master logic
// Everything below runs on thread 0 of the master CTA only.

DEVI void m_finish(CqkState& s, double lam) {
  s.status = ST_SOLVED;
  s.cmd.lam = lam;
  s.cmd.phase = PH_FINAL;
  s.cmd.compact = 0;
}

DEVI void m_stop(CqkState& s, int32_t status) {
  s.status = status;
  s.cmd.phase = PH_DONE;
  s.cmd.compact = 0;
}

// newton.py:106-121 secant_step; false on ContractViolation
DEVI bool m_secant(const CqkState& s, double& out) {
  const double lo = s.lo, hi = s.hi, plo = s.phi_lo, phi = s.phi_hi, r = s.r_res;
  if (!(lo < hi) || !(plo < r && r < phi)) return false;
  double lam = lo + (r - plo) * (hi - lo) / (phi - plo);
  if (!(lo < lam && lam < hi)) lam = lo + 0.5 * (hi - lo);
  out = lam;
  return true;
}

// newton.py:328-336 (exact repeat, bracket width, advance) + compaction policy
DEVI void m_post_step(CqkState& s, double next) {
  const double lam = s.cmd.lam;
  if (next == lam) { m_finish(s, lam); return; }
  if (isfinite(s.lo) && isfinite(s.hi)) {
    const double w = s.hi - s.lo;
    if (w < s.tau * fmax(fabs(s.hi), fabs(s.lo))) { m_finish(s, next); return; }
  }
  s.cmd.lam = next;
  s.iterations += 1;
  if (s.iterations > s.max_iter) { m_stop(s, ST_MAXITER); return; }
  s.cmd.phase = PH_SCAN;
  s.cmd.compact = 0;
  // The fixed tests are needed only while some element fixed at the current
  // multipliers can still be physically present: the last compaction (if
  // any) removed everything fixed at fhi_phys / flo_phys.
  s.cmd.live_lo = s.fixing && s.cmd.fix_hi != s.fhi_phys;
  s.cmd.live_hi = s.fixing && s.cmd.fix_lo != s.flo_phys;
  if (s.fixing) {  // a purely local (per-rank) byte decision
    const int64_t present = s.fixed_local - s.fixed_removed;
    if (present > 0 && (double)present >= s.compact_ratio * (double)s.phys_count) {
      s.cmd.compact = 1;
      s.pending_phys = s.phys_count - present;
    }
  }
}

DEVI void m_secant_or_fail(CqkState& s) {
  double nx;
  if (m_secant(s, nx)) m_post_step(s, nx);
  else m_stop(s, ST_CONTRACT);
}

// tot: 0 value, 1 abs_bx, 2 core, 3 tie_lo, 4 tie_hi, 5..7 lower-fix
// (sum, abs, count), 8..10 upper-fix (sum, abs, count) -- summed over all
// ranks; loc: the same vector of this rank alone (local bookkeeping only).
DEVI void m_after_scan(CqkState& s, const double* tot, const double* loc, double* trace) {
  s.phi_evals += 1;
  const bool side_scan = s.cmd.side != 0;
  s.cmd.adopt = 0;
  if (side_scan) {  // the fused pass read every element; this scan only the side list
    s.elems_scan += s.side_local;
    s.cmd.side = 0;
  } else {
    s.elems_scan += s.phys_count;
  }
  if (s.cmd.compact) {
    s.elems_written += s.pending_phys;
    s.fixed_removed += s.phys_count - s.pending_phys;
    s.phys_count = s.pending_phys;
    s.cmd.compact = 0;
    s.fhi_phys = s.cmd.fix_hi;  // everything fixed at these multipliers is gone
    s.flo_phys = s.cmd.fix_lo;
  }
  const double lam = s.cmd.lam;
  const double value = tot[0], abs_bx = tot[1];
  const double dplus = tot[2] + tot[3], dminus = tot[2] + tot[4];
  if (trace && s.trace_len < s.trace_cap) {
    double* row = trace + 4 * s.trace_len++;
    row[0] = lam; row[1] = value; row[2] = dminus; row[3] = dplus;
  }
  const double diff = value - s.r_res;
  const double scale = abs_bx + s.fixed_abs + fabs(s.r_orig);
  if (fabs(diff) < s.tau * scale) { m_finish(s, lam); return; }  // criterion 1
  if (diff < 0) { s.lo = lam; s.phi_lo = value; s.has_plo = 1; }
  else { s.hi = lam; s.phi_hi = value; s.has_phi = 1; }
  if (s.fixing) {
    // newton.py:165-206 (phi > r fixes lower, phi < r upper); par_solve_cqk
    // picks the direction by the sign of diff (parallel.py:235-236).
    int dir;
    if (s.variant == V_PAR) dir = diff > 0 ? 1 : -1;
    else {
      const double rr = value - diff;
      dir = value > rr ? 1 : (value < rr ? -1 : 0);
    }
    if (dir != 0) {
      const double total = dir > 0 ? tot[5] : tot[8];
      const double tabs = dir > 0 ? tot[6] : tot[9];
      const int64_t cnt = (int64_t)(dir > 0 ? tot[7] : tot[10]);
      if (cnt > 0) {
        s.r_res -= total;
        s.fixed_abs += tabs;
        s.fixed_count += cnt;
        s.fixed_local += (int64_t)(dir > 0 ? loc[7] : loc[10]);
        if (s.has_plo) s.phi_lo -= total;
        if (s.has_phi) s.phi_hi -= total;
        if (dir > 0) s.cmd.fix_hi = lam;
        else s.cmd.fix_lo = lam;
      }
    }
    // fused start: with the guess g the fused pass left every element it
    // classified as fixed in that direction (t < l on the whole interval for
    // +1) out of the survivor lists; if g is the direction just taken, those
    // are all fixed now and the survivors are the working set.
    // Fixed-but-present elements (side-list ones with t == l, ...) stay
    // under the live fixed tests (fhi_phys unchanged).
    if (side_scan && s.cmd.guess == dir && dir != 0 && (dir > 0 ? s.rem_plus : s.rem_minus) > 0) {
      const int64_t rem = (int64_t)(dir > 0 ? s.rem_plus_loc : s.rem_minus_loc);
      s.fixed_removed += rem;
      s.phys_count -= rem;
      s.cmd.adopt = dir;
      s.compact_ratio = s.compact_ratio_adopt;
    }
  }
  s.cmd.guess = 0;
  if (diff < 0) {
    if (dplus > 0) {
      const double step = -diff / dplus;
      if (step < s.tau) { m_finish(s, lam + step); return; }  // criterion 2
      const double tilde = lam + step;
      if (tilde < s.hi) m_post_step(s, tilde);
      else m_secant_or_fail(s);
    } else {
      s.cmd.phase = PH_BP; s.cmd.right = 1; s.cmd.edge = s.lo;
    }
  } else {
    if (dminus > 0) {
      const double step = -diff / dminus;
      if (-step < s.tau) { m_finish(s, lam + step); return; }
      const double tilde = lam + step;
      if (tilde > s.lo) m_post_step(s, tilde);
      else m_secant_or_fail(s);
    } else {
      s.cmd.phase = PH_BP; s.cmd.right = 0; s.cmd.edge = s.hi;
    }
  }
}

// newton.py:280-298 / 312-326 after the breakpoint search; tot: 0 best, 1 found
DEVI void m_after_bp(CqkState& s, const double* tot) {
  s.elems_bp += s.phys_count;
  const bool found = tot[1] > 0;
  const double bp = tot[0];
  if (s.cmd.right) {
    if (found && bp < s.hi) m_post_step(s, bp);
    else if (s.has_phi) m_secant_or_fail(s);
    else m_stop(s, ST_INFEASIBLE);
  } else {
    if (found && bp > s.lo) m_post_step(s, bp);
    else if (s.has_plo) m_secant_or_fail(s);
    else m_stop(s, ST_INFEASIBLE);
  }
}

// tot: 0 s_all, 1 q_all, 2 s_J, 3 q_J, 4 |J|, 5..14 first offending index of
// the ten validate() checks in the reference's order (core.py:135-165).
constexpr int kValidateSlot = 5;
// The checks in the reference's order: d,a,b finite; l,u NaN; r finite;
// d>0; b>0; l<=u; l!=+inf; u!=-inf.  Classes c0 <= c < c1 are decided.
DEVI bool m_validate(CqkState& s, int c0, int c1) {
  const int32_t field_of[10] = {0, 1, 2, 3, 4, 0, 2, 6, 3, 4};
  for (int c = c0; c < c1; ++c) {
    if (c == 5 && !isfinite(s.r_orig)) {
      s.domain_field = 5;
      s.domain_index = -1;
      m_stop(s, ST_DOMAIN);
      return false;
    }
    if (s.vidx[c] < (double)s.n) {
      s.domain_field = field_of[c];
      s.domain_index = (int64_t)s.vidx[c];
      m_stop(s, ST_DOMAIN);
      return false;
    }
  }
  return true;
}

// pass 0 checked d, a, b (and l, u only when xbar made it read them); the
// l / u checks otherwise ride on the first phi scan, which reads l and u
// anyway -- the verdict (the first failing check in the reference's order)
// is identical, 16 B/element cheaper.
DEVI void m_after_lambda0(CqkState& s, const double* tot) {
  if (s.check) {
    for (int c = 0; c < 10; ++c) s.vidx[c] = tot[kValidateSlot + c];
    if (s.has_xbar) {
      if (!m_validate(s, 0, 10)) return;
    } else {
      if (!m_validate(s, 0, 3)) return;  // d, a, b finiteness precede everything
      s.cmd.check_lu = 1;
    }
  }
  if (!s.lam0_given) {
    double lam;
    if (s.has_xbar && tot[4] > 0) lam = (s.r_orig - tot[2]) / tot[3];
    else lam = (s.r_orig - tot[0]) / tot[1];
    s.lam0 = lam;
    s.cmd.lam = lam;
  }
  s.cmd.phase = PH_SCAN;
}

// Fused start.  The sample pass: tot 0 sum b a/d, 1 sum b^2/d, 2 elements
// over the sample tiles -> the estimated lambda0 and the half-width of the
// interval the fused pass classifies against.  With the direction guess
// (fixing solves) the sample tiles carry all five arrays (40 B per sampled
// element) and stay in shared memory for the guess epoch (m_after_guess).
DEVI void m_after_sample(CqkState& s, const double* tot, double local_count) {
  const bool guess = s.fixing && s.fused_guess;
  if (guess) s.elems_scan += (int64_t)local_count;
  else s.elems_sample += (int64_t)local_count;
  const double scale = (double)s.n / fmax(tot[2], 1.0);
  const double est = (s.r_orig - tot[0] * scale) / (tot[1] * scale);
  s.cmd.lam = est;
  // relative half-width (default 2e-3; sampled estimates land within ~5e-4 of
  // lambda0 on the generator families)
  s.cmd.edge = isfinite(est) ? s.fused_width * fabs(est) : 0.0;
  s.cmd.guess = 0;
  s.cmd.phase = guess ? PH_GUESS : PH_FUSED;
}

// The guess epoch: tot 0 sum b x, 1 sum (b x)^2, 2 elements, 3 sum |b x| at
// the estimate over the kept sample tiles (no memory traffic) -> the sign of
// phi(lambda0) - r, i.e. which bound the first iteration will fix
// (newton.py:165-206), when the sampled estimate is clear of zero by six
// standard errors.  The survivor list pays only if several scans follow it,
// and a small initial residual means a short solve (C2 families:
// |phi(lambda0) - r| / sum|b x| of 1e-3 .. 2e-2 took 3-4 phi evaluations,
// 3e-2 .. 9e-2 took 5-7), so the list is written only above kGuessResid.
// The decision is global: a working set adopted by only some CTAs would leave
// the others streaming their whole tiles (static tile ownership).  A wrong or
// missing guess costs bytes only: the list is then simply not adopted.
constexpr double kGuessResid = 0.025;
DEVI void m_after_guess(CqkState& s, const double* tot) {
  const double m = fmax(tot[2], 1.0), N = (double)s.n;
  const double mean = tot[0] / m;
  const double var = fmax(tot[1] / m - mean * mean, 0.0);
  const double diff = N * mean - s.r_orig, se = N * sqrt(var / m), scale = N * tot[3] / m;
  const bool clear = fabs(diff) > 6.0 * se && fabs(diff) > kGuessResid * scale && isfinite(diff);
  s.cmd.guess = clear ? (diff > 0 ? 1 : -1) : 0;
  if (s.fused_guess >= 2) s.cmd.guess = s.fused_guess == 2 ? 1 : -1;  // forced (tests)
  s.cmd.phase = PH_FUSED;
}

// The fused pass: tot 0 s_all, 1 q_all (the lambda0 sums, same per-element
// terms and order as pass 0), 2 the first failing validate() check as
// class * 2^40 + index (min), 3..5 lower at-bound (sum bl, sum |bl|, count),
// 6..8 upper at-bound, 9 / 10 interior with t >= 0 (sum b^2/d, sum b a/d),
// 11 / 12 elements left out of the survivor lists by the CTAs guessing +1
// (their below elements) / -1 (above), 13 side-list elements, 14 survivors
// written.  loc: this rank's vector.
constexpr int kFusedK = 15;
constexpr double kVKey = 1099511627776.0;  // 2^40
DEVI void m_after_fused(CqkState& s, const double* tot, const double* loc) {
  s.elems_scan += s.phys_count;  // 40 B per element: d, a, b, l, u
  s.side_local = (int64_t)loc[13];
  s.surv_local = (int64_t)loc[14];
  s.elems_written += s.side_local + s.surv_local;  // side list + survivors (40 B per element)
  if (s.check) {
    for (int c = 0; c < 10; ++c) s.vidx[c] = (double)s.n;
    if (tot[2] < HUGE_VAL) {
      const double c = floor(tot[2] / kVKey);
      s.vidx[(int)c] = tot[2] - c * kVKey;
    }
    if (!m_validate(s, 0, 10)) return;
  }
  const double lam = (s.r_orig - tot[0]) / tot[1];  // m_after_lambda0's formula
  s.lam0 = lam;
  const double ia = s.cmd.lam - s.cmd.edge, ib = s.cmd.lam + s.cmd.edge;
  s.cmd.lam = lam;
  s.cmd.phase = PH_SCAN;
  s.cmd.check_lu = 0;
  s.cmd.edge = 0.0;
  s.rem_plus = tot[11];
  s.rem_minus = tot[12];
  s.rem_plus_loc = loc[11];
  s.rem_minus_loc = loc[12];
  if (ia <= lam && lam <= ib) {  // the classification holds at lambda0: scan the side list only
    const double pos = lam * tot[9] + tot[10];
    s.agg[0] = tot[3] + tot[6] + pos;
    s.agg[1] = tot[4] + tot[7] + pos;
    s.agg[2] = tot[9];
    s.agg[3] = s.agg[4] = 0.0;  // no exact tie outside the side list
    for (int k = 0; k < 3; ++k) {
      s.agg[5 + k] = tot[3 + k];
      s.agg[8 + k] = tot[6 + k];
    }
    s.agg_lo_loc = loc[5];
    s.agg_hi_loc = loc[8];
    s.cmd.side = 1;
  } else {
    s.cmd.side = 0;  // a full first scan (the side list is dropped)
    s.cmd.guess = 0;  // and the survivors, classified on the wrong interval
  }
}

// the side scan's totals plus the aggregates (glob: all ranks, loc: this rank)
DEVI void m_add_aggregates(const CqkState& s, double* glob, double* loc) {
  for (int k = 0; k < 11; ++k) glob[k] += s.agg[k];
  loc[7] += s.agg_lo_loc;
  loc[10] += s.agg_hi_loc;
}

// ------------------------------------------------------------ element ops
// core.py:195-211 for one element; returns false if the element is already
// (logically) fixed and therefore not part of the active set.
// chk_lo / chk_hi: a lower / upper fixing multiplier exists (finite), so
// the stateless fixed test is needed at all (never divide by infinities).
template <typename T, bool FIX>
DEVI bool elem_scan(T d, T a, T b, T l, T u, T lam, T fhi, T flo, bool chk_lo, bool chk_hi,
                    double (&acc)[kMaxK]) {
  const T yd = rcp_div(d);  // one reciprocal serves t, t(fix) and w
  const T t = t_of_y(d, a, b, lam, yd);
  const bool alo = t <= l, ahi = t >= u;
  if (FIX) {
    if (chk_lo && alo && t_of_y(d, a, b, fhi, yd) <= l) return false;
    if (chk_hi && ahi && t_of_y(d, a, b, flo, yd) >= u) return false;
  }
  const T x = clip(t, l, u);
  const T bx = mul_rn(b, x);
  const double bxd = (double)bx;
  acc[0] += bxd;
  acc[1] += fabs(bxd);
  const bool interior = !(alo || ahi);
  const bool tlo = alo && t == l && l < u;
  const bool thi = ahi && t == u && l < u;
  if (interior || tlo || thi) {
    const double w = (double)w_of(b, d, yd);
    if (interior) acc[2] += w;
    else if (tlo) acc[3] += w;
    else acc[4] += w;
  }
  if (FIX) {
    if (alo) { acc[5] += bxd; acc[6] += fabs(bxd); acc[7] += 1.0; }
    if (ahi) { acc[8] += bxd; acc[9] += fabs(bxd); acc[10] += 1.0; }
  }
  return true;
}

// newton.py:129-162 for one element (lower bound first, then upper)
template <typename T>
DEVI void elem_bp(T d, T a, T b, T l, T u, double edge, bool right, double& best, double& found) {
  const T bds[2] = {l, u};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const T bd = bds[s];
    if (!isfinite((double)bd)) continue;
    const double bp = (double)div_rn(sub_rn(mul_rn(d, bd), a), b);
    if (right ? bp > edge : bp < edge) {
      best = right ? fmin(best, bp) : fmax(best, bp);
      found += 1.0;
    }
  }
}

// final x for one element: clip(t(lam*)) except variables fixed earlier,
// which keep their bound (fix_variables writes x[newly] = bound).
template <typename T, bool FIX>
DEVI T elem_final(T d, T a, T b, T l, T u, T lam, T fhi, T flo, bool chk_lo, bool chk_hi) {
  const T yd = rcp_div(d);
  T x = clip(t_of_y(d, a, b, lam, yd), l, u);
  if (FIX) {
    if (chk_lo && t_of_y(d, a, b, fhi, yd) <= l) x = l;
    else if (chk_hi && t_of_y(d, a, b, flo, yd) >= u) x = u;
  }
  return x;
}

}  // namespace cqk

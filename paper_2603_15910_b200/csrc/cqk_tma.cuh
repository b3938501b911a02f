// cqk_tma.cuh -- TMA-pipelined persistent CQK solve (sm_100a, fp64).
//
// Same single-launch solve as cqk_solve_kernel (the Newton state machine of
// cqk_solver.cuh, replayed on CTA 0's thread 0), with a Blackwell streaming
// engine underneath every pass:
//
//   * tiles of kTileC elements; CTA c owns tiles c, c+G, c+2G, ... so at any
//     moment the whole grid streams one contiguous window of every array;
//   * one producer warp per CTA (one elected lane) keeps kStagesC tiles of
//     all streamed arrays in flight into shared memory with 1-D bulk TMA
//     copies (cp.async.bulk ... mbarrier::complete_tx) -- ~160 KB in flight
//     per SM without spending registers on it;
//   * kConsW consumer warps evaluate the element math out of shared memory
//     and release each stage with one mbarrier arrive per warp;
//   * compaction writes the survivors of CTA c densely into CTA c's own tile
//     slots of the scratch arrays (slot q = tile c + qG), so later passes
//     stream the same tile layout, from the front of scratch, with the same
//     producer; a CTA only ever rewrites slots it has already fully loaded
//     (in place is safe) and a proxy fence orders those generic stores before
//     the next pass's bulk loads.
//
// Per-element arithmetic (elem_scan / elem_bp / elem_final), the fixed-order
// reductions and the grid step are those of the warp-segment kernel, so the
// decisions, counters and tolerances are unchanged; only the summation order
// (and hence rounding-level bits) differs between the two engines.
#pragma once
#include "cqk_kernels.cuh"

namespace cqk {

#ifndef CQK_TMA_TILE
#define CQK_TMA_TILE 960
#endif
#ifndef CQK_TMA_STAGES
#define CQK_TMA_STAGES 4
#endif
#ifndef CQK_TMA_CONSW
#define CQK_TMA_CONSW 15
#endif
// Switches (CQK_TMA_FLAGS, default 12): bit 0 disables the next-pass
// speculation across the grid step; bit 2 issues it after the masterless
// combine instead of during the arrival wait (its HBM reads then do not delay
// the partial-row loads); bit 3 speculates 2 (CQK) / 3 (simplex) tiles instead
// of a full pipeline.  Measured (A/B, one box): bits 2+3 -2% on C2 and C1,
// neutral at n = 1e8.
__constant__ int c_tma_flags;
#define kSpecDepthC ((c_tma_flags & 8) ? 2 : kStagesC)  // next-pass tiles speculated (CQK)

constexpr int kTileC = CQK_TMA_TILE;      // elements per array per tile
constexpr int kStagesC = CQK_TMA_STAGES;
constexpr int kArrMaxC = 6;               // d, a, b, l, u, xbar
constexpr int kConsW = CQK_TMA_CONSW;     // consumer warps
constexpr int kConsT = 32 * kConsW;
constexpr int kTmaThreads = kConsT + 32;  // + one producer warp
constexpr int kStageElemsC = kArrMaxC * kTileC;
constexpr size_t kSmemC = (size_t)kStagesC * kStageElemsC * sizeof(double);
constexpr int kEptC = kTileC / kConsT;    // elements per consumer thread per tile
constexpr int kVpt = kEptC / 2;           // double2 vectors per thread per array
static_assert(kEptC % 2 == 0 && kEptC * kConsT == kTileC, "tile must split into double2 per thread");

DEVI void mbar_init_count(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
DEVI void mbar_arrive1(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Shared-window (u32) forms: the addresses are converted once per kernel.
__constant__ int c_tma_flags_w;  // bit 1 of CQK_TMA_FLAGS: spin with test_wait
DEVI void mbar_wait_s(unsigned bar, unsigned phase) {
  if (c_tma_flags_w & 2) {
    asm volatile(
        "{\n.reg .pred p;\nTWAIT_%=:\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TWAIT_%=;\n}" ::"r"(bar), "r"(phase) : "memory");
    return;
  }
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(bar), "r"(phase) : "memory");
}
DEVI void mbar_arrive_s(unsigned bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
DEVI void mbar_expect_tx_s(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
DEVI void tma_load_1d_s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
DEVI void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
DEVI void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kConsT) : "memory"); }

// Tile / slot geometry.  Every tile of kTileC elements is split into kConsW
// warp sub-segments of kSeg = 32 * kEptC elements; lane l of warp w owns the
// sub-segment elements 64u + 2l + v (u < kVpt, v < 2), i.e. conflict-free
// 16-byte shared loads.  Original layout: tile t covers [t*T, min((t+1)*T, n)).
// Scratch layout: slot q of CTA c is tile index c + q*G, and warp w's
// survivors fill sub-segment w of the CTA's slots 0, 1, ... densely -- so
// compaction needs no CTA-wide prefix (no barrier), stays deterministic, and a
// warp only ever rewrites sub-segments it has already consumed.
constexpr int kSeg = 32 * kEptC;
static_assert(kSeg * kConsW == kTileC, "warp sub-segments tile the tile");

DEVI int e_loc(int lane, int j) { return 64 * (j >> 1) + 2 * lane + (j & 1); }

// Tiles (original arrays, nslots < 0: tile t = c + qG covers
// [t*T, min((t+1)*T, n))) or the nslots scratch slots of this CTA.
struct TileWalk {
  int64_t n, ntiles;
  int nslots;
};

// Streamed array set, passed by value so the pointers live in registers.
struct Src {
  const double* p[kArrMaxC];
};

struct TPipe {
  double* buf;
  unsigned full, empty;  // shared-window addresses of the mbarrier arrays (8 B each)
  unsigned pc;  // tiles through the pipeline since kernel start (same on both sides)
};

// Producer (one lane): NA arrays of every tile of the walk, 16-byte granular
// (the odd last element of an odd-length array is read by its consumer
// straight from global memory).
// Pipeline geometry: ST stages of STRIDE elements (NA arrays of kTileC each).
// The 5/6-array passes use kStagesC stages of kArrMaxC arrays; the 3-array
// lambda0 pass re-cuts the same shared memory into twice as many stages (its
// own mbarriers and counter), keeping the same bytes in flight.
constexpr int kStages3 = kStagesC * 2;
constexpr int kStride3 = 3 * kTileC;

template <int NA, int ST = kStagesC, int STRIDE = kStageElemsC, int TT = kTileC>
DEVI int produce(const Src src, const TileWalk& tw, TPipe& pp, int skip = 0, int maxn = 1 << 30) {
  const int64_t step = (int64_t)gridDim.x * TT;
  const int64_t end = tw.nslots < 0 ? tw.n : ((int64_t)blockIdx.x + (int64_t)tw.nslots * gridDim.x) * TT;
  int s = pp.pc % ST;
  unsigned ph = ((pp.pc / ST) & 1) ^ 1;  // parity of the previous use of stage s
  bool first_round = pp.pc < (unsigned)ST;
  int issued = 0;
  for (int64_t base = ((int64_t)blockIdx.x + (int64_t)skip * gridDim.x) * TT; base < end && issued < maxn;
       base += step) {
    if (!first_round) mbar_wait_s(pp.empty + 8 * s, ph);
    const int64_t left = tw.n - base;
    const int cnt = tw.nslots < 0 && left < TT ? (int)left : TT;
    const unsigned bytes = ((unsigned)cnt * 8u) & ~15u;
    const unsigned fb = pp.full + 8 * s;
    mbar_expect_tx_s(fb, NA * bytes);
    if (bytes) {
      const unsigned dst = smem_u32(pp.buf) + (unsigned)(s * STRIDE) * 8u;
#pragma unroll
      for (int k = 0; k < NA; ++k) tma_load_1d_s(dst + k * TT * 8u, src.p[k] + base, bytes, fb);
    }
    ++pp.pc;
    ++issued;
    if (++s == ST) { s = 0; ph ^= 1; first_round = false; }
  }
  return issued;
}

// Consumers: wait for and release n issued tiles without using them (a
// speculative prefetch the next phase did not want).
template <int ST = kStagesC>
DEVI void drain(TPipe& pp, int n) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < n; ++i) {
    const int s = pp.pc % ST;
    mbar_wait_s(pp.full + 8 * s, (pp.pc / ST) & 1);
    __syncwarp();
    if (lane == 0) mbar_arrive_s(pp.empty + 8 * s);
    ++pp.pc;
  }
}

// What a consumer warp sees of one tile: its sub-segment of every array in
// shared memory (sm + k*T), the matching global sub-segment (base of the
// warp's elements) and how many of its kSeg elements are valid.
struct WTile {
  const double* sm;   // stage + kSeg * warp
  int64_t gbase;      // element index of the sub-segment's first element
  int wcnt;           // valid elements of this warp's sub-segment (0..kSeg)
  bool patch;         // odd original tile: element wcnt-1 is not in the stage
  int q;              // slot / tile ordinal of this CTA in the pass
};

// Consumer warps: body(WTile) per tile, then release the stage.
// m_w >= 0: scratch walk with this warp's element count m_w.
template <int ST = kStagesC, int STRIDE = kStageElemsC, int TT = kTileC, typename Body>
DEVI void consume(const TileWalk& tw, TPipe& pp, int64_t m_w, Body&& body) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kSeg = TT / kConsW;
  const int64_t step = (int64_t)gridDim.x * TT;
  const bool scratch = tw.nslots >= 0;
  const int64_t end = scratch ? ((int64_t)blockIdx.x + (int64_t)tw.nslots * gridDim.x) * TT : tw.n;
  int s = pp.pc % ST;
  unsigned ph = (pp.pc / ST) & 1;
  // valid elements of this warp's sub-segment still ahead (scratch walk)
  int64_t left_w = m_w;
  WTile wt;
  wt.q = 0;
  for (int64_t base = (int64_t)blockIdx.x * TT; base < end; base += step, ++wt.q) {
    wt.sm = pp.buf + (size_t)s * STRIDE + kSeg * warp;
    wt.gbase = base + kSeg * warp;
    const int64_t left = scratch ? left_w : tw.n - wt.gbase;
    wt.wcnt = left <= 0 ? 0 : (left < kSeg ? (int)left : kSeg);
    wt.patch = !scratch && (wt.wcnt & 1) && wt.wcnt < kSeg;
    left_w -= kSeg;
    mbar_wait_s(pp.full + 8 * s, ph);
    if (wt.wcnt > 0) body(wt);
    __syncwarp();
    if (lane == 0) mbar_arrive_s(pp.empty + 8 * s);
    ++pp.pc;
    if (++s == ST) { s = 0; ph ^= 1; }
  }
}

// The final pass with dynamic tile assignment.  It reduces nothing (x is a
// per-element map), so tile order is free, and CTAs that stream faster take
// more tiles: the last CTA of a static final pass finished 40 us (C3) /
// 35 us (simplex 1e8) after the first.  Static prefix: this CTA's tiles
// c + qG, q < D -- exactly the tiles the speculation issues -- then tiles
// G*D + k from a grid-wide counter; a tile index of -1 ends the walk.  The
// producer publishes each dynamic tile's index in s_tix[stage] before the
// stage's arrive (release), consumers read it after the wait (acquire).
template <int NA, int ST, int STRIDE, int TT>
DEVI void produce_final_dyn(const Src src, int64_t n, TPipe& pp, int skip, int D, unsigned* ctr,
                            long long* s_tix) {
  const int64_t G = gridDim.x, ntiles = (n + TT - 1) / TT;
  int s = pp.pc % ST;
  unsigned ph = ((pp.pc / ST) & 1) ^ 1;
  bool first_round = pp.pc < (unsigned)ST;
  auto issue = [&](int64_t t) {
    if (!first_round) mbar_wait_s(pp.empty + 8 * s, ph);
    const unsigned fb = pp.full + 8 * s;
    s_tix[s] = t;
    unsigned bytes = 0;
    if (t >= 0) {
      const int64_t left = n - t * TT;
      bytes = ((unsigned)(left < TT ? left : TT) * 8u) & ~15u;
    }
    mbar_expect_tx_s(fb, NA * bytes);
    if (bytes) {
      const unsigned dst = smem_u32(pp.buf) + (unsigned)(s * STRIDE) * 8u;
#pragma unroll
      for (int k = 0; k < NA; ++k) tma_load_1d_s(dst + k * TT * 8u, src.p[k] + t * TT, bytes, fb);
    }
    ++pp.pc;
    if (++s == ST) { s = 0; ph ^= 1; first_round = false; }
  };
  for (int q = skip; q < D; ++q) {
    const int64_t t = (int64_t)blockIdx.x + q * G;
    if (t >= ntiles) break;
    issue(t);
  }
  for (;;) {
    const int64_t t = G * D + (int64_t)atomicAdd(ctr, 1u);
    if (t >= ntiles) break;
    issue(t);
  }
  issue(-1);
}

template <int ST, int STRIDE, int TT, typename Body>
DEVI void consume_final_dyn(int64_t n, TPipe& pp, int D, const long long* s_tix, Body&& body) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kSegT = TT / kConsW;
  const int64_t G = gridDim.x, ntiles = (n + TT - 1) / TT;
  int s = pp.pc % ST;
  unsigned ph = (pp.pc / ST) & 1;
  bool dyn = false;
  WTile wt;
  wt.q = 0;
  for (int q = 0;; ++q) {
    if (!dyn && (q >= D || (int64_t)blockIdx.x + q * G >= ntiles)) dyn = true;
    mbar_wait_s(pp.full + 8 * s, ph);
    const int64_t t = dyn ? (int64_t)s_tix[s] : (int64_t)blockIdx.x + q * G;
    if (t >= 0) {
      wt.sm = pp.buf + (size_t)s * STRIDE + kSegT * warp;
      wt.gbase = t * TT + kSegT * warp;
      const int64_t left = n - wt.gbase;
      wt.wcnt = left <= 0 ? 0 : (left < kSegT ? (int)left : kSegT);
      wt.patch = (wt.wcnt & 1) && wt.wcnt < kSegT;
      if (wt.wcnt > 0) body(wt);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_s(pp.empty + 8 * s);
    ++pp.pc;
    if (++s == ST) { s = 0; ph ^= 1; }
    if (t < 0) break;
  }
}

template <bool FULL = false, int TT = kTileC>
DEVI void tile_load(const WTile& wt, int k, const double* garr, double (&v)[TT / kConsT],
                    double fill = 0.0) {
  constexpr int EPT = TT / kConsT, VPT = EPT / 2;
  const int lane = threadIdx.x & 31;
  const double* sarr = wt.sm + k * TT;
#pragma unroll
  for (int u = 0; u < VPT; ++u) {
    const double2 w = *reinterpret_cast<const double2*>(sarr + 64 * u + 2 * lane);
    v[2 * u] = w.x;
    v[2 * u + 1] = w.y;
  }
  if (!FULL) {
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if (e_loc(lane, j) >= wt.wcnt) v[j] = fill;  // neutral values beyond the data
    if (wt.patch) {
      const int e = wt.wcnt - 1;  // even: the (v = 0) element of pair e / 2
#pragma unroll
      for (int u = 0; u < VPT; ++u)
        if (64 * u + 2 * lane == e) v[2 * u] = ld_scratch(garr + wt.gbase + e);
    }
  }
}

// ------------------------------------------------------------ fast element math
// The fast division of div_y (cqk_device.cuh) is bit-identical to __ddiv_rn
// whenever numerator and divisor lie in [2^-500, 2^500).  The range test
// runs on the exponent bits with integer ops (no FP64 compares, no branch per
// division); a warp whose tile holds any operand outside it recomputes its
// quotients with __ddiv_rn in one warp-uniform (practically never taken)
// branch -- so the per-element path is straight-line code.
DEVI bool exp_ok(double x) {  // biased exponent in [523, 1522]
  return (((unsigned)__double2hiint(x) & 0x7ff00000u) - (523u << 20)) < (1000u << 20);
}
DEVI double div_fast(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double r = fma(q0, -b, a);
  return fma(y, r, q0);
}

// t, w = b*b/d and the stateless fixed tests (t(fix_hi) <= l, t(fix_lo) >= u,
// cqk_solver.cuh elem_scan) for the kEptC elements of this thread; CLO / CHI
// (warp-uniform, dispatched at compile time): which fixed tests are live.
template <bool CLO, bool CHI>
DEVI void tile_t(const double (&D)[kEptC], const double (&A)[kEptC], const double (&B)[kEptC],
                 const double (&L)[kEptC], const double (&U)[kEptC], double lam, double fhi,
                 double flo, double (&T)[kEptC], double (&W)[kEptC], bool (&FXL)[kEptC],
                 bool (&FXH)[kEptC]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < kEptC; ++j) {
    const double yd = rcp_div(D[j]);
    const double num = add_rn(mul_rn(B[j], lam), A[j]);
    T[j] = div_fast(num, D[j], yd);
    W[j] = (double)(mul_rn(B[j], B[j]) * yd);
    ok = ok && exp_ok(num) && exp_ok(D[j]);
    FXL[j] = FXH[j] = false;
    if (CLO) {
      const double nh = add_rn(mul_rn(B[j], fhi), A[j]);
      FXL[j] = div_fast(nh, D[j], yd) <= L[j];
      ok = ok && exp_ok(nh);
    }
    if (CHI) {
      const double nl = add_rn(mul_rn(B[j], flo), A[j]);
      FXH[j] = div_fast(nl, D[j], yd) >= U[j];
      ok = ok && exp_ok(nl);
    }
  }
  if (!__all_sync(0xffffffffu, ok)) {
#pragma unroll
    for (int j = 0; j < kEptC; ++j) {
      T[j] = div_rn(add_rn(mul_rn(B[j], lam), A[j]), D[j]);
      if (CLO) FXL[j] = div_rn(add_rn(mul_rn(B[j], fhi), A[j]), D[j]) <= L[j];
      if (CHI) FXH[j] = div_rn(add_rn(mul_rn(B[j], flo), A[j]), D[j]) >= U[j];
    }
  }
}

// Compile-time dispatch of the two fixed-test flags.
#define CQK_DISPATCH_FIXED(CLO_RT, CHI_RT, CALL)          \
  do {                                                    \
    if (CLO_RT) {                                         \
      if (CHI_RT) { constexpr bool CLO = true, CHI = true; CALL; }   \
      else { constexpr bool CLO = true, CHI = false; CALL; }         \
    } else {                                              \
      if (CHI_RT) { constexpr bool CLO = false, CHI = true; CALL; }  \
      else { constexpr bool CLO = false, CHI = false; CALL; }        \
    }                                                     \
  } while (0)

// ------------------------------------------------------------ consumer passes
template <bool CHECK, bool XBAR>
DEVI void t_lambda0(const CqkParams<double>& p, const TileWalk& tw, TPipe& pp,
                    double (&acc)[kMaxK]) {
  const int lane = threadIdx.x & 31;
  constexpr int ST = XBAR ? kStagesC : kStages3;
  constexpr int STRIDE = XBAR ? kStageElemsC : kStride3;
  consume<ST, STRIDE>(tw, pp, -1, [&](const WTile& wt) {
    double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC], X[kEptC];
    if (wt.wcnt == kSeg) {
      tile_load<true>(wt, 0, p.d, D);
      tile_load<true>(wt, 1, p.a, A);
      tile_load<true>(wt, 2, p.b, B);
      if (XBAR) {
        tile_load<true>(wt, 3, p.l, L);
        tile_load<true>(wt, 4, p.u, U);
        tile_load<true>(wt, 5, p.xbar, X);
      }
    } else {
      tile_load(wt, 0, p.d, D, 1.0);
      tile_load(wt, 1, p.a, A);
      tile_load(wt, 2, p.b, B, 1.0);
      if (XBAR) {
        tile_load(wt, 3, p.l, L);
        tile_load(wt, 4, p.u, U);
        tile_load(wt, 5, p.xbar, X);
      }
    }
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kEptC; ++j) {
      const bool valid = e_loc(lane, j) < wt.wcnt;
      const double y = rcp_nr(D[j]);
      const double s = mul_rn(B[j], A[j] * y);
      const double q = mul_rn(B[j], B[j] * y);
      if (valid) { acc[0] += s; acc[1] += q; }
      if (XBAR && valid && L[j] < X[j] && X[j] < U[j]) { acc[2] += s; acc[3] += q; acc[4] += 1.0; }
      if (CHECK) {
        bool b_ = !(D[j] > 0.0 && D[j] < HUGE_VAL) || !(fabs(A[j]) < HUGE_VAL) ||
                  !(B[j] > 0.0 && B[j] < HUGE_VAL);
        if (XBAR) b_ = b_ || !(L[j] <= U[j]) || L[j] == HUGE_VAL || U[j] == -HUGE_VAL;
        bad = bad || (valid && b_);
      }
    }
    if (CHECK && __any_sync(0xffffffffu, bad)) {  // rare: locate the first offenders
#pragma unroll
      for (int j = 0; j < kEptC; ++j) {
        const int e = e_loc(lane, j);
        if (e >= wt.wcnt) continue;
        const double gi = (double)(p.offset + wt.gbase + e);
        const double d = D[j], a = A[j], b = B[j];
        if (!isfinite(d)) acc[5] = fmin(acc[5], gi);
        if (!isfinite(a)) acc[6] = fmin(acc[6], gi);
        if (!isfinite(b)) acc[7] = fmin(acc[7], gi);
        if (!(d > 0.0)) acc[10] = fmin(acc[10], gi);
        if (!(b > 0.0)) acc[11] = fmin(acc[11], gi);
        if (XBAR) {
          const double l = L[j], u = U[j];
          if (isnan(l)) acc[8] = fmin(acc[8], gi);
          if (isnan(u)) acc[9] = fmin(acc[9], gi);
          if (!(l <= u)) acc[12] = fmin(acc[12], gi);
          if (l == HUGE_VAL) acc[13] = fmin(acc[13], gi);
          if (u == -HUGE_VAL) acc[14] = fmin(acc[14], gi);
        }
      }
    }
  });
}

// One tile of the phi scan (core.py:182-212 per element, as elem_scan in
// cqk_solver.cuh) for this thread's kEptC elements; keep[j]: the element is
// (logically) active.  Straight-line: predicated accumulation, counts in
// integer registers, the l / u validation on one warp-uniform branch.
template <bool FIX, bool CHK, bool FULL, bool CLO, bool CHI>
DEVI void scan_tile(const CqkParams<double>& p, const WTile& wt, const Src& src, double lam,
                    double fhi, double flo, double (&acc)[kMaxK], int (&nfix)[2],
                    bool (&keep)[kEptC]) {
  const int lane = threadIdx.x & 31;
  double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC];
  tile_load<FULL>(wt, 0, src.p[0], D, 1.0);
  tile_load<FULL>(wt, 1, src.p[1], A);
  tile_load<FULL>(wt, 2, src.p[2], B, 1.0);
  tile_load<FULL>(wt, 3, src.p[3], L);
  tile_load<FULL>(wt, 4, src.p[4], U);
  if (CHK) {  // validate()'s l / u checks ride on the first scan
    bool bad = false;
#pragma unroll
    for (int j = 0; j < kEptC; ++j) {
      const bool valid = FULL || e_loc(lane, j) < wt.wcnt;
      bad = bad || (valid && (!(L[j] <= U[j]) || L[j] == HUGE_VAL || U[j] == -HUGE_VAL));
    }
    if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
      for (int j = 0; j < kEptC; ++j) {
        const int e = e_loc(lane, j);
        if (!FULL && e >= wt.wcnt) continue;
        const double gi = (double)(p.offset + wt.gbase + e);
        const double l = L[j], u = U[j];
        if (isnan(l)) acc[kCheckLuSlot] = fmin(acc[kCheckLuSlot], gi);
        if (isnan(u)) acc[kCheckLuSlot + 1] = fmin(acc[kCheckLuSlot + 1], gi);
        if (!(l <= u)) acc[kCheckLuSlot + 2] = fmin(acc[kCheckLuSlot + 2], gi);
        if (l == HUGE_VAL) acc[kCheckLuSlot + 3] = fmin(acc[kCheckLuSlot + 3], gi);
        if (u == -HUGE_VAL) acc[kCheckLuSlot + 4] = fmin(acc[kCheckLuSlot + 4], gi);
      }
    }
  }
  double T[kEptC], W[kEptC];
  bool FXL[kEptC], FXH[kEptC];
  tile_t<CLO, CHI>(D, A, B, L, U, lam, fhi, flo, T, W, FXL, FXH);
  bool tie_any = false;
#pragma unroll
  for (int j = 0; j < kEptC; ++j) {
    const bool valid = FULL || e_loc(lane, j) < wt.wcnt;
    const double t = T[j], l = L[j], u = U[j];
    const bool alo = t <= l, ahi = t >= u;
    bool fixed = false;
    if (CLO) fixed = fixed || (alo && FXL[j]);
    if (CHI) fixed = fixed || (ahi && FXH[j]);
    const bool kp = valid && !fixed;
    keep[j] = kp;
    const double x = clip(t, l, u);
    const double bx = mul_rn(B[j], x);
    const double bxk = kp ? bx : 0.0;
    acc[0] += bxk;
    acc[1] += fabs(bxk);
    const bool interior = !(alo || ahi);
    acc[2] += (kp && interior) ? W[j] : 0.0;
    // an exact tie t == l or t == u (the one-sided slopes) -- rare
    tie_any = tie_any || (kp && !interior && t == x);
    if (FIX) {
      const bool lo = kp && alo, hi = kp && ahi;
      const double bl = lo ? bx : 0.0, bh = hi ? bx : 0.0;
      acc[5] += bl;
      acc[6] += fabs(bl);
      acc[8] += bh;
      acc[9] += fabs(bh);
      nfix[0] += lo;
      nfix[1] += hi;
    }
  }
  if (__any_sync(0xffffffffu, tie_any)) {
#pragma unroll
    for (int j = 0; j < kEptC; ++j) {
      const double t = T[j], l = L[j], u = U[j];
      const bool lt = l < u;
      if (keep[j] && t <= l && lt && t == l) acc[3] += W[j];
      if (keep[j] && t >= u && lt && t == u) acc[4] += W[j];
    }
  }
}

// phi scan over the walk (m_w >= 0: this warp's scratch count); with
// `compact` every warp appends its survivors to its own scratch
// sub-segments.  Returns this warp's new element count.
template <bool FIX, bool CHK>
DEVI int64_t t_scan(const CqkParams<double>& p, const Cmd& c, const TileWalk& tw, int64_t m_w,
                    const Src src, bool compact, TPipe& pp, double (&acc)[kMaxK]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned ltm = (1u << lane) - 1u;
  const double lam = c.lam, fhi = c.fix_hi, flo = c.fix_lo;
  const bool chk_lo = FIX && c.live_lo, chk_hi = FIX && c.live_hi;
  int nfix[2] = {0, 0};
  int64_t out_m = 0;  // survivors so far: slots [0, q_out) full plus off_out in slot q_out
  int64_t q_out = 0;
  int off_out = 0;
  const int64_t g = gridDim.x;
  consume(tw, pp, m_w, [&](const WTile& wt) {
    bool keep[kEptC];
    if (wt.wcnt == kSeg)
      CQK_DISPATCH_FIXED(chk_lo, chk_hi, (scan_tile<FIX, CHK, true, CLO, CHI>(
                                             p, wt, src, lam, fhi, flo, acc, nfix, keep)));
    else
      CQK_DISPATCH_FIXED(chk_lo, chk_hi, (scan_tile<FIX, CHK, false, CLO, CHI>(
                                             p, wt, src, lam, fhi, flo, acc, nfix, keep)));
    if (FIX && compact) {
      // survivor r of this tile (r < kSeg) lands at sub-segment offset
      // off_out + r: slot q_out or, after one wrap, q_out + 1
      const int64_t b0 = ((int64_t)blockIdx.x + q_out * g) * kTileC + kSeg * warp;
      const int64_t b1 = b0 + g * kTileC;
      // the survivors' values come back from the (still held) stage
      double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC];
      if (wt.wcnt == kSeg) {
        tile_load<true>(wt, 0, src.p[0], D);
        tile_load<true>(wt, 1, src.p[1], A);
        tile_load<true>(wt, 2, src.p[2], B);
        tile_load<true>(wt, 3, src.p[3], L);
        tile_load<true>(wt, 4, src.p[4], U);
      } else {
        tile_load(wt, 0, src.p[0], D);
        tile_load(wt, 1, src.p[1], A);
        tile_load(wt, 2, src.p[2], B);
        tile_load(wt, 3, src.p[3], L);
        tile_load(wt, 4, src.p[4], U);
      }
      int r = off_out;
#pragma unroll
      for (int j = 0; j < kEptC; ++j) {
        const unsigned bal = __ballot_sync(0xffffffffu, keep[j]);
        if (keep[j]) {
          const int o = r + __popc(bal & ltm);
          const int64_t pos = o < kSeg ? b0 + o : b1 + (o - kSeg);
          p.sd[pos] = D[j]; p.sa[pos] = A[j]; p.sb[pos] = B[j]; p.sl[pos] = L[j]; p.su[pos] = U[j];
        }
        r += __popc(bal);
      }
      out_m += r - off_out;
      off_out = r;
      if (off_out >= kSeg) { off_out -= kSeg; ++q_out; }
    }
  });
  if (FIX) { acc[7] += (double)nfix[0]; acc[10] += (double)nfix[1]; }
  if (FIX && compact) fence_proxy_async_global();  // generic stores -> next pass's bulk loads
  return out_m;
}

DEVI void t_bp(const CqkParams<double>& p, const Cmd& c, bool fix, const TileWalk& tw,
               int64_t m_w, const Src src, TPipe& pp, double (&acc)[kMaxK]) {
  const int lane = threadIdx.x & 31;
  const double lam = c.lam, fhi = c.fix_hi, flo = c.fix_lo;
  const bool right = c.right != 0;
  consume(tw, pp, m_w, [&](const WTile& wt) {
    double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC];
    tile_load(wt, 0, src.p[0], D, 1.0);
    tile_load(wt, 1, src.p[1], A);
    tile_load(wt, 2, src.p[2], B, 1.0);
    tile_load(wt, 3, src.p[3], L);
    tile_load(wt, 4, src.p[4], U);
#pragma unroll
    for (int j = 0; j < kEptC; ++j) {
      if (e_loc(lane, j) >= wt.wcnt) continue;
      if (fix) {  // only the logically active set takes part
        const double yd = rcp_div(D[j]);
        const double t = t_of_y(D[j], A[j], B[j], lam, yd);
        if (isfinite(c.fix_hi) && t <= L[j] && t_of_y(D[j], A[j], B[j], fhi, yd) <= L[j]) continue;
        if (isfinite(c.fix_lo) && t >= U[j] && t_of_y(D[j], A[j], B[j], flo, yd) >= U[j]) continue;
      }
      elem_bp<double>(D[j], A[j], B[j], L[j], U[j], c.edge, right, acc[0], acc[1]);
    }
  });
}

template <bool FIX, bool FULL, bool CLO, bool CHI>
DEVI void final_tile(const CqkParams<double>& p, const WTile& wt, double lam, double fhi,
                     double flo) {
  const int lane = threadIdx.x & 31;
  double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC];
  tile_load<FULL>(wt, 0, p.d, D, 1.0);
  tile_load<FULL>(wt, 1, p.a, A);
  tile_load<FULL>(wt, 2, p.b, B, 1.0);
  tile_load<FULL>(wt, 3, p.l, L);
  tile_load<FULL>(wt, 4, p.u, U);
  double T[kEptC], W[kEptC], X[kEptC];
  bool FXL[kEptC], FXH[kEptC];
  tile_t<CLO, CHI>(D, A, B, L, U, lam, fhi, flo, T, W, FXL, FXH);
#pragma unroll
  for (int j = 0; j < kEptC; ++j) {  // elem_final: fixed variables keep their bound
    double x = clip(T[j], L[j], U[j]);
    if (CLO && FXL[j]) x = L[j];
    else if (CHI && FXH[j]) x = U[j];
    X[j] = x;
  }
#pragma unroll
  for (int u = 0; u < kVpt; ++u) {
    const int e = 64 * u + 2 * lane;
    double* xp = p.x + wt.gbase + e;
    if (FULL || e + 1 < wt.wcnt) store_out(reinterpret_cast<double2*>(xp), make_double2(X[2 * u], X[2 * u + 1]));
    else if (e < wt.wcnt) *xp = X[2 * u];
  }
}

template <bool FIX>
DEVI void t_final(const CqkParams<double>& p, const Cmd& c, const TileWalk& tw, TPipe& pp,
                  int D = -1, const long long* s_tix = nullptr) {
  const double lam = c.lam, fhi = c.fix_hi, flo = c.fix_lo;
  // fixed variables need an explicit test only if lam* left the side of the
  // fixing multiplier (the criterion-2 finish(lam + step) edge)
  const bool chk_lo = FIX && c.lam > c.fix_hi, chk_hi = FIX && c.lam < c.fix_lo;
  auto body = [&](const WTile& wt) {
    if (wt.wcnt == kSeg)
      CQK_DISPATCH_FIXED(chk_lo, chk_hi, (final_tile<FIX, true, CLO, CHI>(p, wt, lam, fhi, flo)));
    else
      CQK_DISPATCH_FIXED(chk_lo, chk_hi, (final_tile<FIX, false, CLO, CHI>(p, wt, lam, fhi, flo)));
  };
  if (D >= 0) consume_final_dyn<kStagesC, kStageElemsC, kTileC>(p.n, pp, D, s_tix, body);
  else consume(tw, pp, -1, body);
}

// ------------------------------------------------------------ fused start
// The first two passes of solve_cqk -- lambda0 sums (core.py:237-257, 24 B
// per element) then the first phi scan at lambda0 (40 B) -- become one 40 B
// pass: a sample pass (kSampleTiles tiles per CTA, spread over its walk)
// estimates lambda0; the fused pass computes the exact lambda0 sums (the same
// per-element terms in the same order as pass 0, so lambda0 is bit-identical)
// and classifies every element against the interval I = [est - h, est + h]:
// below (t(I) < l), above (t(I) > u) or strictly interior with a fixed sign
// of t -- their scan contributions at any lambda0 in I are known in closed
// form (b*l, b*u, lambda0 * sum b^2/d + sum b*a/d) -- or ambiguous, appended
// to a side list in scratch (per-warp sub-segments, as compaction does).
// When lambda0 lands in I the first scan reads only the side list and adds
// the aggregates; otherwise it is an ordinary full scan.  Exact ties t == l /
// t == u can only occur in the side list, so the one-sided slopes are exact.
constexpr int kSampleTiles = 4;

// this CTA's q-th sample tile (orig walk ordinal), -1 past the end
DEVI int64_t sample_tile(int64_t ntiles, int k) {
  const int64_t G = gridDim.x, c = blockIdx.x;
  const int64_t Q = c < ntiles ? (ntiles - c + G - 1) / G : 0;  // tiles of this CTA
  if (Q <= 0) return -1;
  const int64_t q = Q >= kSampleTiles ? (int64_t)k * Q / kSampleTiles : k;
  return q < Q ? c + q * G : -1;
}

// NA arrays of this CTA's sample tiles into the ST x STRIDE pipeline
template <int NA = 3, int ST = kStages3, int STRIDE = kStride3>
DEVI void produce_sample(const Src src, int64_t n, int64_t ntiles, TPipe& pp) {
  for (int k = 0; k < kSampleTiles; ++k) {
    const int64_t t = sample_tile(ntiles, k);
    if (t < 0) break;
    const int s = pp.pc % ST;
    const unsigned ph = ((pp.pc / ST) & 1) ^ 1;
    if (pp.pc >= (unsigned)ST) mbar_wait_s(pp.empty + 8 * s, ph);
    const int64_t left = n - t * kTileC;
    const unsigned bytes = ((unsigned)(left < kTileC ? left : kTileC) * 8u) & ~15u;
    const unsigned fb = pp.full + 8 * s;
    mbar_expect_tx_s(fb, NA * bytes);
    if (bytes) {
      const unsigned dst = smem_u32(pp.buf) + (unsigned)(s * STRIDE) * 8u;
#pragma unroll
      for (int a = 0; a < NA; ++a) tma_load_1d_s(dst + a * kTileC * 8u, src.p[a] + t * kTileC, bytes, fb);
    }
    ++pp.pc;
  }
}

// acc 0 sum b a/d, 1 sum b^2/d, 2 elements (t_lambda0's per-element terms).
// KEEP (direction guess): the tiles stay in their stages (no release) for the
// CTA's guess at the start of the fused pass (t_sample_guess).
template <int ST = kStages3, int STRIDE = kStride3, bool KEEP = false>
DEVI void t_sample(const CqkParams<double>& p, int64_t ntiles, TPipe& pp, double (&acc)[kMaxK]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  static_assert(!KEEP || ST >= kSampleTiles, "kept sample tiles must fit the pipeline");
  for (int k = 0; k < kSampleTiles; ++k) {
    const int64_t t = sample_tile(ntiles, k);
    if (t < 0) break;
    const int s = pp.pc % ST;
    WTile wt;
    wt.sm = pp.buf + (size_t)s * STRIDE + kSeg * warp;
    wt.gbase = t * kTileC + kSeg * warp;
    const int64_t left = p.n - wt.gbase;
    wt.wcnt = left <= 0 ? 0 : (left < kSeg ? (int)left : kSeg);
    wt.patch = (wt.wcnt & 1) && wt.wcnt < kSeg;
    wt.q = k;
    mbar_wait_s(pp.full + 8 * s, (pp.pc / ST) & 1);
    if (wt.wcnt > 0) {
      double D[kEptC], A[kEptC], B[kEptC];
      tile_load<false, kTileC>(wt, 0, p.d, D, 1.0);
      tile_load<false, kTileC>(wt, 1, p.a, A);
      tile_load<false, kTileC>(wt, 2, p.b, B, 1.0);
#pragma unroll
      for (int j = 0; j < kEptC; ++j) {
        if (e_loc(lane, j) >= wt.wcnt) continue;
        const double y = rcp_nr(D[j]);
        acc[0] += mul_rn(B[j], A[j] * y);
        acc[1] += mul_rn(B[j], B[j] * y);
        acc[2] += 1.0;
      }
    }
    __syncwarp();
    if (!KEEP && lane == 0) mbar_arrive_s(pp.empty + 8 * s);
    ++pp.pc;
  }
}





DEVI int sample_count(int64_t ntiles) {
  int k = 0;
  while (k < kSampleTiles && sample_tile(ntiles, k) >= 0) ++k;
  return k;
}
DEVI void t_sample_guess(const CqkParams<double>& p, double lam, int64_t ntiles, const TPipe& pp,
                         double (&acc)[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ns = sample_count(ntiles);
  for (int k = 0; k < ns; ++k) {
    const int64_t t = sample_tile(ntiles, k);
    const int s = (pp.pc - ns + k) % kStagesC;
    WTile wt;
    wt.sm = pp.buf + (size_t)s * kStageElemsC + kSeg * warp;
    wt.gbase = t * kTileC + kSeg * warp;
    const int64_t left = p.n - wt.gbase;
    wt.wcnt = left <= 0 ? 0 : (left < kSeg ? (int)left : kSeg);
    wt.patch = (wt.wcnt & 1) && wt.wcnt < kSeg;
    wt.q = k;
    if (wt.wcnt <= 0) continue;
    double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC];
    tile_load(wt, 0, p.d, D, 1.0);
    tile_load(wt, 1, p.a, A);
    tile_load(wt, 2, p.b, B, 1.0);
    tile_load(wt, 3, p.l, L);
    tile_load(wt, 4, p.u, U);
#pragma unroll
    for (int j = 0; j < kEptC; ++j) {
      if (e_loc(lane, j) >= wt.wcnt) continue;
      const double x = clip(div_rn(add_rn(mul_rn(B[j], lam), A[j]), D[j]), L[j], U[j]);
      const double bx = mul_rn(B[j], x);
      acc[0] += bx;
      acc[1] += bx * bx;
      acc[2] += 1.0;
      acc[3] += fabs(bx);
    }
  }
}
DEVI void release_sample(int64_t ntiles, const TPipe& pp) {
  const int ns = sample_count(ntiles);
  __syncwarp();
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < ns; ++k) mbar_arrive_s(pp.empty + 8 * ((pp.pc - ns + k) % kStagesC));
}

// Append the elements with keep[j] of this warp's tile (values from the held
// stage) to the warp's sub-segments of the scratch set dst: slot q_out at
// offset off_out.
DEVI void append_tile(double* const (&dst)[5], const WTile& wt, const Src& src,
                      const bool (&keep)[kEptC], int64_t& q_out, int& off_out, int64_t& out_m) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned ltm = (1u << lane) - 1u;
  const int64_t g = gridDim.x;
  const int64_t b0 = ((int64_t)blockIdx.x + q_out * g) * kTileC + kSeg * warp;
  const int64_t b1 = b0 + g * kTileC;
  double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC];
  if (wt.wcnt == kSeg) {
    tile_load<true>(wt, 0, src.p[0], D);
    tile_load<true>(wt, 1, src.p[1], A);
    tile_load<true>(wt, 2, src.p[2], B);
    tile_load<true>(wt, 3, src.p[3], L);
    tile_load<true>(wt, 4, src.p[4], U);
  } else {
    tile_load(wt, 0, src.p[0], D);
    tile_load(wt, 1, src.p[1], A);
    tile_load(wt, 2, src.p[2], B);
    tile_load(wt, 3, src.p[3], L);
    tile_load(wt, 4, src.p[4], U);
  }
  int r = off_out;
#pragma unroll
  for (int j = 0; j < kEptC; ++j) {
    const unsigned bal = __ballot_sync(0xffffffffu, keep[j]);
    if (keep[j]) {
      const int o = r + __popc(bal & ltm);
      const int64_t pos = o < kSeg ? b0 + o : b1 + (o - kSeg);
      dst[0][pos] = D[j]; dst[1][pos] = A[j]; dst[2][pos] = B[j]; dst[3][pos] = L[j]; dst[4][pos] = U[j];
    }
    r += __popc(bal);
  }
  out_m += r - off_out;
  off_out = r;
  if (off_out >= kSeg) { off_out -= kSeg; ++q_out; }
}

constexpr double kBracketEps = 16.0 * 2.220446049250313e-16;

template <bool CHECK, bool FULL>
DEVI void fused_tile(const CqkParams<double>& p, const WTile& wt, const Src& src, double lam_hat,
                     double h2, int guess, double (&acc)[kMaxK], int& nlo, int& nhi, int& nside,
                     bool (&side)[kEptC], bool& anyside_out, bool (&surv)[kEptC]) {
  const int lane = threadIdx.x & 31;
  double D[kEptC], A[kEptC], B[kEptC], L[kEptC], U[kEptC];
  tile_load<FULL>(wt, 0, src.p[0], D, 1.0);
  tile_load<FULL>(wt, 1, src.p[1], A);
  tile_load<FULL>(wt, 2, src.p[2], B, 1.0);
  tile_load<FULL>(wt, 3, src.p[3], L);
  tile_load<FULL>(wt, 4, src.p[4], U);
    if (CHECK) {  // all ten validate() checks; the first failing one as class * 2^40 + index
      // the common case in predicate logic (no short-circuit branches): 0 < d, b < inf,
      // |a| < inf, l <= u (false for NaN), l < +inf, u > -inf
      bool bad = false;
#pragma unroll
      for (int j = 0; j < kEptC; ++j) {
        const bool good = (D[j] > 0.0) & (D[j] < HUGE_VAL) & (fabs(A[j]) < HUGE_VAL) & (B[j] > 0.0) &
                          (B[j] < HUGE_VAL) & (L[j] <= U[j]) & (L[j] < HUGE_VAL) & (U[j] > -HUGE_VAL);
        bad |= (FULL || e_loc(lane, j) < wt.wcnt) & !good;
      }
      if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
        for (int j = 0; j < kEptC; ++j) {
          const int e = e_loc(lane, j);
          if (e >= wt.wcnt) continue;
          const double gi = (double)(p.offset + wt.gbase + e);
          const double d = D[j], a = A[j], b = B[j], l = L[j], u = U[j];
          int cls = -1;  // validate()'s order (core.py:135-165); 5 is r (host-side)
          if (!isfinite(d)) cls = 0;
          else if (!isfinite(a)) cls = 1;
          else if (!isfinite(b)) cls = 2;
          else if (isnan(l)) cls = 3;
          else if (isnan(u)) cls = 4;
          else if (!(d > 0.0)) cls = 6;
          else if (!(b > 0.0)) cls = 7;
          else if (!(l <= u)) cls = 8;
          else if (l == HUGE_VAL) cls = 9;
          else if (u == -HUGE_VAL) cls = 10;
          if (cls >= 0) acc[2] = fmin(acc[2], (double)(cls > 5 ? cls - 1 : cls) * kVKey + gi);
        }
      }
    }
    // A conservative bracket of the rounded t(lambda) over I: tm = lam^ b/d
    // + a/d (one reciprocal), widened by the interval (hw) and by 16 eps of
    // the magnitudes involved -- far above the few-ulp error of the bracket
    // and of t's own roundings (b*lam, + a, / d).  Misjudging an element only
    // costs a side-list slot, so only the certain verdicts must be certain.
    bool anyside = false;
#pragma unroll
    for (int j = 0; j < kEptC; ++j) {
      const bool valid = FULL || e_loc(lane, j) < wt.wcnt;
      const double yd = rcp_div(D[j]);
      const double by = B[j] * yd, ay = A[j] * yd;  // b/d, a/d
      const double qj = B[j] * by, sj = B[j] * ay;  // the lambda0 terms b^2/d, b a/d
      const double pm = lam_hat * by;
      const double tm = pm + ay;
      const double w2 = h2 * by + kBracketEps * (fabs(pm) + fabs(ay));
      const double tlo = tm - w2, thi = tm + w2;
      const double l = L[j], u = U[j];
      const bool rng = exp_ok(D[j]);  // the reciprocal is accurate here
      const bool below = rng & (thi < l), above = rng & (tlo > u);
      const bool inner = rng & (tlo > l) & (thi < u) & (tlo >= 0.0);  // interior, t >= 0
      const double bl = mul_rn(B[j], l), bu = mul_rn(B[j], u);
      const bool vb = valid & below, va = valid & above, vp = valid & inner;
      acc[0] += valid ? sj : 0.0;
      acc[1] += valid ? qj : 0.0;
      acc[3] += vb ? bl : 0.0;
      acc[4] += vb ? fabs(bl) : 0.0;
      acc[6] += va ? bu : 0.0;
      acc[7] += va ? fabs(bu) : 0.0;
      acc[9] += vp ? qj : 0.0;
      acc[10] += vp ? sj : 0.0;
      nlo += vb;
      nhi += va;
      side[j] = valid & !below & !above & !inner;
      nside += side[j];
      anyside |= side[j];
      surv[j] = valid & !(guess > 0 ? below : above);  // (guess 0: not used)
    }
    anyside_out = anyside;
}

// The fused pass (slots: m_after_fused).  The side list goes to the side
// scratch set; with a direction guess (fixing solves) every element the
// guessed fixing would not drop also goes to the compaction scratch -- the
// working set of the following scans if the side scan confirms the guess.
// Returns this warp's side-list count; *surv_m its survivor count.
template <bool CHECK>
DEVI int64_t t_fused(const CqkParams<double>& p, const Cmd& c, const TileWalk& tw,
                     const Src src, TPipe& pp, double (&acc)[kMaxK], int guess, int64_t* surv_m) {
  // I = [lam^ - h, lam^ + h] as the host-side check sees it; h2 also covers
  // the rounding of the interval ends
  const double lam_hat = c.lam, h2 = c.edge + kBracketEps * fabs(c.lam);
  double* const dside[5] = {p.vd, p.va, p.vb, p.vl, p.vu};
  double* const dsurv[5] = {p.sd, p.sa, p.sb, p.sl, p.su};
  int64_t out_m = 0, q_out = 0, sv_m = 0, q_sv = 0;
  int off_out = 0, off_sv = 0;
  int nlo = 0, nhi = 0, nside = 0;
  consume(tw, pp, -1, [&](const WTile& wt) {
    bool side[kEptC], surv[kEptC], anyside;
    if (wt.wcnt == kSeg)
      fused_tile<CHECK, true>(p, wt, src, lam_hat, h2, guess, acc, nlo, nhi, nside, side, anyside, surv);
    else
      fused_tile<CHECK, false>(p, wt, src, lam_hat, h2, guess, acc, nlo, nhi, nside, side, anyside, surv);
    if (__any_sync(0xffffffffu, anyside)) append_tile(dside, wt, src, side, q_out, off_out, out_m);
    if (guess != 0) append_tile(dsurv, wt, src, surv, q_sv, off_sv, sv_m);
  });
  acc[5] += (double)nlo;
  acc[8] += (double)nhi;
  acc[11] += guess > 0 ? (double)nlo : 0.0;  // left out of this CTA's survivor list
  acc[12] += guess < 0 ? (double)nhi : 0.0;
  acc[13] += (double)nside;
  if ((threadIdx.x & 31) == 0) acc[14] += (double)sv_m;  // a warp total: counted once
  fence_proxy_async_global();  // generic stores -> the next passes' bulk loads
  *surv_m = sv_m;
  return out_m;
}

// ------------------------------------------------------------ the kernel
template <bool FIX>
__global__ void __launch_bounds__(kTmaThreads, 1) cqk_tma_kernel(CqkParams<double> p) {
  extern __shared__ __align__(128) unsigned char s_dyn[];
  __shared__ __align__(8) unsigned long long s_full[kStagesC], s_empty[kStagesC];
  __shared__ __align__(8) unsigned long long s_full3[kStages3], s_empty3[kStages3];
  __shared__ double s_red[kConsW + 1][kMaxK];
  __shared__ double s_tot[kMaxK];
  __shared__ Cmd s_cmd;
  __shared__ CqkState s_st;  // the decision state (every CTA's replica single-GPU, else CTA 0's)
  __shared__ unsigned s_gen0;
  __shared__ int s_abort;
  __shared__ int s_nslots;   // scratch slots of this CTA (max over its warps)
  __shared__ int s_nsl_new;  // ... being formed by a compacting pass
  __shared__ int s_nsl_side, s_nsl_side_new;  // side-list slots (fused start)
  __shared__ int s_nsl_surv;  // the fused pass's guessed survivors (compaction scratch)
  __shared__ int s_spec;     // tiles of the next pass issued across the grid step
  __shared__ int s_spec_scr; // ... and their walk: 0 original arrays, 1 scratch, 2 side list
  __shared__ unsigned long long s_probe_last;  // timeline probe: last consumer warp done
  __shared__ unsigned long long s_probe_pre;   // ... last warp (incl. producer) at the reduction
  __shared__ long long s_tix[kStagesC];        // dynamic final pass: tile index per stage
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == kConsW;
  const bool master = blockIdx.x == 0;
  TPipe pp{reinterpret_cast<double*>(s_dyn), smem_u32(s_full), smem_u32(s_empty), 0u};
  TPipe pp3{reinterpret_cast<double*>(s_dyn), smem_u32(s_full3), smem_u32(s_empty3), 0u};  // lambda0
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesC; ++s) {
      mbar_init_count(&s_full[s], 1);
      mbar_init_count(&s_empty[s], kConsW);
    }
    for (int s = 0; s < kStages3; ++s) {
      mbar_init_count(&s_full3[s], 1);
      mbar_init_count(&s_empty3[s], kConsW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_gen0 = ld_acquire(p.sync.gen);
    s_abort = 0;
    s_nslots = 0;
    s_nsl_new = 0;
    s_nsl_side = s_nsl_side_new = s_nsl_surv = 0;
    s_spec = 0;
    s_spec_scr = 0;
    s_probe_last = 0;
    s_probe_pre = 0;
    s_st = p.init;  // host-initialised, passed by value (every CTA: single-GPU replicas)
    s_cmd = s_st.cmd;
    if (master) tl_record(p.sync, 0, -1, p.n, 0);
    if (master && p.ar.tiles) *p.ar.tiles_next = 0u;
  }
  __syncthreads();
  const int64_t ntiles = (p.n + kTileC - 1) / kTileC;
  const TileWalk orig{p.n, ntiles, -1};
  const Src src_orig{{p.d, p.a, p.b, p.l, p.u, nullptr}};
  const Src src_scr{{p.sd, p.sa, p.sb, p.sl, p.su, nullptr}};
  const Src src_side{{p.vd, p.va, p.vb, p.vl, p.vu, nullptr}};
  const Src src_l0x{{p.d, p.a, p.b, p.l, p.u, p.xbar}};
  const bool prod_lane = producer && lane == 0;
  const int has_xbar = p.xbar != nullptr;
  const int check = p.init.check;  // immutable during the solve
  bool in_scratch = false;
  bool side_pending = false;  // the fused pass left a side list in the side scratch
  bool adopt_pending = false; // the side scan may have adopted the guessed survivors
  int64_t m_w = -1;  // this warp's scratch element count (consumers, once in scratch)
  int64_t m_side = 0, m_surv = 0;  // this warp's side-list / guessed-survivor counts
  int g_cta = 0;  // the direction guess the fused pass wrote its survivor lists for
  const bool guess_mode = FIX && p.init.fused_guess != 0;
  // The producer lane issues the first tiles of the most likely next pass (a
  // phi scan / breakpoint pass over the current working set -- or, before
  // any compaction, the final pass over the original arrays) while the grid
  // step is in flight: the loads do not depend on lambda.
  auto speculate = [&](int kind) {  // 0 original arrays, 1 scratch, 2 side list
    const TileWalk nw{p.n, ntiles, kind == 0 ? -1 : (kind == 1 ? s_nslots : s_nsl_side)};
    const Src& sr = kind == 0 ? src_orig : (kind == 1 ? src_scr : src_side);
    s_spec = (c_tma_flags & 1) ? 0 : produce<5>(sr, nw, pp, 0, kSpecDepthC);
    s_spec_scr = kind;
  };
  const bool probe = blockIdx.x == 1 && p.sync.timeline;  // timeline detail columns 10-15
  const bool single = p.ar.rows != nullptr;  // masterless grid step: every CTA decides
  GridSync dsync = p.sync;                   // the decision's timeline rows: CTA 0 only
  if (!master) dsync.timeline = nullptr;
  double* const dtrace = master ? p.trace : nullptr;
  for (unsigned epoch = 1;; ++epoch) {
    const Cmd c = s_cmd;
    int spec = s_spec;
    if (probe && threadIdx.x == 0) tl_mark(p.sync, epoch, 10);
    if (c.phase == PH_DONE || s_abort) {
      if (!producer) drain(pp, spec);  // never leave bulk copies in flight
      break;
    }
    const bool side_walk = side_pending && c.phase == PH_SCAN && c.side;
    if (side_pending && c.phase != PH_FUSED) side_pending = false;
    if (adopt_pending) {  // the epoch after the side scan: adopt the guessed survivors?
      adopt_pending = false;
      if (c.adopt != 0 && c.adopt == g_cta) {
        in_scratch = true;
        m_w = m_surv;
      }
    }
    // speculated tiles of another walk than this epoch's (a guess the
    // decision did not take, a side list not scanned) are dropped
    if (spec > 0 && c.phase != PH_FINAL && s_spec_scr != (side_walk ? 2 : (in_scratch ? 1 : 0))) {
      if (!producer) drain(pp, spec);
      spec = 0;
    }
    const TileWalk work{p.n, ntiles, side_walk ? s_nsl_side : (in_scratch ? s_nslots : -1)};
    const Src wsrc = side_walk ? src_side : (in_scratch ? src_scr : src_orig);
    const int64_t m_walk = side_walk ? m_side : m_w;
    if (c.phase == PH_FINAL) {
      if (blockIdx.x <= 1 && threadIdx.x == 0) tl_mark(p.sync, epoch, 10 + 2 * blockIdx.x);
      const bool reuse = spec > 0 && s_spec_scr == 0;  // the speculated tiles are the final's
      const bool dyn = p.ar.dyn_final != 0;          // single GPU: dynamic tile assignment
      const int D = kSpecDepthC;                     // its static prefix: the speculation's tiles
      if (p.x) {
        if (prod_lane) {
          if (dyn) produce_final_dyn<5, kStagesC, kStageElemsC, kTileC>(src_orig, p.n, pp, reuse ? spec : 0, D,
                                                                        p.ar.tiles, s_tix);
          else produce<5>(src_orig, orig, pp, reuse ? spec : 0);
        } else if (!producer) {
          if (!reuse) drain(pp, spec);
          t_final<FIX>(p, c, orig, pp, dyn ? D : -1, s_tix);
        }
      } else if (!producer) {
        drain(pp, spec);
      }
      if (p.sync.timeline) {  // uniform: CTA 0 / 1 end, and the last CTA's end
        __syncthreads();
        if (threadIdx.x == 0 && epoch < (unsigned)kTimelineCap) {
          if (blockIdx.x <= 1) tl_mark(p.sync, epoch, 11 + 2 * blockIdx.x);
          atomicMax(reinterpret_cast<unsigned long long*>(p.sync.timeline + kTimelineCols * epoch + 15),
                    globaltimer());
        }
      }
      break;
    }
    double acc[kMaxK];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) acc[k] = 0.0;
    bool is_master = false;
    if (c.phase == PH_LAMBDA0) {
#pragma unroll
      for (int k = kValidateSlot; k < kValidateSlot + 10; ++k) acc[k] = HUGE_VAL;
      if (prod_lane) {
        if (has_xbar) produce<6>(src_l0x, orig, pp);
        else produce<3, kStages3, kStride3>(src_l0x, orig, pp3);
      } else if (!producer) {
        if (check && has_xbar) t_lambda0<true, true>(p, orig, pp, acc);
        else if (check) t_lambda0<true, false>(p, orig, pp3, acc);
        else if (has_xbar) t_lambda0<false, true>(p, orig, pp, acc);
        else t_lambda0<false, false>(p, orig, pp3, acc);
      }
      const int ops[15] = {OP_SUM, OP_SUM, OP_SUM, OP_SUM, OP_SUM, OP_MIN, OP_MIN, OP_MIN,
                           OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN};
      double a15[15];
#pragma unroll
      for (int k = 0; k < 15; ++k) a15[k] = acc[k];
      block_reduce<15, kConsW>(a15, ops, s_red, s_tot);
      is_master = grid_step_any<15>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch,
                                   [&] { if (prod_lane) speculate(0); }, (c_tma_flags & 4) != 0);
      if (is_master && warp == 0) {
        if (lane == 0) tl_record(dsync, epoch, PH_LAMBDA0, p.n, 0);
        double glob[15];
        const bool ok = exchange_totals<15>(p.ex, epoch, ops, s_tot, glob, master);
        if (lane == 0) {
          if (ok) m_after_lambda0(s_st, glob);
          else {
            m_stop(s_st, ST_TIMEOUT);
            raise_timeout(p.sync);
          }
        }
      }
    } else if (c.phase == PH_SAMPLE) {
      // with the direction guess the sample tiles carry all five arrays and
      // stay in the main pipeline's stages (no speculation across this step)
      if (guess_mode) {
        if (prod_lane) produce_sample<5, kStagesC, kStageElemsC>(src_orig, p.n, ntiles, pp);
        else if (!producer) t_sample<kStagesC, kStageElemsC, true>(p, ntiles, pp, acc);
      } else {
        if (prod_lane) produce_sample(src_l0x, p.n, ntiles, pp3);
        else if (!producer) t_sample(p, ntiles, pp3, acc);
      }
      const int ops[3] = {OP_SUM, OP_SUM, OP_SUM};
      double a3[3] = {acc[0], acc[1], acc[2]};
      block_reduce<3, kConsW>(a3, ops, s_red, s_tot);
      is_master = grid_step_any<3>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch,
                                   [&] { if (prod_lane && !guess_mode) speculate(0); }, (c_tma_flags & 4) != 0);
      if (is_master && warp == 0) {
        if (lane == 0) tl_record(dsync, epoch, PH_SAMPLE, p.n, 0);
        double glob[3];
        const bool ok = exchange_totals<3>(p.ex, epoch, ops, s_tot, glob, master);
        if (lane == 0) {
          if (ok) m_after_sample(s_st, glob, s_tot[2]);
          else {
            m_stop(s_st, ST_TIMEOUT);
            raise_timeout(p.sync);
          }
        }
      }
    } else if (c.phase == PH_GUESS) {
      // phi at the estimate over the kept sample tiles, then free their
      // stages: the producer speculates the fused pass's first tiles across
      // this grid step
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
      if (!producer) {
        t_sample_guess(p, c.lam, ntiles, pp, a4);
        release_sample(ntiles, pp);
      }
      const int ops[4] = {OP_SUM, OP_SUM, OP_SUM, OP_SUM};
      block_reduce<4, kConsW>(a4, ops, s_red, s_tot);
      is_master = grid_step_any<4>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch,
                                   [&] { if (prod_lane) speculate(0); }, (c_tma_flags & 4) != 0);
      if (is_master && warp == 0) {
        if (lane == 0) tl_record(dsync, epoch, PH_GUESS, p.n, 0);
        double glob[4];
        const bool ok = exchange_totals<4>(p.ex, epoch, ops, s_tot, glob, master);
        if (lane == 0) {
          if (ok) m_after_guess(s_st, glob);
          else {
            m_stop(s_st, ST_TIMEOUT);
            raise_timeout(p.sync);
          }
        }
      }
    } else if (c.phase == PH_FUSED) {
      g_cta = c.guess;  // the global guess (every CTA alike)
      acc[2] = HUGE_VAL;  // the first failing validate() check (min)
      if (prod_lane) produce<5>(src_orig, orig, pp, spec);
      else if (!producer) {
        int64_t sv = 0;
        const int64_t mm = check ? t_fused<true>(p, c, orig, src_orig, pp, acc, g_cta, &sv)
                                 : t_fused<false>(p, c, orig, src_orig, pp, acc, g_cta, &sv);
        m_side = mm;
        m_surv = sv;
        if (lane == 0) {
          atomicMax(&s_nsl_side_new, (int)((mm + kSeg - 1) / kSeg));
          atomicMax(&s_nsl_new, (int)((sv + kSeg - 1) / kSeg));
        }
      }
      side_pending = true;  // speculate the side list: the likely next walk
      int ops[kFusedK];
      double aK[kFusedK];
#pragma unroll
      for (int k = 0; k < kFusedK; ++k) { ops[k] = k == 2 ? OP_MIN : OP_SUM; aK[k] = acc[k]; }
      block_reduce<kFusedK, kConsW>(aK, ops, s_red, s_tot);
      is_master = grid_step_any<kFusedK>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch, [&] {
        if (prod_lane) {
          s_nsl_side = s_nsl_side_new;
          s_nsl_side_new = 0;
          s_nsl_surv = s_nsl_new;
          s_nsl_new = 0;
          speculate(2);
        }
      }, (c_tma_flags & 4) != 0);
      if (is_master && warp == 0) {
        double loc[kFusedK], glob[kFusedK];
#pragma unroll
        for (int k = 0; k < kFusedK; ++k) loc[k] = s_tot[k];
        if (lane == 0) tl_record(dsync, epoch, PH_FUSED, p.n, 0);
        const bool ok = exchange_totals<kFusedK>(p.ex, epoch, ops, loc, glob, master);
        if (lane == 0) {
          if (ok) m_after_fused(s_st, glob, loc);
          else {
            m_stop(s_st, ST_TIMEOUT);
            raise_timeout(p.sync);
          }
        }
      }
    } else if (c.phase == PH_SCAN && c.check_lu) {
#pragma unroll
      for (int k = kCheckLuSlot; k < kMaxK; ++k) acc[k] = HUGE_VAL;
      if (prod_lane) produce<5>(src_orig, orig, pp, spec);
      else if (!producer) t_scan<FIX, true>(p, c, orig, -1, src_orig, false, pp, acc);
      int ops[kMaxK];
#pragma unroll
      for (int k = 0; k < kMaxK; ++k) ops[k] = k < kCheckLuSlot ? OP_SUM : OP_MIN;
      block_reduce<kMaxK, kConsW>(acc, ops, s_red, s_tot);
      is_master = grid_step_any<kMaxK>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch,
                                   [&] { if (prod_lane) speculate(in_scratch ? 1 : 0); }, (c_tma_flags & 4) != 0);
      if (is_master && warp == 0) {
        double loc[kMaxK], glob[kMaxK];
#pragma unroll
        for (int k = 0; k < kMaxK; ++k) loc[k] = s_tot[k];
        if (lane == 0) tl_record(dsync, epoch, PH_SCAN, s_st.phys_count, 0);
        const bool ok = exchange_totals<kMaxK>(p.ex, epoch, ops, s_tot, glob, master);
        if (lane != 0) {
        } else if (!ok) {
          m_stop(s_st, ST_TIMEOUT);
          raise_timeout(p.sync);
        } else {
          s_st.cmd.check_lu = 0;
          s_st.vidx[3] = glob[11];  // l NaN
          s_st.vidx[4] = glob[12];  // u NaN
          s_st.vidx[7] = glob[13];  // l <= u
          s_st.vidx[8] = glob[14];  // l == +inf
          s_st.vidx[9] = glob[15];  // u == -inf
          if (m_validate(s_st, 3, 10)) m_after_scan(s_st, glob, loc, dtrace);
        }
      }
    } else if (c.phase == PH_SCAN) {
      const bool compact = FIX && c.compact;
      if (prod_lane) {
        produce<5>(wsrc, work, pp, spec);
        if (probe) tl_mark(p.sync, epoch, 13);
      } else if (!producer) {
        const int64_t mm = t_scan<FIX, false>(p, c, work, m_walk, wsrc, compact, pp, acc);
        if (probe && threadIdx.x == 0) tl_mark(p.sync, epoch, 11);
        if (probe && lane == 0) atomicMax(&s_probe_last, (unsigned long long)globaltimer());
        if (compact) {
          m_w = mm;
          if (lane == 0) atomicMax(&s_nsl_new, (int)((mm + kSeg - 1) / kSeg));
        }
      }
      if (compact) in_scratch = true;
      // the side list is consumed: the working set is the original arrays, or
      // -- if the decision adopts them -- the fused pass's guessed survivors
      const bool spec_surv = side_walk && c.guess != 0;
      if (side_walk) adopt_pending = true;
      constexpr int K = FIX ? 11 : 5;
      int ops[K];
      double aK[K];
#pragma unroll
      for (int k = 0; k < K; ++k) { ops[k] = OP_SUM; aK[k] = acc[k]; }
      if (probe && lane == 0) atomicMax(&s_probe_pre, (unsigned long long)globaltimer());
      block_reduce<K, kConsW>(aK, ops, s_red, s_tot);  // (its barrier orders the atomicMax above)
      if (probe && threadIdx.x == 0) {
        tl_mark(p.sync, epoch, 12);
        if (p.sync.timeline && epoch < (unsigned)kTimelineCap) {
          p.sync.timeline[kTimelineCols * epoch + 14] = (long long)s_probe_last;
          p.sync.timeline[kTimelineCols * epoch + 15] = (long long)s_probe_pre;
        }
        s_probe_last = 0;
        s_probe_pre = 0;
      }
      is_master = grid_step_any<K>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch, [&] {
        if (prod_lane) {
          if (compact) {  // nobody else reads s_nslots before the next epoch
            s_nslots = s_nsl_new;
            s_nsl_new = 0;
          }
          if (spec_surv) s_nslots = s_nsl_surv;  // the likely (guessed) next walk
          speculate(spec_surv ? 1 : (in_scratch ? 1 : 0));
        }
      }, (c_tma_flags & 4) != 0);
      if (is_master && warp == 0) {
        double loc[11], glob[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) loc[k] = glob[k] = k < K ? s_tot[k] : 0.0;
        if (lane == 0) tl_record(dsync, epoch, PH_SCAN, s_st.phys_count, s_st.cmd.compact);
        const bool ok = exchange_totals<K>(p.ex, epoch, ops, s_tot, glob, master);
        if (lane == 0) {
          if (ok && c.side) m_add_aggregates(s_st, glob, loc);
          if (ok) m_after_scan(s_st, glob, loc, dtrace);
          else {
            m_stop(s_st, ST_TIMEOUT);
            raise_timeout(p.sync);
          }
        }
      }
    } else if (c.phase == PH_BP) {
      acc[0] = c.right ? HUGE_VAL : -HUGE_VAL;
      if (prod_lane) produce<5>(wsrc, work, pp, spec);
      else if (!producer) t_bp(p, c, FIX, work, m_walk, wsrc, pp, acc);
      int ops[2] = {c.right ? OP_MIN : OP_MAX, OP_SUM};
      double a2[2] = {acc[0], acc[1]};
      block_reduce<2, kConsW>(a2, ops, s_red, s_tot);
      is_master = grid_step_any<2>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch,
                                   [&] { if (prod_lane) speculate(in_scratch ? 1 : 0); }, (c_tma_flags & 4) != 0);
      if (is_master && warp == 0) {
        if (lane == 0) tl_record(dsync, epoch, PH_BP, s_st.phys_count, 0);
        double glob[2];
        const bool ok = exchange_totals<2>(p.ex, epoch, ops, s_tot, glob, master);
        if (lane == 0) {
          if (ok) m_after_bp(s_st, glob);
          else {
            m_stop(s_st, ST_TIMEOUT);
            raise_timeout(p.sync);
          }
        }
      }
    } else {
      break;
    }
    if (threadIdx.x == 0) {
      if (is_master) {
        const int ph = s_st.cmd.phase;
        if (master && (ph == PH_FINAL || ph == PH_DONE)) publish_state(p.out, s_st, p.sync);  // for the host
        s_cmd = s_st.cmd;
        if (!single) master_release(p.sync, s_gen0 + epoch, s_st.cmd, &p.st->cmd);
        if (master) tl_mark(p.sync, epoch, 5);
      } else if (!s_abort) {
        if (!wait_release(p.sync, s_gen0 + epoch, &p.st->cmd, &s_cmd)) s_abort = 1;
        if (blockIdx.x == 1) tl_mark(p.sync, epoch, 7);
      }
    }
    __syncthreads();
  }
}

// Scratch elements per array for the tile-slot layout (whole tiles).
inline int64_t tma_scratch_elems(int64_t n) { return (n + kTileC - 1) / kTileC * kTileC; }

}  // namespace cqk

// cqk_tma_spx.cuh -- TMA-pipelined persistent simplex / l1 projection
// (newton_project_simplex simplex.py:218-308, project_l1 simplex.py:311-333).
//
// The state machine is spx_solve_kernel's (s_after_init / s_after_scan /
// s_after_snap, cqk_kernels.cuh); underneath, the single streamed array (y,
// or the compacted working values w) goes through the same bulk-copy
// producer / consumer-warp pipeline as the CQK engine (cqk_tma.cuh), with
// 30 KB tiles (kTileY elements, 256 per consumer warp, 6 stages in flight)
// and the same warp sub-segment compaction (values only, 8 B per survivor).
#pragma once
#include "cqk_tma.cuh"

namespace cqk {

constexpr int kTileY = 256 * kConsW;                              // 3840 elements
constexpr int kSegY = kTileY / kConsW;                           // 256 per warp
constexpr int kEptY = kTileY / kConsT;                           // 8 per lane
constexpr int kStagesY = (int)(kSmemC / (kTileY * sizeof(double)));  // 6
static_assert(kStagesY >= 2, "pipeline needs at least two stages");

template <bool L1>
DEVI double spx_wv(double y) { return L1 ? fabs(y) : y; }

// MODE 0: sum / max of w; 1: phi scan (+ compaction); 2: max(-w) snap.
template <bool L1, int MODE, bool FULL>
DEVI void spx_tile(const WTile& wt, const double* src, bool scratch, double lam, bool fix,
                   double fhi, double (&acc)[kMaxK], int (&cnt)[2], bool (&keep)[kEptY],
                   double (&Wv)[kEptY]) {
  const int lane = threadIdx.x & 31;
  double Y[kEptY];
  tile_load<FULL, kTileY>(wt, 0, src, Y);
#pragma unroll
  for (int j = 0; j < kEptY; ++j) {
    const bool valid = FULL || e_loc(lane, j) < wt.wcnt;
    const double w = scratch ? Y[j] : spx_wv<L1>(Y[j]);  // scratch already holds w
    Wv[j] = w;
    if (MODE == 0) {
      keep[j] = false;
      acc[0] += valid ? w : 0.0;
      acc[1] = valid ? fmax(acc[1], w) : acc[1];
      continue;
    }
    const double v = add_rn(w, lam);
    const bool drop = fix && !(v > 0.0) && !(add_rn(w, fhi) > 0.0);
    const bool kp = valid && !drop;
    keep[j] = kp;
    if (MODE == 1) {
      const bool pos = v > 0.0;
      acc[0] += (kp && pos) ? v : 0.0;
      cnt[0] += kp && pos;
      cnt[1] += kp && v == 0.0;
    } else {
      acc[0] = kp ? fmax(acc[0], -w) : acc[0];
      cnt[0] += kp;
    }
  }
}

template <bool L1, int MODE>
DEVI int64_t t_spx(const SpxParams<double>& p, const Cmd& c, bool fix, const TileWalk& tw,
                   int64_t m_w, bool compact, TPipe& pp, double (&acc)[kMaxK]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned ltm = (1u << lane) - 1u;
  const bool scratch = tw.nslots >= 0;
  const double* src = scratch ? p.sy : p.y;
  const double lam = c.lam, fhi = c.fix_hi;
  int cnt[2] = {0, 0};
  int64_t out_m = 0, q_out = 0;
  int off_out = 0;
  const int64_t g = gridDim.x;
  consume<kStagesY, kTileY, kTileY>(tw, pp, m_w, [&](const WTile& wt) {
    bool keep[kEptY];
    double Wv[kEptY];
    if (wt.wcnt == kSegY) spx_tile<L1, MODE, true>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv);
    else spx_tile<L1, MODE, false>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv);
    if (MODE == 1 && compact) {  // warp sub-segment compaction of the values w
      const int64_t b0 = ((int64_t)blockIdx.x + q_out * g) * kTileY + kSegY * warp;
      const int64_t b1 = b0 + g * kTileY;
      int r = off_out;
#pragma unroll
      for (int j = 0; j < kEptY; ++j) {
        const unsigned bal = __ballot_sync(0xffffffffu, keep[j]);
        if (keep[j]) {
          const int o = r + __popc(bal & ltm);
          p.sy[o < kSegY ? b0 + o : b1 + (o - kSegY)] = Wv[j];
        }
        r += __popc(bal);
      }
      out_m += r - off_out;
      off_out = r;
      if (off_out >= kSegY) { off_out -= kSegY; ++q_out; }
    }
  });
  if (MODE == 1) { acc[1] += (double)cnt[0]; acc[2] += (double)cnt[1]; }
  if (MODE == 2) acc[1] += (double)cnt[0];
  if (MODE == 1 && compact) fence_proxy_async_global();
  return out_m;
}

template <bool L1, bool FULL>
DEVI void spx_final_tile(const SpxParams<double>& p, const WTile& wt, bool copy, double lam) {
  const int lane = threadIdx.x & 31;
  double Y[kEptY], X[kEptY];
  tile_load<FULL, kTileY>(wt, 0, p.y, Y);
#pragma unroll
  for (int j = 0; j < kEptY; ++j) {
    const double w = spx_wv<L1>(Y[j]);
    const double v = add_rn(w, lam);
    const double pos = v > 0.0 ? v : 0.0;  // np.maximum(0, w + lam)
    double x = pos;
    if (L1) {
      const double sg = Y[j] > 0.0 ? 1.0 : (Y[j] < 0.0 ? -1.0 : 0.0);
      x = mul_rn(sg, pos);
    }
    X[j] = copy ? Y[j] : x;
  }
#pragma unroll
  for (int u = 0; u < kEptY / 2; ++u) {
    const int e = 64 * u + 2 * lane;
    double* xp = p.x + wt.gbase + e;
    if (FULL || e + 1 < wt.wcnt) store_out(reinterpret_cast<double2*>(xp), make_double2(X[2 * u], X[2 * u + 1]));
    else if (e < wt.wcnt) *xp = X[2 * u];
  }
}

template <bool L1>
__global__ void __launch_bounds__(kTmaThreads, 1) spx_tma_kernel(SpxParams<double> p) {
  extern __shared__ __align__(128) unsigned char s_dyn[];
  __shared__ __align__(8) unsigned long long s_full[kStagesY], s_empty[kStagesY];
  __shared__ double s_red[kConsW + 1][kMaxK];
  __shared__ double s_tot[kMaxK];
  __shared__ Cmd s_cmd;
  __shared__ SpxState s_st;  // master (CTA 0) only
  __shared__ unsigned s_gen0;
  __shared__ int s_abort;
  __shared__ int s_nslots, s_nsl_new;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == kConsW;
  const bool prod_lane = producer && lane == 0;
  const bool master = blockIdx.x == 0;
  TPipe pp{reinterpret_cast<double*>(s_dyn), smem_u32(s_full), smem_u32(s_empty), 0u};
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesY; ++s) {
      mbar_init_count(&s_full[s], 1);
      mbar_init_count(&s_empty[s], kConsW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_gen0 = ld_acquire(p.sync.gen);
    s_abort = 0;
    s_nslots = s_nsl_new = 0;
    if (master) {
      s_st = *p.st;
      s_cmd = s_st.cmd;
      tl_record(p.sync, 0, -1, p.n, 0);
    } else {
      load_l2(&s_cmd, &p.st->cmd);
    }
  }
  __syncthreads();
  const bool fix = p.st->fixing != 0;
  const int64_t ntiles = (p.n + kTileY - 1) / kTileY;
  const TileWalk orig{p.n, ntiles, -1};
  bool in_scratch = false;
  int64_t m_w = -1;
  for (unsigned epoch = 1;; ++epoch) {
    const Cmd c = s_cmd;
    if (c.phase == PH_DONE || s_abort) break;
    const TileWalk work{p.n, ntiles, in_scratch ? s_nslots : -1};
    if (c.phase == PH_FINAL || c.phase == PH_COPY) {
      if (p.x) {
        const bool copy = c.phase == PH_COPY;
        if (prod_lane) {
          produce<1, kStagesY, kTileY, kTileY>(Src{{p.y}}, orig, pp);
        } else if (!producer) {
          const double lam = c.lam;
          consume<kStagesY, kTileY, kTileY>(orig, pp, -1, [&](const WTile& wt) {
            if (wt.wcnt == kSegY) spx_final_tile<L1, true>(p, wt, copy, lam);
            else spx_final_tile<L1, false>(p, wt, copy, lam);
          });
        }
      }
      break;
    }
    double acc[kMaxK];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) acc[k] = 0.0;
    int ops[3] = {OP_SUM, OP_SUM, OP_SUM};
    int mode;
    const Src wsrc{{in_scratch ? p.sy : p.y}};
    if (c.phase == PH_LAMBDA0) {
      mode = 0;
      acc[1] = -HUGE_VAL;
      ops[1] = OP_MAX;
      if (prod_lane) produce<1, kStagesY, kTileY, kTileY>(Src{{p.y}}, orig, pp);
      else if (!producer) t_spx<L1, 0>(p, c, false, orig, -1, false, pp, acc);
    } else if (c.phase == PH_SCAN) {
      mode = 1;
      const bool compact = fix && c.compact;
      if (prod_lane) {
        produce<1, kStagesY, kTileY, kTileY>(wsrc, work, pp);
      } else if (!producer) {
        const int64_t mm = t_spx<L1, 1>(p, c, fix, work, m_w, compact, pp, acc);
        if (compact) {
          m_w = mm;
          if (lane == 0) atomicMax(&s_nsl_new, (int)((mm + kSegY - 1) / kSegY));
        }
      }
      if (compact) in_scratch = true;
    } else if (c.phase == PH_SNAP) {
      mode = 2;
      acc[0] = -HUGE_VAL;
      ops[0] = OP_MAX;
      if (prod_lane) produce<1, kStagesY, kTileY, kTileY>(wsrc, work, pp);
      else if (!producer) t_spx<L1, 2>(p, c, fix, work, m_w, false, pp, acc);
    } else {
      break;
    }
    double a3[3] = {acc[0], acc[1], acc[2]};
    block_reduce<3>(a3, ops, s_red, s_tot);  // (its barrier orders the atomicMax above)
    if (mode == 1 && fix && c.compact && threadIdx.x == 0) {
      s_nslots = s_nsl_new;
      s_nsl_new = 0;
    }
    const bool is_master = grid_step<3>(p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch);
    if (threadIdx.x == 0) {
      if (is_master) {
        tl_record(p.sync, epoch, c.phase, mode == 0 ? p.n : s_st.phys_count, s_st.cmd.compact);
        double loc[3] = {s_tot[0], s_tot[1], s_tot[2]}, glob[3];
        if (!exchange_totals(p.ex, epoch, 3, ops, loc, glob)) {
          s_st.status = ST_TIMEOUT;
          s_st.cmd.phase = PH_DONE;
        } else if (mode == 0) s_after_init(s_st, glob);
        else if (mode == 1) s_after_scan(s_st, glob, loc, p.trace);
        else s_after_snap(s_st, glob);
        const int ph = s_st.cmd.phase;
        if (ph == PH_FINAL || ph == PH_DONE || ph == PH_COPY) *p.st = s_st;
        s_cmd = s_st.cmd;
        master_release(p.sync, s_gen0 + epoch, s_st.cmd, &p.st->cmd);
        tl_mark(p.sync, epoch, 5);
      } else if (!s_abort) {
        if (!wait_release(p.sync, s_gen0 + epoch, &p.st->cmd, &s_cmd)) s_abort = 1;
        if (blockIdx.x == 1) tl_mark(p.sync, epoch, 7);
      }
    }
    __syncthreads();
  }
}

inline int64_t tma_scratch_elems_y(int64_t n) { return (n + kTileY - 1) / kTileY * kTileY; }

}  // namespace cqk

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
#define kSpecDepthY ((c_tma_flags & 8) ? 3 : kStagesY)  // next-pass tiles speculated (simplex)
static_assert(kStagesY >= 2, "pipeline needs at least two stages");

template <bool L1>
DEVI double spx_wv(double y) { return L1 ? fabs(y) : y; }

// Start "auto": the first scan (at the tight start lam0 = r - max w, an upper
// bound of the root) also counts its positive t = w + lam0 in kHistB buckets of
// width r / kHistB (integer counts: order-independent, hence deterministic).
// With one bucket of margin for rounding, an element in bucket j has
// t >= (j - 1) r / kHistB, so phi(lam0 - k r / kHistB) >= (r / kHistB)
// sum_{j > k} c_j (j - 1 - k): the largest k making that >= r gives an upper
// bound of the root within about a bucket of it.  The master takes it in
// place of the first Newton step when smaller, which skips the linear
// shrinking phase of Newton-from-above on spread data (u01: 8 grid epochs -> 4).
constexpr int kHistB = 1024;
static_assert(kHistB == 2 * kTmaThreads, "hist_bound: two buckets per thread");
static_assert((kHistB & (kHistB - 1)) == 0, "power of two");
// Tail mode: once the physical working set fits one SM's shared memory, the
// master CTA gathers it (from the warp sub-segments, whose counts every warp
// published in its last compacting pass, or from y itself) and runs the
// remaining Newton iterations alone -- a block reduction and the state
// machine per iteration, no grid barrier -- then releases the grid into the
// final pass.  Single-GPU solves only.
constexpr int kTailY = 16384;  // elements (128 KB of the stage memory)
static_assert(kTailY * sizeof(double) <= kSmemC, "tail set must fit the stage memory");

// Gather the working set into V[0, m) (master CTA, all threads).  The
// (CTA, warp) pairs' counts are scanned into exclusive offsets in shared
// memory behind V; then every thread copies elements e = tid, tid + nt, ...,
// finding its pair by binary search -- kGatherBatch searches in lockstep, then
// their loads together (a per-pair loop serialised one L2 round trip per
// element; serial searches cost ~2 us more).
constexpr int kGatherBatch = 8;
constexpr int kMaxGridY = 256;  // tail mode needs gridDim.x <= this (one CTA per SM)
constexpr int kGatherPer = (kMaxGridY * kConsW + kTmaThreads - 1) / kTmaThreads;  // pairs per thread
static_assert(kTailY * sizeof(double) + 4 * (kMaxGridY * kConsW + 1) <= kSmemC,
              "tail set + pair offsets must fit the stage memory");
template <bool L1>
DEVI int tail_gather(const SpxParams<double>& p, bool in_scratch, double* V, int* s_scan) {
  const int nt = blockDim.x, tid = threadIdx.x;
  if (!in_scratch) {
    const int m = (int)p.n;
    for (int i = tid; i < m; i += nt) V[i] = spx_wv<L1>(p.y[i]);
    __syncthreads();  // the tail iterations read V in per-thread runs, not in this stride
    return m;
  }
  int* off = reinterpret_cast<int*>(V + kTailY);  // [pairs + 1] exclusive offsets
  // pairs k = c * kConsW + w, a contiguous block of them per thread, in order
  const int pairs = (int)gridDim.x * kConsW;
  const int per = (pairs + nt - 1) / nt;
  const int k0 = min(tid * per, pairs), k1 = min(k0 + per, pairs);
  int cnt[kGatherPer], mine = 0;  // per <= kGatherPer: gridDim.x <= kMaxGridY
#pragma unroll
  for (int j = 0; j < kGatherPer; ++j) {
    cnt[j] = k0 + j < k1 ? __ldcg(p.wcnt + k0 + j) : 0;
    mine += cnt[j];
  }
  // block exclusive scan of `mine` (warp inclusive scans + warp totals)
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_scan[warp] = incl;
  __syncthreads();
  int wpre = 0, total = 0;
  for (int w = 0; w < nw; ++w) {
    const int v = s_scan[w];
    wpre += w < warp ? v : 0;
    total += v;
  }
  int o = wpre + incl - mine;
#pragma unroll
  for (int j = 0; j < kGatherPer; ++j) {
    if (k0 + j < k1) off[k0 + j] = o;
    o += cnt[j];
  }
  if (tid == 0) off[pairs] = total;
  __syncthreads();
  const int64_t g = gridDim.x;
  // the kGatherBatch searches advance in lockstep (independent shared loads
  // per step) and then their global loads issue together
  const int steps = 32 - __clz(pairs);  // ceil(log2(pairs + 1))
  for (int e0 = tid; e0 < total; e0 += kGatherBatch * nt) {
    int lo[kGatherBatch], hi[kGatherBatch], e[kGatherBatch];
#pragma unroll
    for (int b = 0; b < kGatherBatch; ++b) {
      e[b] = min(e0 + b * nt, total - 1);
      lo[b] = 0;  // largest k with off[k] <= e: off[lo] <= e < off[hi]
      hi[b] = pairs;
    }
    for (int st = 0; st < steps; ++st) {
#pragma unroll
      for (int b = 0; b < kGatherBatch; ++b) {
        const int mid = (lo[b] + hi[b]) >> 1;
        if (hi[b] - lo[b] > 1) {
          if (off[mid] <= e[b]) lo[b] = mid;
          else hi[b] = mid;
        }
      }
    }
    double v[kGatherBatch];
#pragma unroll
    for (int b = 0; b < kGatherBatch; ++b) {
      const int i = e[b] - off[lo[b]], c = lo[b] / kConsW, w = lo[b] % kConsW;
      v[b] = __ldcg(p.sy + ((int64_t)c + (int64_t)(i / kSegY) * g) * kTileY + kSegY * w + (i % kSegY));
    }
#pragma unroll
    for (int b = 0; b < kGatherBatch; ++b)
      if (e0 + b * nt < total) V[e0 + b * nt] = v[b];
  }
  __syncthreads();
  return total;
}

// MODE 0: sum / max of w; 1: phi scan (+ compaction); 2: max(-w) snap;
// 3: MODE 0's sums in the same order plus the capture of w >= lam (the
// threshold T of the capture start, s_after_sample).
template <bool L1, int MODE, bool FULL, bool HIST = false>
DEVI void spx_tile(const WTile& wt, const double* src, bool scratch, double lam, bool fix,
                   double fhi, double (&acc)[kMaxK], int (&cnt)[2], bool (&keep)[kEptY],
                   double (&Wv)[kEptY], int* s_hist, double hscale, uint32_t* signw = nullptr) {
  const int lane = threadIdx.x & 31;
  double Y[kEptY];
  tile_load<FULL, kTileY>(wt, 0, src, Y);
  if (MODE == 3 && L1 && signw) {  // capture start, l1: the sign bits for the sparse final
    uint32_t b[kEptY];
#pragma unroll
    for (int j = 0; j < kEptY; ++j)
      b[j] = __ballot_sync(0xffffffffu, (FULL || e_loc(lane, j) < wt.wcnt) && Y[j] < 0.0);
    static_assert(kEptY == 8, "two 16-byte stores of sign words");
    if (lane == 0) {
      reinterpret_cast<uint4*>(signw)[0] = make_uint4(b[0], b[1], b[2], b[3]);
      reinterpret_cast<uint4*>(signw)[1] = make_uint4(b[4], b[5], b[6], b[7]);
    }
  }
#pragma unroll
  for (int j = 0; j < kEptY; ++j) {
    const bool valid = FULL || e_loc(lane, j) < wt.wcnt;
    const double w = scratch ? Y[j] : spx_wv<L1>(Y[j]);  // scratch already holds w
    Wv[j] = w;
    if (MODE == 0 || MODE == 3) {
      keep[j] = MODE == 3 && valid && w >= lam;
      acc[0] += valid ? w : 0.0;
      acc[1] = valid ? fmax(acc[1], w) : acc[1];
      if (MODE == 3) cnt[0] += keep[j];
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
      if (HIST && kp && pos) atomicAdd(&s_hist[min(kHistB - 1, (int)(v * hscale))], 1);
    } else {
      acc[0] = kp ? fmax(acc[0], -w) : acc[0];
      cnt[0] += kp;
    }
  }
}

template <bool L1, int MODE>
DEVI int64_t t_spx(const SpxParams<double>& p, const Cmd& c, bool fix, const TileWalk& tw,
                   int64_t m_w, bool compact, TPipe& pp, double (&acc)[kMaxK],
                   int* s_hist = nullptr, double hscale = 0.0) {
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
    if (MODE == 3) {  // the capture start's fused pass (original tiles, static walk)
      uint32_t* sw = L1 && p.signs
                         ? p.signs + ((wt.gbase - kSegY * warp) / kTileY * kConsW + warp) * kEptY
                         : nullptr;
      if (wt.wcnt == kSegY)
        spx_tile<L1, MODE, true>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv, s_hist, hscale, sw);
      else
        spx_tile<L1, MODE, false>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv, s_hist, hscale, sw);
    } else if (MODE == 1 && s_hist) {
      if (wt.wcnt == kSegY)
        spx_tile<L1, MODE, true, true>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv, s_hist, hscale);
      else
        spx_tile<L1, MODE, false, true>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv, s_hist, hscale);
    } else if (wt.wcnt == kSegY) {
      spx_tile<L1, MODE, true>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv, s_hist, hscale);
    } else {
      spx_tile<L1, MODE, false>(wt, src, scratch, lam, fix, fhi, acc, cnt, keep, Wv, s_hist, hscale);
    }
    bool any_keep = false;
#pragma unroll
    for (int j = 0; j < kEptY; ++j) any_keep = any_keep || keep[j];
    // survivors are rare in projections: most tiles have none to write
    if ((MODE == 1 || MODE == 3) && compact && __any_sync(0xffffffffu, any_keep)) {  // warp sub-segment compaction
      const int64_t b0 = ((int64_t)blockIdx.x + q_out * g) * kTileY + kSegY * warp;
      const int64_t b1 = b0 + g * kTileY;
      int r = off_out;
#pragma unroll
      for (int j = 0; j < kEptY; ++j) {
        const unsigned bal = __ballot_sync(0xffffffffu, keep[j]);
        if (keep[j]) {
          const int o = r + __popc(bal & ltm);
          const int64_t pos = o < kSegY ? b0 + o : b1 + (o - kSegY);
          p.sy[pos] = Wv[j];
          if (MODE == 3 && p.sidx) p.sidx[pos] = wt.gbase + e_loc(lane, j);  // for the sparse final
        }
        r += __popc(bal);
      }
      out_m += r - off_out;
      off_out = r;
      if (off_out >= kSegY) { off_out -= kSegY; ++q_out; }
    }
  });
  if (MODE == 1) { acc[1] += (double)cnt[0]; acc[2] += (double)cnt[1]; }
  if (MODE == 1 && compact && lane == 0) acc[3] += (double)out_m;  // survivors written (a warp total)
  if (MODE == 2) acc[1] += (double)cnt[0];
  if (MODE == 3) acc[2] += (double)cnt[0];
  if ((MODE == 1 || MODE == 3) && compact) fence_proxy_async_global();
  return out_m;
}

// The capture start's sample: this CTA's sample tiles (cqk_tma.cuh
// sample_tile, over the simplex tiling) of y; acc 0 sum w, 1 sum w^2,
// 2 elements, 3 max w.
DEVI void produce_sample_y(const double* y, int64_t n, int64_t ntiles, TPipe& pp) {
  for (int k = 0; k < kSampleTiles; ++k) {
    const int64_t t = sample_tile(ntiles, k);
    if (t < 0) break;
    const int s = pp.pc % kStagesY;
    const unsigned ph = ((pp.pc / kStagesY) & 1) ^ 1;
    if (pp.pc >= (unsigned)kStagesY) mbar_wait_s(pp.empty + 8 * s, ph);
    const int64_t left = n - t * kTileY;
    const unsigned bytes = ((unsigned)(left < kTileY ? left : kTileY) * 8u) & ~15u;
    const unsigned fb = pp.full + 8 * s;
    mbar_expect_tx_s(fb, bytes);
    if (bytes) tma_load_1d_s(smem_u32(pp.buf) + (unsigned)(s * kTileY) * 8u, y + t * kTileY, bytes, fb);
    ++pp.pc;
  }
}
template <bool L1>
DEVI void t_sample_y(const SpxParams<double>& p, int64_t ntiles, TPipe& pp, double (&acc)[kMaxK]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < kSampleTiles; ++k) {
    const int64_t t = sample_tile(ntiles, k);
    if (t < 0) break;
    const int s = pp.pc % kStagesY;
    WTile wt;
    wt.sm = pp.buf + (size_t)s * kTileY + kSegY * warp;
    wt.gbase = t * kTileY + kSegY * warp;
    const int64_t left = p.n - wt.gbase;
    wt.wcnt = left <= 0 ? 0 : (left < kSegY ? (int)left : kSegY);
    wt.patch = (wt.wcnt & 1) && wt.wcnt < kSegY;
    wt.q = k;
    mbar_wait_s(pp.full + 8 * s, (pp.pc / kStagesY) & 1);
    if (wt.wcnt > 0) {
      double Y[kEptY];
      tile_load<false, kTileY>(wt, 0, p.y, Y);
#pragma unroll
      for (int j = 0; j < kEptY; ++j) {
        if (e_loc(lane, j) >= wt.wcnt) continue;
        const double w = spx_wv<L1>(Y[j]);
        acc[0] += w;
        acc[1] += w * w;
        acc[2] += 1.0;
        acc[3] = fmax(acc[3], w);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_s(pp.empty + 8 * s);
    ++pp.pc;
  }
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

// The sparse final of the capture start (cmd.sparse): every element the
// fused pass did not capture has w + lam* < 0, so its x is a zero -- signed
// like sign(y) * 0 for l1 (the sign bits the fused pass recorded), +0 for
// the simplex -- and is written without re-reading y (8 B per element
// instead of 16).  After a grid barrier each warp scatters the x of the
// elements it captured (their indices sit in the fused pass's slots), with
// spx_final_tile's formula: x = max(0, w + lam), sign restored for l1.
template <bool L1>
DEVI void spx_sparse_final(const SpxParams<double>& p, double lam, int64_t ntiles, int64_t m_cap) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t G = gridDim.x;
  if (warp < kConsW) {
    // groups of kGrp tiles: their sign words are loaded together (lane
    // 8k + j holds word j of the group's k-th tile), then the stores follow,
    // so the warp does not wait one load latency per tile
    constexpr int kGrp = 4;
    static_assert(kGrp * kEptY <= 32, "one sign word per lane");
    for (int64_t t0 = blockIdx.x; t0 < ntiles; t0 += kGrp * G) {
      uint32_t mine = 0u;
      if (L1) {
        const int k = lane / kEptY, j = lane % kEptY;
        const int64_t t = t0 + k * G;
        if (t < ntiles) mine = __ldcg(p.signs + (t * kConsW + warp) * kEptY + j);
      }
#pragma unroll
      for (int k = 0; k < kGrp; ++k) {
        const int64_t t = t0 + k * G;
        const int64_t gbase = t * kTileY + kSegY * warp;
        const int64_t left = p.n - gbase;
        const int wcnt = t >= ntiles || left <= 0 ? 0 : (left < kSegY ? (int)left : kSegY);
        uint32_t sg[kEptY];
#pragma unroll
        for (int j = 0; j < kEptY; ++j) sg[j] = L1 ? __shfl_sync(0xffffffffu, mine, k * kEptY + j) : 0u;
        if (wcnt <= 0) continue;
#pragma unroll
        for (int u = 0; u < kEptY / 2; ++u) {
          const int e = 64 * u + 2 * lane;
          const double x0 = (L1 && ((sg[2 * u] >> lane) & 1u)) ? -0.0 : 0.0;
          const double x1 = (L1 && ((sg[2 * u + 1] >> lane) & 1u)) ? -0.0 : 0.0;
          double* xp = p.x + gbase + e;
          if (e + 1 < wcnt) store_out(reinterpret_cast<double2*>(xp), make_double2(x0, x1));
          else if (e < wcnt) *xp = x0;
        }
      }
    }
  }
  // grid barrier (the launch's final-tile counter, which arrives zero):
  // every zero is written before any scatter
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p.ar.tiles, 1u);
    const unsigned long long t0 = globaltimer();
    unsigned polls = 0;
    while (ld_acquire(p.ar.tiles) < (unsigned)G) {
      if ((++polls & 255u) == 0 && globaltimer() - t0 > kSpinTimeoutNs) {
        raise_timeout(p.sync);
        break;
      }
    }
  }
  __syncthreads();
  if (warp < kConsW) {
    for (int64_t i = lane; i < m_cap; i += 32) {
      const int64_t pos = ((int64_t)blockIdx.x + (i / kSegY) * G) * kTileY + kSegY * warp + (i % kSegY);
      const int64_t idx = __ldcg(p.sidx + pos);
      const double yv = p.y[idx];
      const double v = add_rn(spx_wv<L1>(yv), lam);
      const double pos_v = v > 0.0 ? v : 0.0;  // np.maximum(0, w + lam)
      double x = pos_v;
      if (L1) {
        const double sgv = yv > 0.0 ? 1.0 : (yv < 0.0 ? -1.0 : 0.0);
        x = mul_rn(sgv, pos_v);
      }
      p.x[idx] = x;
    }
  }
}

// The sparse output (output="sparse", simplex.py:296-300 / 328-331): with the
// captured list adopted, the nonzero x are among the captured elements; each
// warp appends its captured elements' nonzero x as (index, value) pairs
// through a grid counter (the host sorts them by index) -- no dense x at all.
template <bool L1>
DEVI void spx_sparse_output(const SpxParams<double>& p, double lam, int64_t m_cap) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t G = gridDim.x;
  if (warp >= kConsW) return;
  for (int64_t i = lane; i < m_cap; i += 32) {
    const int64_t pos = ((int64_t)blockIdx.x + (i / kSegY) * G) * kTileY + kSegY * warp + (i % kSegY);
    const int64_t idx = __ldcg(p.sidx + pos);
    const double yv = p.y[idx];
    const double v = add_rn(spx_wv<L1>(yv), lam);
    if (!(v > 0.0)) continue;  // simplex.py:298: tvals > 0
    double x = v;
    if (L1) x = mul_rn(yv > 0.0 ? 1.0 : (yv < 0.0 ? -1.0 : 0.0), v);
    const unsigned long long slot = atomicAdd(p.out_cnt, 1ull);
    if ((int64_t)slot < p.out_cap) {
      p.out_idx[slot] = idx;
      p.out_val[slot] = x;
    }
  }
}

// Master CTA: sum the per-CTA bucket rows (integers, any order), suffix-scan
// c_j and j c_j from the top, and take the largest k whose lower bound
// (r / kHistB) sum_{j > k} c_j (j - 1 - k) reaches r.  Two buckets per
// thread (kHistB == 2 * blockDim.x); all sums are exact integers.
DEVI void hist_bound(const SpxParams<double>& p, double lam0, double r, int* s_hist, SpxState& st) {
  __shared__ long long s_w1[32], s_w2[32];
  __shared__ int s_kbest;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const int G = (int)gridDim.x;
  // thread t owns buckets kb = kHistB - 2 - 2t + {1, 0}: idx' = 2t, 2t+1 from the top
  const int k_hi = kHistB - 1 - 2 * t, k_lo = k_hi - 1;
  const long long c_hi = __ldcg(p.hist + k_hi), c_lo = __ldcg(p.hist + k_lo);
  (void)G;
  // inclusive scans (from the top) of c and j*c over this thread's pair
  long long a1 = c_hi + c_lo, a2 = (long long)k_hi * c_hi + (long long)k_lo * c_lo;
  long long i1 = a1, i2 = a2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v1 = __shfl_up_sync(0xffffffffu, i1, o), v2 = __shfl_up_sync(0xffffffffu, i2, o);
    if (lane >= o) { i1 += v1; i2 += v2; }
  }
  if (lane == 31) { s_w1[warp] = i1; s_w2[warp] = i2; }
  if (t == 0) s_kbest = -1;
  __syncthreads();
  long long b1 = 0, b2 = 0;
  for (int w = 0; w < warp && w < nw; ++w) { b1 += s_w1[w]; b2 += s_w2[w]; }
  // sums over j > k: for k_hi everything before this thread; for k_lo add c_hi
  const long long S1_hi = b1 + i1 - a1, S2_hi = b2 + i2 - a2;
  const long long S1_lo = S1_hi + c_hi, S2_lo = S2_hi + (long long)k_hi * c_hi;
  const double bw = r / kHistB, need = r * (1.0 + 1e-12);
  int kb = -1;
  if (k_hi < kHistB - 1 && bw * (double)(S2_hi - (long long)(1 + k_hi) * S1_hi) >= need) kb = k_hi;
  else if (bw * (double)(S2_lo - (long long)(1 + k_lo) * S1_lo) >= need) kb = k_lo;
  if (kb >= 0) atomicMax(&s_kbest, kb);  // an integer max: order-independent
  __syncthreads();
  if (t == 0) st.lam_hist = s_kbest >= 0 ? lam0 - (double)s_kbest * bw : NAN;
  (void)s_hist;
}

template <bool L1>
__global__ void __launch_bounds__(kTmaThreads, 1) spx_tma_kernel(SpxParams<double> p) {
  extern __shared__ __align__(128) unsigned char s_dyn[];
  __shared__ __align__(8) unsigned long long s_full[kStagesY], s_empty[kStagesY];
  __shared__ double s_red[kConsW + 1][kMaxK];
  __shared__ double s_tot[kMaxK];
  __shared__ Cmd s_cmd;
  __shared__ SpxState s_st;  // the decision state (every CTA's replica single-GPU, else CTA 0's)
  __shared__ unsigned s_gen0;
  __shared__ int s_abort;
  __shared__ int s_nslots, s_nsl_new;
  __shared__ int s_spec, s_spec_scr;  // next-pass tiles issued across the grid step
  __shared__ int s_tail;              // master: finish the iterations in this CTA
  __shared__ int s_scan[kConsW + 1];
  __shared__ int s_hist[kHistB];      // start "auto": first-scan bucket counts
  __shared__ long long s_tix[kStagesY];  // dynamic final pass: tile index per stage
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
    s_spec = s_spec_scr = 0;
    s_tail = 0;
    s_st = p.init;  // every CTA: single-GPU replicas of the state machine
    s_cmd = s_st.cmd;
    if (master) tl_record(p.sync, 0, -1, p.n, 0);
    if (master && p.ar.tiles) *p.ar.tiles_next = 0u;
  }
  for (int k = threadIdx.x; k < kHistB; k += blockDim.x) s_hist[k] = 0;
  // the histograms alternate between launches: this one arrives zero, the
  // other (the previous launch's) is cleared here for the next
  if (master && p.hist_next)
    for (int k = threadIdx.x; k < kHistB; k += blockDim.x) p.hist_next[k] = 0;
  __syncthreads();
  const bool single = p.ar.rows != nullptr;  // masterless grid step: every CTA decides
  GridSync dsync = p.sync;                   // the decision's timeline rows: CTA 0 only
  if (!master) dsync.timeline = nullptr;
  double* const dtrace = master ? p.trace : nullptr;
  const bool fix = p.init.fixing != 0;
  const int64_t ntiles = (p.n + kTileY - 1) / kTileY;
  const TileWalk orig{p.n, ntiles, -1};
  bool in_scratch = false;
  int64_t m_w = -1;
  bool cap_pending = false;  // the capture start's list is in scratch, adoption undecided
  int64_t m_cap = 0;         // this warp's captured elements (the sparse final's scatter)
  // first tiles of the likely next pass, issued while the grid step runs
  // (cqk_tma.cuh: the loads do not depend on lambda)
  auto speculate = [&]() {
    const TileWalk nw{p.n, ntiles, in_scratch ? s_nslots : -1};
    s_spec = (c_tma_flags & 1) ? 0
                               : produce<1, kStagesY, kTileY, kTileY>(Src{{in_scratch ? p.sy : p.y}}, nw,
                                                                      pp, 0, kSpecDepthY);
    s_spec_scr = in_scratch;
  };
  for (unsigned epoch = 1;; ++epoch) {
    const Cmd c = s_cmd;
    int spec = s_spec;
    if (c.phase == PH_DONE || s_abort) {
      if (!producer) drain<kStagesY>(pp, spec);
      break;
    }
    if (cap_pending) {  // the epoch after the fused pass: is the captured list the working set?
      cap_pending = false;
      if (!c.side) {
        in_scratch = false;
        m_w = -1;
        if (spec > 0 && s_spec_scr && c.phase != PH_FINAL && c.phase != PH_COPY) {
          if (!producer) drain<kStagesY>(pp, spec);  // speculated from the list
          spec = 0;
        }
      }
    }
    const TileWalk work{p.n, ntiles, in_scratch ? s_nslots : -1};
    if (c.phase == PH_FINAL && c.sparse && p.out_idx && p.sidx) {  // output="sparse"
      if (!producer) drain<kStagesY>(pp, spec);
      spx_sparse_output<L1>(p, c.lam, m_cap);
      break;
    }
    const bool sparse = c.phase == PH_FINAL && c.sparse && p.x && p.sidx && p.ar.tiles;
    if (sparse) {  // the capture start's final: signed zeros + a scatter, y not re-read
      if (blockIdx.x <= 1 && threadIdx.x == 0) tl_mark(p.sync, epoch, 10 + 2 * blockIdx.x);
      if (!producer) drain<kStagesY>(pp, spec);
      spx_sparse_final<L1>(p, c.lam, ntiles, m_cap);
      if (p.sync.timeline && threadIdx.x == 0 && epoch < (unsigned)kTimelineCap) {
        if (blockIdx.x <= 1) tl_mark(p.sync, epoch, 11 + 2 * blockIdx.x);
        atomicMax(reinterpret_cast<unsigned long long*>(p.sync.timeline + kTimelineCols * epoch + 15),
                  globaltimer());
      }
      break;
    }
    if (c.phase == PH_FINAL || c.phase == PH_COPY) {
      if (blockIdx.x <= 1 && threadIdx.x == 0) tl_mark(p.sync, epoch, 10 + 2 * blockIdx.x);
      const bool reuse = spec > 0 && !s_spec_scr;
      const bool dyn = p.ar.dyn_final != 0;  // single GPU: dynamic tile assignment (cqk_tma.cuh)
      if (p.x) {
        const bool copy = c.phase == PH_COPY;
        if (prod_lane) {
          if (dyn) produce_final_dyn<1, kStagesY, kTileY, kTileY>(Src{{p.y}}, p.n, pp, reuse ? spec : 0,
                                                                   kSpecDepthY, p.ar.tiles, s_tix);
          else produce<1, kStagesY, kTileY, kTileY>(Src{{p.y}}, orig, pp, reuse ? spec : 0);
        } else if (!producer) {
          if (!reuse) drain<kStagesY>(pp, spec);
          const double lam = c.lam;
          auto body = [&](const WTile& wt) {
            if (wt.wcnt == kSegY) spx_final_tile<L1, true>(p, wt, copy, lam);
            else spx_final_tile<L1, false>(p, wt, copy, lam);
          };
          if (dyn) consume_final_dyn<kStagesY, kTileY, kTileY>(p.n, pp, kSpecDepthY, s_tix, body);
          else consume<kStagesY, kTileY, kTileY>(orig, pp, -1, body);
        }
      } else if (!producer) {
        drain<kStagesY>(pp, spec);
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
    int ops[4] = {OP_SUM, OP_SUM, OP_SUM, OP_SUM};
    int mode;
    const Src wsrc{{in_scratch ? p.sy : p.y}};
    if (c.phase == PH_SAMPLE) {
      mode = 4;
      acc[3] = -HUGE_VAL;
      ops[3] = OP_MAX;
      if (prod_lane) produce_sample_y(p.y, p.n, ntiles, pp);
      else if (!producer) t_sample_y<L1>(p, ntiles, pp, acc);
    } else if (c.phase == PH_FUSED) {
      mode = 3;
      acc[1] = -HUGE_VAL;
      ops[1] = OP_MAX;
      if (prod_lane) produce<1, kStagesY, kTileY, kTileY>(Src{{p.y}}, orig, pp, spec);
      else if (!producer) {
        Cmd ct = c;
        ct.lam = c.edge;  // the capture threshold
        const int64_t mm = t_spx<L1, 3>(p, ct, false, orig, -1, true, pp, acc);
        m_w = mm;
        m_cap = mm;
        if (lane == 0) {
          atomicMax(&s_nsl_new, (int)((mm + kSegY - 1) / kSegY));
          if (p.wcnt) p.wcnt[blockIdx.x * kConsW + warp] = (int32_t)(mm < kTailY ? mm : kTailY);
        }
      }
      in_scratch = true;  // speculate the captured list: the likely next walk
      cap_pending = true;
    } else if (c.phase == PH_LAMBDA0) {
      mode = 0;
      acc[1] = -HUGE_VAL;
      ops[1] = OP_MAX;
      if (prod_lane) produce<1, kStagesY, kTileY, kTileY>(Src{{p.y}}, orig, pp, spec);
      else if (!producer) t_spx<L1, 0>(p, c, false, orig, -1, false, pp, acc);
    } else if (c.phase == PH_SCAN) {
      mode = 1;
      const bool compact = fix && c.compact;
      if (prod_lane) {
        produce<1, kStagesY, kTileY, kTileY>(wsrc, work, pp, spec);
      } else if (!producer) {
        const bool hist = c.hist && p.hist;
        const int64_t mm = t_spx<L1, 1>(p, c, fix, work, m_w, compact, pp, acc,
                                        hist ? s_hist : nullptr, (double)kHistB / p.init.r);
        if (compact) {
          m_w = mm;
          if (lane == 0) {
            atomicMax(&s_nsl_new, (int)((mm + kSegY - 1) / kSegY));
            if (p.wcnt) p.wcnt[blockIdx.x * kConsW + warp] = (int32_t)(mm < kTailY ? mm : kTailY);
          }
        }
      }
      if (compact) in_scratch = true;
    } else if (c.phase == PH_SNAP) {
      mode = 2;
      acc[0] = -HUGE_VAL;
      ops[0] = OP_MAX;
      if (prod_lane) produce<1, kStagesY, kTileY, kTileY>(wsrc, work, pp, spec);
      else if (!producer) t_spx<L1, 2>(p, c, fix, work, m_w, false, pp, acc);
    } else {
      break;
    }
    double a4[4] = {acc[0], acc[1], acc[2], acc[3]};
    block_reduce<4, kConsW>(a4, ops, s_red, s_tot);  // (its barrier orders the atomicMax above)
    if (mode == 1 && c.hist && p.hist) {
      // this CTA's nonzero counts into the global histogram (integer atomics:
      // order-independent); each CTA starts at its own offset so the 148
      // CTAs' atomics on a dense histogram do not queue on the same address
      const int rot = (int)((blockIdx.x * 7u) % kHistB);
      for (int i = threadIdx.x; i < kHistB; i += blockDim.x) {
        const int k = (i + rot) & (kHistB - 1);
        if (s_hist[k]) atomicAdd(&p.hist[k], s_hist[k]);
      }
    }
    const bool is_master = grid_step_any<4>(p.ar, p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch, [&] {
      if (prod_lane) {
        if ((mode == 1 && fix && c.compact) || mode == 3) {  // nobody else reads s_nslots before the next epoch
          s_nslots = s_nsl_new;
          s_nsl_new = 0;
        }
        speculate();
      }
    }, (c_tma_flags & 4) != 0);
    if (is_master && mode == 1 && c.hist && p.hist) hist_bound(p, c.lam, s_st.r, s_hist, s_st);
    double glob[4];
    bool xok = true;
    if (is_master && warp == 0) {  // the whole warp: the exchange is warp-level
      if (lane == 0) tl_record(dsync, epoch, c.phase, (mode == 0 || mode >= 3) ? p.n : s_st.phys_count, s_st.cmd.compact);
      xok = exchange_totals<4>(p.ex, epoch, ops, s_tot, glob, master);
    }
    if (threadIdx.x == 0) {
      if (is_master) {
        double loc[4] = {s_tot[0], s_tot[1], s_tot[2], s_tot[3]};
        if (!xok) {
          raise_timeout(p.sync);
          s_st.status = ST_TIMEOUT;
          s_st.cmd.phase = PH_DONE;
        } else if (mode == 4) s_after_sample(s_st, glob, loc[2]);
        else if (mode == 3) s_after_fused(s_st, glob, loc);
        else if (mode == 0) s_after_init(s_st, glob);
        else if (mode == 1) s_after_scan(s_st, glob, loc, dtrace);
        else s_after_snap(s_st, glob);
        const int ph = s_st.cmd.phase;
        s_tail = p.wcnt && p.ex.world <= 1 && gridDim.x <= kMaxGridY && (ph == PH_SCAN || ph == PH_SNAP) &&
                 s_st.phys_count <= kTailY && (in_scratch || p.n <= kTailY);
        if (!s_tail) {
          if (master && (ph == PH_FINAL || ph == PH_DONE || ph == PH_COPY)) publish_state(p.out, s_st, p.sync);
          s_cmd = s_st.cmd;
          if (!single) master_release(p.sync, s_gen0 + epoch, s_st.cmd, &p.st->cmd);
          if (master) tl_mark(p.sync, epoch, 5);
        } else if (!master) {  // single-GPU: the master finishes alone, then releases once
          s_tail = 0;
          if (!wait_release(p.sync, s_gen0 + 1, &p.st->cmd, &s_cmd)) s_abort = 1;
        }
      } else if (!s_abort) {
        if (!wait_release(p.sync, s_gen0 + epoch, &p.st->cmd, &s_cmd)) s_abort = 1;
        if (blockIdx.x == 1) tl_mark(p.sync, epoch, 7);
      }
    }
    __syncthreads();
    if (master && s_tail) {  // uniform in the master CTA; the other CTAs wait for the release
      if (!producer) drain<kStagesY>(pp, s_spec);  // the stage memory becomes the tail set
      __syncthreads();
      if (threadIdx.x == 0) tl_mark(p.sync, epoch, 14);
      double* V = reinterpret_cast<double*>(s_dyn);
      const int m = tail_gather<L1>(p, in_scratch, V, s_scan);
      if (threadIdx.x == 0) tl_mark(p.sync, epoch, 15);
      for (unsigned it = 1;; ++it) {
        const Cmd tc = s_st.cmd;
        if (tc.phase != PH_SCAN && tc.phase != PH_SNAP) break;
        const bool scan = tc.phase == PH_SCAN;
        const double lam = tc.lam, fhi = tc.fix_hi;
        double a3[3] = {scan ? 0.0 : -HUGE_VAL, 0.0, 0.0};
        int n0 = 0, n1 = 0;
        // contiguous runs per thread (>= 2: tiny sets sum pairwise-sequentially,
        // as the tiled passes do), then the fixed-order block reduction
        const int per = max(2, (m + (int)blockDim.x - 1) / (int)blockDim.x);
        const int i0 = min(m, (int)threadIdx.x * per), i1 = min(m, i0 + per);
        for (int i = i0; i < i1; ++i) {
          const double w = V[i];
          const double v = add_rn(w, lam);
          const bool kp = !(fix && !(v > 0.0) && !(add_rn(w, fhi) > 0.0));
          if (scan) {
            a3[0] += (kp && v > 0.0) ? v : 0.0;
            n0 += kp && v > 0.0;
            n1 += kp && v == 0.0;
          } else {
            a3[0] = kp ? fmax(a3[0], -w) : a3[0];
            n0 += kp;
          }
        }
        a3[1] = (double)n0;
        a3[2] = (double)n1;
        int tops[3] = {scan ? OP_SUM : OP_MAX, OP_SUM, OP_SUM};
        block_reduce<3>(a3, tops, s_red, s_tot);  // all 16 warps hold tail elements
        if (threadIdx.x == 0) {
          tl_record(p.sync, epoch + it, tc.phase, m, 0);
          if (scan) s_after_scan(s_st, s_tot, s_tot, p.trace);
          else s_after_snap(s_st, s_tot);
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        const int ph = s_st.cmd.phase;
        if (ph == PH_FINAL || ph == PH_DONE || ph == PH_COPY) publish_state(p.out, s_st, p.sync);
        s_cmd = s_st.cmd;
        s_spec = 0;
        s_tail = 0;
        master_release(p.sync, single ? s_gen0 + 1 : s_gen0 + epoch, s_st.cmd, &p.st->cmd);
        tl_mark(p.sync, epoch, 5);
      }
      __syncthreads();
    }
  }
}

inline int64_t tma_scratch_elems_y(int64_t n) { return (n + kTileY - 1) / kTileY * kTileY; }

}  // namespace cqk

// cqk_kernels.cuh -- the persistent CQK and simplex/l1 kernels and the
// batched row-wise simplex kernel (sm_100a, fp64 / fp32).
#pragma once
#include "cqk_solver.cuh"

namespace cqk {

// ------------------------------------------------------------ chunk loads
// A warp streams its segment in chunks of 32 * VN * UNR elements; lane `ln`
// owns elements base + u*32*VN + ln*VN + v.  Full chunks use 16-byte vector
// loads; the ragged tail uses guarded scalar loads with a neutral fill.
constexpr int kUnroll = 2;

constexpr int kUnrollY = 8;  // single-array passes: 8 x 16 B in flight per lane

template <typename T, bool SCRATCH, int UNR = kUnroll>
DEVI void load_chunk(const T* p, int64_t base, int64_t m, int lane, bool full, T fill,
                     T (&out)[Vec<T>::n * UNR]) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n;
  if (full) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const V* q = reinterpret_cast<const V*>(p + base + (int64_t)u * 32 * VN + lane * VN);
      V v = SCRATCH ? ld_scratch(q) : ld_stream(q);
      unpack<V, T>(v, &out[u * VN]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < VN * UNR; ++j) {
      const int64_t e = base + (int64_t)(j / VN) * 32 * VN + lane * VN + (j % VN);
      out[j] = e < m ? (SCRATCH ? ld_scratch(p + e) : ld_stream(p + e)) : fill;
    }
  }
}

// Memory-level parallelism without registers: each warp keeps c_prefetch[0]
// chunks of every streamed array in flight into L2 with bulk prefetches
// (cp.async.bulk.prefetch.L2, one instruction per array-chunk, issued by
// distinct lanes), so the vector loads of a chunk mostly hit L2.
// [0]: chunks ahead for the 3..5-array CQK passes, [1]: for the single-array
// simplex / l1 passes (set per launch by the ABI; CQK_PREFETCH env override).
__constant__ int c_prefetch[2];

DEVI void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Prefetch chunks [c0, c0 + nchunk) of NARR arrays (chunk = CH elements of T)
// of a segment of m elements; lane k handles (array k % NARR, chunk k / NARR).
template <typename T, int NARR, int UNR = kUnroll>
DEVI void prefetch_chunks(const T* const (&arr)[NARR], int64_t c0, int nchunk, int64_t m,
                          int lane) {
  constexpr int CH = 32 * Vec<T>::n * UNR;
  if (nchunk > 0 && lane < NARR * nchunk) {
    const int64_t e = (c0 + lane / NARR) * CH;
    if (e < m) {
      const int64_t cnt = m - e < CH ? m - e : CH;
      const unsigned bytes = (unsigned)(cnt * sizeof(T)) & ~15u;
      if (bytes) bulk_prefetch_l2(arr[lane % NARR] + e, bytes);
    }
  }
}

template <typename T, int UNR = kUnroll>
DEVI int64_t chunk_index(int64_t base, int lane, int j) {
  constexpr int VN = Vec<T>::n;
  return base + (int64_t)(j / VN) * 32 * VN + lane * VN + (j % VN);
}

DEVI void store_out(double2* p, double2 v) { __stcs(p, v); }
DEVI void store_out(float4* p, float4 v) { __stcs(p, v); }

// Word-wise L2 (coherent) copy of master-owned structures.
template <typename S>
DEVI void load_l2(S* dst, const S* src) {
  static_assert(sizeof(S) % 8 == 0, "8-byte multiple");
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(dst);
#pragma unroll 4
  for (int i = 0; i < (int)(sizeof(S) / 8); ++i) d[i] = __ldcg(s + i);
}

// The master's final state goes straight to mapped (pinned) host memory: the
// host reads it after the stream synchronises -- no device-to-host copy is
// queued behind the kernel.  The grid's barrier-timeout flag rides along.
template <typename S>
DEVI void publish_state(S* out, S& st, const GridSync& sy) {
  st.err = *(volatile int*)sy.error;
  *out = st;
}

// ------------------------------------------------------------ barrier
// Fixed-master grid step: CTA 0 owns the solver state in shared memory for
// the whole kernel.  Every CTA publishes partials[blockIdx.x][0..K) and
// arrives; CTA 0 waits for all arrivals, reduces the rows in a fixed order
// into s_tot (deterministic, no float atomics) and returns true; the caller
// then runs the state machine and master_release()s the others, which wait
// in wait_release() and pick up the new command with one L2 round trip.
template <int K>
DEVI bool grid_step(double* partials, const double* s_cta, const int (&ops)[K],
                    const GridSync& sy, double (*s_red)[kMaxK], double* s_tot, int* s_abort,
                    unsigned epoch) {
  if (threadIdx.x < K) partials[(int64_t)blockIdx.x * kMaxK + threadIdx.x] = s_cta[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 1) tl_mark(sy, epoch, 6);
  if (threadIdx.x == 0) {
    // release-add: the CTA's partial row (ordered before by bar.sync) is
    // visible to the master's acquire -- cheaper than fence.sc + atomic
    unsigned prev;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(sy.arrive)
                 : "memory");
    if (prev == gridDim.x - 1) tl_last(sy, epoch, blockIdx.x);
  }
  if (blockIdx.x != 0) return false;
  // The whole master CTA reduces: thread 0 spins on the arrival count (timer
  // checked every 256 polls -- reading %globaltimer is not free); then
  // thread t folds rows t, t+blockDim, ... (one L2 round trip: K loads of one
  // 128-byte row each), warps combine with xor butterflies and warp 0 takes
  // the warp totals in order -- a fixed order, no float atomics.
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    unsigned polls = 0;
    while (ld_relaxed(sy.arrive) < gridDim.x) {  // relaxed polls, one acquire fence
      if ((++polls & 255u) == 0 && globaltimer() - t0 > kSpinTimeoutNs) {
        raise_timeout(sy);
        *s_abort = 1;
        break;
      }
    }
    fence_acquire_gpu();
    if (!*s_abort) *sy.arrive = 0u;  // nobody arrives again before the release
    tl_mark(sy, epoch, 4);
  }
  __syncthreads();
  if (*(volatile int*)s_abort) return false;
  if (threadIdx.x == 0) tl_mark(sy, epoch, 16);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = ops[k] == OP_SUM ? 0.0 : ops[k] == OP_MIN ? HUGE_VAL : -HUGE_VAL;
  for (int c = threadIdx.x; c < (int)gridDim.x; c += blockDim.x) {
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __ldcg(partials + (int64_t)c * kMaxK + k);
#pragma unroll
    for (int k = 0; k < K; ++k)
      acc[k] = ops[k] == OP_SUM ? acc[k] + v[k] : ops[k] == OP_MIN ? fmin(acc[k], v[k]) : fmax(acc[k], v[k]);
  }
  if (threadIdx.x == 0) tl_mark(sy, epoch, 17);
  // only the warps that hold rows combine (identities elsewhere; this also
  // keeps a TMA producer warp out of the shuffles, see block_reduce)
  const int nw = min((int)(blockDim.x >> 5), (int)((gridDim.x + 31) >> 5));
  if (warp < nw) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double v = ops[k] == OP_SUM ? warp_sum(acc[k]) : ops[k] == OP_MIN ? warp_min(acc[k])
                                                                             : warp_max(acc[k]);
      if (lane == 0) s_red[warp][k] = v;
    }
  }
  if (threadIdx.x == 0) tl_mark(sy, epoch, 18);
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    double v = s_red[0][k];
    for (int w = 1; w < nw; ++w) {
      const double o = s_red[w][k];
      v = ops[k] == OP_SUM ? v + o : ops[k] == OP_MIN ? fmin(v, o) : fmax(v, o);
    }
    s_tot[k] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) tl_mark(sy, epoch, 19);
  return !*(volatile int*)s_abort;
}

// Single GPU (grid_step_any with GridAR rows): every CTA publishes its
// partial row with a tagged release store (ar_arrive), then combines all rows
// itself in the same fixed order as grid_step's master -- bit-identical
// totals -- (ar_combine): thread c acquires row c's tag and reads its values,
// so the wait and the load are one round trip per row and no arrival counter
// is contended.  Every CTA then runs the deterministic state machine on its
// own replica of the state: no release round trip.  ar_combine returns false
// (s_abort set) on a spin timeout.
template <int K>
DEVI constexpr int ar_tag_slot() { return K < kMaxK ? kMaxK - 1 : kMaxK; }

template <int K>
DEVI void ar_arrive(const GridAR& ar, const double* s_cta, const GridSync& sy, unsigned epoch) {
  static_assert(K <= kMaxK && kMaxK < kArStride, "row layout");
  if (threadIdx.x == 0) {
    const int G = (int)gridDim.x;
    double* row = ar.rows + ((size_t)(epoch & 1u) * G + blockIdx.x) * kArStride;
#pragma unroll
    for (int k = 0; k < K; ++k) row[k] = s_cta[k];
    // release: the values above are visible to whoever acquires the tag
    st_release_gpu_u64(reinterpret_cast<unsigned long long*>(row + ar_tag_slot<K>()), ar.tag | epoch);
    if (blockIdx.x == 1) tl_mark(sy, epoch, 6);
  }
}

template <int K>
DEVI bool ar_combine(const GridAR& ar, const int (&ops)[K], const GridSync& sy,
                     double (*s_red)[kMaxK], double* s_tot, int* s_abort, unsigned epoch) {
  const int G = (int)gridDim.x;
  const double* rows = ar.rows + (size_t)(epoch & 1u) * G * kArStride;
  const unsigned long long want = ar.tag | epoch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = ops[k] == OP_SUM ? 0.0 : ops[k] == OP_MIN ? HUGE_VAL : -HUGE_VAL;
  bool late = false;
  for (int c = threadIdx.x; c < G; c += blockDim.x) {
    const double* row = rows + (int64_t)c * kArStride;
    const unsigned long long* tag = reinterpret_cast<const unsigned long long*>(row + ar_tag_slot<K>());
    if (ld_acquire_gpu_u64(tag) != want) {
      const unsigned long long t0 = globaltimer();
      unsigned polls = 0;
      while (ld_acquire_gpu_u64(tag) != want) {
        if ((++polls & 255u) == 0 && globaltimer() - t0 > kSpinTimeoutNs) {
          late = true;
          break;
        }
      }
    }
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __ldcg(row + k);
#pragma unroll
    for (int k = 0; k < K; ++k)
      acc[k] = ops[k] == OP_SUM ? acc[k] + v[k] : ops[k] == OP_MIN ? fmin(acc[k], v[k]) : fmax(acc[k], v[k]);
  }
  if (__syncthreads_or(late)) {
    if (threadIdx.x == 0) {
      raise_timeout(sy);
      *s_abort = 1;
    }
    __syncthreads();
    return false;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) tl_mark(sy, epoch, 4);
  const int nw = min((int)(blockDim.x >> 5), (G + 31) >> 5);
  if (warp < nw) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double v = ops[k] == OP_SUM ? warp_sum(acc[k]) : ops[k] == OP_MIN ? warp_min(acc[k])
                                                                             : warp_max(acc[k]);
      if (lane == 0) s_red[warp][k] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    double v = s_red[0][k];
    for (int w = 1; w < nw; ++w) {
      const double o = s_red[w][k];
      v = ops[k] == OP_SUM ? v + o : ops[k] == OP_MIN ? fmin(v, o) : fmax(v, o);
    }
    s_tot[k] = v;
  }
  __syncthreads();
  return true;
}

// The grid step of either design; true = this CTA runs the decision (every
// CTA single-GPU, the master otherwise).
// `overlap` (the producer lane's next-pass speculation) runs once this CTA
// has arrived when masterless, before the arrival otherwise.
template <int K, class F>
DEVI bool grid_step_any(const GridAR& ar, double* partials, const double* s_cta, const int (&ops)[K],
                        const GridSync& sy, double (*s_red)[kMaxK], double* s_tot, int* s_abort,
                        unsigned epoch, F&& overlap, bool late = false) {
  if (ar.rows) {
    ar_arrive<K>(ar, s_cta, sy, epoch);
    if (!late) overlap();
    const bool ok = ar_combine<K>(ar, ops, sy, s_red, s_tot, s_abort, epoch);
    if (late) overlap();
    return ok;
  }
  overlap();
  return grid_step<K>(partials, s_cta, ops, sy, s_red, s_tot, s_abort, epoch);
}

// Master (CTA 0, thread 0): publish the next command and release the grid.
DEVI void master_release(const GridSync& sy, unsigned target, const Cmd& cmd, Cmd* gcmd) {
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(&cmd);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(gcmd);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Cmd) / 8); ++i) __stcg(d + i, s[i]);
  st_release(sy.gen, target);  // release orders the command (and state) stores
}

// Non-master CTAs (thread 0): wait for the release, then fetch the command.
DEVI bool wait_release(const GridSync& sy, unsigned target, const Cmd* gcmd, Cmd* out) {
  const unsigned long long t0 = globaltimer();
  unsigned polls = 0;
  while ((int)(ld_relaxed(sy.gen) - target) < 0) {
    if ((++polls & 255u) == 0 && globaltimer() - t0 > kSpinTimeoutNs) {
      raise_timeout(sy);
      return false;
    }
  }
  fence_acquire_gpu();
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(gcmd);
  unsigned long long w[sizeof(Cmd) / 8];
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Cmd) / 8); ++i) w[i] = __ldcg(s + i);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(out);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Cmd) / 8); ++i) d[i] = w[i];
  return true;
}

// ------------------------------------------------------------ CQK passes
// pass 0: lambda0 sums (core.py:237-257) fused with validate (core.py:126-165)
template <typename T, bool CHECK, bool XBAR>
DEVI void lambda0_pass(const CqkParams<T>& p, int64_t seg_lo, int64_t m, double (&acc)[kMaxK]) {
  constexpr int E = Vec<T>::n * kUnroll, CH = 32 * E;
  const int lane = threadIdx.x & 31;
  const T* const pf[5] = {p.d + seg_lo, p.a + seg_lo, p.b + seg_lo, p.l + seg_lo, p.u + seg_lo};
  const T* const pf3[3] = {pf[0], pf[1], pf[2]};
  if (XBAR) prefetch_chunks<T, 5>(pf, 0, c_prefetch[0], m, lane);
  else prefetch_chunks<T, 3>(pf3, 0, c_prefetch[0], m, lane);
  for (int64_t base = 0; base < m; base += CH) {
    if (XBAR) prefetch_chunks<T, 5>(pf, base / CH + c_prefetch[0], c_prefetch[0] > 0 ? 1 : 0, m, lane);
    else prefetch_chunks<T, 3>(pf3, base / CH + c_prefetch[0], c_prefetch[0] > 0 ? 1 : 0, m, lane);
    const bool full = base + CH <= m;
    T D[E], A[E], B[E], L[E], U[E], X[E];
    load_chunk<T, false>(p.d + seg_lo, base, m, lane, full, T(1), D);
    load_chunk<T, false>(p.a + seg_lo, base, m, lane, full, T(0), A);
    load_chunk<T, false>(p.b + seg_lo, base, m, lane, full, T(1), B);
    if (XBAR) {  // l, u are otherwise validated during the first scan
      load_chunk<T, false>(p.l + seg_lo, base, m, lane, full, T(0), L);
      load_chunk<T, false>(p.u + seg_lo, base, m, lane, full, T(0), U);
    }
    if (XBAR) load_chunk<T, false>(p.xbar + seg_lo, base, m, lane, full, T(0), X);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int64_t e = chunk_index<T>(base, lane, j);
      if (!full && e >= m) continue;
      const T y = rcp_nr(D[j]);
      const double s = (double)mul_rn(B[j], A[j] * y);
      const double q = (double)mul_rn(B[j], B[j] * y);
      acc[0] += s;
      acc[1] += q;
      if (XBAR && L[j] < X[j] && X[j] < U[j]) { acc[2] += s; acc[3] += q; acc[4] += 1.0; }
      if (CHECK) {
        const double gi = (double)(p.offset + seg_lo + e);
        const T d = D[j], a = A[j], b = B[j], l = L[j], u = U[j];
        if (!isfinite((double)d)) acc[5] = fmin(acc[5], gi);
        if (!isfinite((double)a)) acc[6] = fmin(acc[6], gi);
        if (!isfinite((double)b)) acc[7] = fmin(acc[7], gi);
        if (!(d > T(0))) acc[10] = fmin(acc[10], gi);
        if (!(b > T(0))) acc[11] = fmin(acc[11], gi);
        if (XBAR) {
          if (isnan((double)l)) acc[8] = fmin(acc[8], gi);
          if (isnan((double)u)) acc[9] = fmin(acc[9], gi);
          if (!(l <= u)) acc[12] = fmin(acc[12], gi);
          if ((double)l == HUGE_VAL) acc[13] = fmin(acc[13], gi);
          if ((double)u == -HUGE_VAL) acc[14] = fmin(acc[14], gi);
        }
      }
    }
  }
}

// validate()'s l / u checks on the first scan: segment-local first index per
// check in 32-bit registers (cheap in the register-tight scan loop), turned
// into global double indices in slots 11..15 after the loop.
constexpr int kCheckLuSlot = 11;  // slots 11..15: l NaN, u NaN, l<=u, l!=+inf, u!=-inf
template <typename T>
DEVI void check_lu(T l, T u, unsigned li, unsigned (&first)[5]) {
  if (isnan((double)l)) first[0] = min(first[0], li);
  if (isnan((double)u)) first[1] = min(first[1], li);
  if (!(l <= u)) first[2] = min(first[2], li);
  if ((double)l == HUGE_VAL) first[3] = min(first[3], li);
  if ((double)u == -HUGE_VAL) first[4] = min(first[4], li);
}

template <typename T, bool FIX, bool SRC_SCRATCH, bool CHK = false>
DEVI void scan_pass(const CqkParams<T>& p, const Cmd& c, int64_t seg_lo, int64_t& m,
                    bool compact, double (&acc)[kMaxK]) {
  constexpr int E = Vec<T>::n * kUnroll, CH = 32 * E;
  const int lane = threadIdx.x & 31;
  const T* sd = (SRC_SCRATCH ? p.sd : p.d) + seg_lo;
  const T* sa = (SRC_SCRATCH ? p.sa : p.a) + seg_lo;
  const T* sb = (SRC_SCRATCH ? p.sb : p.b) + seg_lo;
  const T* sl = (SRC_SCRATCH ? p.sl : p.l) + seg_lo;
  const T* su = (SRC_SCRATCH ? p.su : p.u) + seg_lo;
  const T lam = (T)c.lam, fhi = (T)c.fix_hi, flo = (T)c.fix_lo;
  const bool chk_lo = FIX && isfinite(c.fix_hi), chk_hi = FIX && isfinite(c.fix_lo);
  const unsigned lt = (1u << lane) - 1u;
  const T* const pf[5] = {sd, sa, sb, sl, su};
  prefetch_chunks<T, 5>(pf, 0, c_prefetch[0], m, lane);
  unsigned first[5] = {~0u, ~0u, ~0u, ~0u, ~0u};
  int64_t out_m = 0;
  for (int64_t base = 0; base < m; base += CH) {
    prefetch_chunks<T, 5>(pf, base / CH + c_prefetch[0], c_prefetch[0] > 0 ? 1 : 0, m, lane);
    const bool full = base + CH <= m;
    T D[E], A[E], B[E], L[E], U[E];
    load_chunk<T, SRC_SCRATCH>(sd, base, m, lane, full, T(1), D);
    load_chunk<T, SRC_SCRATCH>(sa, base, m, lane, full, T(0), A);
    load_chunk<T, SRC_SCRATCH>(sb, base, m, lane, full, T(1), B);
    load_chunk<T, SRC_SCRATCH>(sl, base, m, lane, full, T(0), L);
    load_chunk<T, SRC_SCRATCH>(su, base, m, lane, full, T(0), U);
    bool keep[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const bool valid = full || chunk_index<T>(base, lane, j) < m;
      if (CHK && valid) check_lu<T>(L[j], U[j], (unsigned)chunk_index<T>(base, lane, j), first);
      keep[j] = valid && elem_scan<T, FIX>(D[j], A[j], B[j], L[j], U[j], lam, fhi, flo, chk_lo,
                                           chk_hi, acc);
    }
    if (FIX && compact) {
      // warp-ballot stream compaction into this warp's own scratch range;
      // write positions never overtake the read front (in-place safe).
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const unsigned mask = __ballot_sync(0xffffffffu, keep[j]);
        if (keep[j]) {
          const int64_t pos = seg_lo + out_m + __popc(mask & lt);
          p.sd[pos] = D[j]; p.sa[pos] = A[j]; p.sb[pos] = B[j]; p.sl[pos] = L[j]; p.su[pos] = U[j];
        }
        out_m += __popc(mask);
      }
    }
  }
  if (FIX && compact) m = out_m;
  if (CHK) {
#pragma unroll
    for (int k = 0; k < 5; ++k)
      if (first[k] != ~0u) acc[kCheckLuSlot + k] = (double)(p.offset + seg_lo + (int64_t)first[k]);
  }
}

template <typename T, bool SRC_SCRATCH>
DEVI void bp_pass(const CqkParams<T>& p, const Cmd& c, bool fix, int64_t seg_lo, int64_t m,
                  double (&acc)[kMaxK]) {
  constexpr int E = Vec<T>::n * kUnroll, CH = 32 * E;
  const int lane = threadIdx.x & 31;
  const T* sd = (SRC_SCRATCH ? p.sd : p.d) + seg_lo;
  const T* sa = (SRC_SCRATCH ? p.sa : p.a) + seg_lo;
  const T* sb = (SRC_SCRATCH ? p.sb : p.b) + seg_lo;
  const T* sl = (SRC_SCRATCH ? p.sl : p.l) + seg_lo;
  const T* su = (SRC_SCRATCH ? p.su : p.u) + seg_lo;
  const T lam = (T)c.lam, fhi = (T)c.fix_hi, flo = (T)c.fix_lo;
  const bool right = c.right != 0;
  const T* const pf[5] = {sd, sa, sb, sl, su};
  prefetch_chunks<T, 5>(pf, 0, c_prefetch[0], m, lane);
  for (int64_t base = 0; base < m; base += CH) {
    prefetch_chunks<T, 5>(pf, base / CH + c_prefetch[0], c_prefetch[0] > 0 ? 1 : 0, m, lane);
    const bool full = base + CH <= m;
    T D[E], A[E], B[E], L[E], U[E];
    load_chunk<T, SRC_SCRATCH>(sd, base, m, lane, full, T(1), D);
    load_chunk<T, SRC_SCRATCH>(sa, base, m, lane, full, T(0), A);
    load_chunk<T, SRC_SCRATCH>(sb, base, m, lane, full, T(1), B);
    load_chunk<T, SRC_SCRATCH>(sl, base, m, lane, full, T(0), L);
    load_chunk<T, SRC_SCRATCH>(su, base, m, lane, full, T(0), U);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (!full && chunk_index<T>(base, lane, j) >= m) continue;
      if (fix) {  // only the logically active set takes part
        const T yd = rcp_div(D[j]);
        const T t = t_of_y(D[j], A[j], B[j], lam, yd);
        if (isfinite(c.fix_hi) && t <= L[j] && t_of_y(D[j], A[j], B[j], fhi, yd) <= L[j]) continue;
        if (isfinite(c.fix_lo) && t >= U[j] && t_of_y(D[j], A[j], B[j], flo, yd) >= U[j]) continue;
      }
      elem_bp<T>(D[j], A[j], B[j], L[j], U[j], c.edge, right, acc[0], acc[1]);
    }
  }
}

template <typename T, bool FIX>
DEVI void final_pass(const CqkParams<T>& p, const Cmd& c, int64_t seg_lo, int64_t m) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n, E = VN * kUnroll, CH = 32 * E;
  const int lane = threadIdx.x & 31;
  const T lam = (T)c.lam, fhi = (T)c.fix_hi, flo = (T)c.fix_lo;
  // fixed variables need an explicit test only if lam* left the side of the
  // fixing multiplier (the criterion-2 finish(lam + step) edge)
  const bool chk_lo = FIX && c.lam > c.fix_hi, chk_hi = FIX && c.lam < c.fix_lo;
  T* x = p.x + seg_lo;
  const T* const pf[5] = {p.d + seg_lo, p.a + seg_lo, p.b + seg_lo, p.l + seg_lo, p.u + seg_lo};
  prefetch_chunks<T, 5>(pf, 0, c_prefetch[0], m, lane);
  for (int64_t base = 0; base < m; base += CH) {
    prefetch_chunks<T, 5>(pf, base / CH + c_prefetch[0], c_prefetch[0] > 0 ? 1 : 0, m, lane);
    const bool full = base + CH <= m;
    T D[E], A[E], B[E], L[E], U[E];
    load_chunk<T, false>(p.d + seg_lo, base, m, lane, full, T(1), D);
    load_chunk<T, false>(p.a + seg_lo, base, m, lane, full, T(0), A);
    load_chunk<T, false>(p.b + seg_lo, base, m, lane, full, T(1), B);
    load_chunk<T, false>(p.l + seg_lo, base, m, lane, full, T(0), L);
    load_chunk<T, false>(p.u + seg_lo, base, m, lane, full, T(0), U);
    T X[E];
#pragma unroll
    for (int j = 0; j < E; ++j)
      X[j] = elem_final<T, FIX>(D[j], A[j], B[j], L[j], U[j], lam, fhi, flo, chk_lo, chk_hi);
    if (full) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        V v;
        T* vv = reinterpret_cast<T*>(&v);
#pragma unroll
        for (int q = 0; q < VN; ++q) vv[q] = X[u * VN + q];
        store_out(reinterpret_cast<V*>(x + base + (int64_t)u * 32 * VN + lane * VN), v);
      }
    } else {
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const int64_t e = chunk_index<T>(base, lane, j);
        if (e < m) x[e] = X[j];
      }
    }
  }
}

// ------------------------------------------------------------ CQK kernel
template <typename T, bool FIX>
__global__ void __launch_bounds__(kThreads, 1) cqk_solve_kernel(CqkParams<T> p) {
  __shared__ double s_red[kWarps][kMaxK];
  __shared__ double s_tot[kMaxK];
  __shared__ Cmd s_cmd;
  __shared__ CqkState s_st;  // master (CTA 0) only
  __shared__ unsigned s_gen0;
  __shared__ int s_abort;
  const int warp = threadIdx.x >> 5;
  const bool master = blockIdx.x == 0;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp, W = (int64_t)gridDim.x * kWarps;
  int64_t seg_lo, seg_hi;
  warp_segment(p.n, gw, W, seg_lo, seg_hi);
  int64_t m = seg_hi - seg_lo;  // this warp's physical working-set size
  bool in_scratch = false;
  if (threadIdx.x == 0) {
    s_gen0 = ld_acquire(p.sync.gen);
    s_abort = 0;
    if (master) {
      s_st = p.init;  // host-initialised, passed by value
      s_cmd = s_st.cmd;
      tl_record(p.sync, 0, -1, p.n, 0);
    } else {
      s_cmd = p.init.cmd;
    }
  }
  __syncthreads();
  const int has_xbar = p.xbar != nullptr;
  const int check = p.init.check;  // immutable during the solve
  for (unsigned epoch = 1;; ++epoch) {
    const Cmd c = s_cmd;
    if (c.phase == PH_DONE || s_abort) break;
    if (c.phase == PH_FINAL) {
      if (p.x) final_pass<T, FIX>(p, c, seg_lo, seg_hi - seg_lo);
      break;
    }
    double acc[kMaxK];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) acc[k] = 0.0;
    bool is_master = false;
    if (c.phase == PH_LAMBDA0) {
#pragma unroll
      for (int k = kValidateSlot; k < kValidateSlot + 10; ++k) acc[k] = HUGE_VAL;
      const int64_t m0 = seg_hi - seg_lo;
      if (check && has_xbar) lambda0_pass<T, true, true>(p, seg_lo, m0, acc);
      else if (check) lambda0_pass<T, true, false>(p, seg_lo, m0, acc);
      else if (has_xbar) lambda0_pass<T, false, true>(p, seg_lo, m0, acc);
      else lambda0_pass<T, false, false>(p, seg_lo, m0, acc);
      const int ops[15] = {OP_SUM, OP_SUM, OP_SUM, OP_SUM, OP_SUM, OP_MIN, OP_MIN, OP_MIN,
                           OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN};
      double a15[15];
#pragma unroll
      for (int k = 0; k < 15; ++k) a15[k] = acc[k];
      block_reduce<15>(a15, ops, s_red, s_tot);
      is_master = grid_step<15>(p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch);
      if (is_master && threadIdx.x == 0) {
        tl_record(p.sync, epoch, PH_LAMBDA0, p.n, 0);
        double glob[15];
        if (exchange_totals_1(p.ex, epoch, 15, ops, s_tot, glob)) m_after_lambda0(s_st, glob);
        else {
          m_stop(s_st, ST_TIMEOUT);
          raise_timeout(p.sync);
        }
      }
    } else if (c.phase == PH_SCAN && c.check_lu) {
      // first scan (original arrays, never compacting) with validate()'s l / u checks
#pragma unroll
      for (int k = kCheckLuSlot; k < kMaxK; ++k) acc[k] = HUGE_VAL;
      scan_pass<T, FIX, false, true>(p, c, seg_lo, m, false, acc);
      int ops[kMaxK];
#pragma unroll
      for (int k = 0; k < kMaxK; ++k) ops[k] = k < kCheckLuSlot ? OP_SUM : OP_MIN;
      block_reduce<kMaxK>(acc, ops, s_red, s_tot);
      is_master = grid_step<kMaxK>(p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch);
      if (is_master && threadIdx.x == 0) {
        double loc[kMaxK], glob[kMaxK];
#pragma unroll
        for (int k = 0; k < kMaxK; ++k) loc[k] = s_tot[k];
        tl_record(p.sync, epoch, PH_SCAN, s_st.phys_count, 0);
        if (!exchange_totals_1(p.ex, epoch, kMaxK, ops, loc, glob)) {
          m_stop(s_st, ST_TIMEOUT);
          raise_timeout(p.sync);
        } else {
          s_st.cmd.check_lu = 0;
          s_st.vidx[3] = glob[11];  // l NaN
          s_st.vidx[4] = glob[12];  // u NaN
          s_st.vidx[7] = glob[13];  // l <= u
          s_st.vidx[8] = glob[14];  // l == +inf
          s_st.vidx[9] = glob[15];  // u == -inf
          if (m_validate(s_st, 3, 10)) m_after_scan(s_st, glob, loc, p.trace);
        }
      }
    } else if (c.phase == PH_SCAN) {
      const bool compact = FIX && c.compact;
      if (in_scratch) scan_pass<T, FIX, true>(p, c, seg_lo, m, compact, acc);
      else scan_pass<T, FIX, false>(p, c, seg_lo, m, compact, acc);
      if (compact) in_scratch = true;
      constexpr int K = FIX ? 11 : 5;
      int ops[K];
      double aK[K];
#pragma unroll
      for (int k = 0; k < K; ++k) { ops[k] = OP_SUM; aK[k] = acc[k]; }
      block_reduce<K>(aK, ops, s_red, s_tot);
      is_master = grid_step<K>(p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch);
      if (is_master && threadIdx.x == 0) {
        double loc[11], glob[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) loc[k] = glob[k] = k < K ? s_tot[k] : 0.0;
        tl_record(p.sync, epoch, PH_SCAN, s_st.phys_count, s_st.cmd.compact);
        if (exchange_totals_1(p.ex, epoch, K, ops, loc, glob)) m_after_scan(s_st, glob, loc, p.trace);
        else {
          m_stop(s_st, ST_TIMEOUT);
          raise_timeout(p.sync);
        }
      }
    } else if (c.phase == PH_BP) {
      acc[0] = c.right ? HUGE_VAL : -HUGE_VAL;
      if (in_scratch) bp_pass<T, true>(p, c, FIX, seg_lo, m, acc);
      else bp_pass<T, false>(p, c, FIX, seg_lo, m, acc);
      int ops[2] = {c.right ? OP_MIN : OP_MAX, OP_SUM};
      double a2[2] = {acc[0], acc[1]};
      block_reduce<2>(a2, ops, s_red, s_tot);
      is_master = grid_step<2>(p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch);
      if (is_master && threadIdx.x == 0) {
        tl_record(p.sync, epoch, PH_BP, s_st.phys_count, 0);
        double glob[2];
        if (exchange_totals_1(p.ex, epoch, 2, ops, s_tot, glob)) m_after_bp(s_st, glob);
        else {
          m_stop(s_st, ST_TIMEOUT);
          raise_timeout(p.sync);
        }
      }
    } else {
      break;
    }
    if (threadIdx.x == 0) {
      if (is_master) {
        const int ph = s_st.cmd.phase;
        if (ph == PH_FINAL || ph == PH_DONE) publish_state(p.out, s_st, p.sync);  // results for the host
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

// ------------------------------------------------------------ simplex / l1
// newton_project_simplex (simplex.py:218-308) / project_l1 (simplex.py:311-333)
// with the formula start: one pass for sum/max (and the l1 inside-ball
// test), then phi passes over the free set, x = max(0, y + lam) (with the
// sign restored for l1).  Dropped variables are those with w + fix_hi <= 0.
struct SpxState {
  Cmd cmd;  // lam, fix_hi (drop iff w + fix_hi <= 0), phase, compact
  double lo, hi, r, tau, lam0, lam0_value;
  int64_t n, active, phys_count, pending_phys, fixed_count, fixed_removed;
  int64_t local_active, fixed_local;  // this rank's share (multi-GPU)
  int64_t iterations, phi_evals, max_iter, elems_scan, elems_written;
  int32_t fixing, status, l1, lam0_given, trace_len, trace_cap, start, hist_ok;
  int32_t err, fused;  // err: barrier-timeout flag at the final write; fused: capture start
  double compact_ratio;
  double lam_hist;  // start "auto": histogram upper bound of the root after the first scan (or NaN)
  int64_t cap_local;  // capture start: elements this rank captured (w >= cmd.edge)
  int32_t sparse_final;  // the captured list was adopted: x = signed zeros + a scatter
  int32_t cap_first;     // TMA engine: the first scan may capture (s_after_init)
};

template <typename T>
struct SpxParams {
  const T* y;
  T* sy;  // scratch (working values w)
  int64_t* sidx;      // capture start: the captured elements' indices (the fused pass's slots)
  uint32_t* signs;    // capture start, l1: y < 0 bits per (tile, warp, j) of the fused pass
  int64_t* out_idx;   // sparse output (output="sparse"): nonzero x as (index, value), any order,
  double* out_val;    // ... up to out_cap entries; out_cnt counts all of them
  unsigned long long* out_cnt;
  int64_t out_cap;
  T* x;
  double* trace;
  int64_t n;  // elements of this rank's shard
  SpxState* st;
  double* partials;
  GridSync sync;
  Exchange ex;
  int32_t* wcnt;  // [grid][consumer warps] scratch counts: enables the TMA kernel's tail mode
  int32_t* hist;       // [kHistB] bucket counts of the first scan (start "auto"); arrives zero
  int32_t* hist_next;  // the next launch's histogram, cleared by this one
  SpxState* out;  // mapped host memory: the final state for the host
  SpxState init;  // the host-initialised state, by value (no H2D copy)
  GridAR ar;      // single-GPU masterless grid step (rows null: master + release)
};

DEVI void s_finish(SpxState& s, double lam) {
  s.status = ST_SOLVED;
  s.cmd.lam = lam;
  s.cmd.phase = PH_FINAL;
  s.cmd.compact = 0;
}

// tot: 0 sum w, 1 max w
DEVI void s_after_init(SpxState& s, const double* tot) {
  if (s.l1 && tot[0] <= s.r) {  // simplex.py:324-325: inside the ball
    s.status = ST_SOLVED;
    s.iterations = -1;
    s.cmd.phase = PH_COPY;
    return;
  }
  // start: 0 = the formula (r - sum y)/n; 1 (default) = min(formula, r - max y),
  // both upper bounds of the root (phi(lam) >= sum(y) + n lam and
  // phi(lam) >= max(y) + lam), the second far tighter on spread data -- the
  // reference's own `lambda0=` route with a better start (simplex.py:246-250).
  // start 3: a given upper bound (the Algorithm-2 merge) tightened the same way
  const double formula = (s.r - tot[0]) / (double)s.n;
  const double tight = s.r - tot[1];
  double lam0;
  if (s.start == 3) lam0 = tight < s.lam0_value ? tight : s.lam0_value;
  else lam0 = s.lam0_given ? s.lam0_value : (s.start && tight < formula ? tight : formula);
  const double mn = -tot[1];
  s.lam0 = lam0 >= mn ? lam0 : mn;  // max(lambda0, min(-y)), simplex.py:250
  s.cmd.lam = s.lam0;
  s.cmd.phase = PH_SCAN;
  s.cmd.hist = s.hist_ok && s.start == 4 && !s.lam0_given && s.fixing;
  s.lam_hist = NAN;
  // First-scan capture (TMA engine): from an upper-bound start the iterates
  // only decrease, so w + lam0 < 0 means zero at every iterate; the first
  // scan already keeps only w > -lam0 - margin (the drop rule of the fixed
  // test with fix_hi = lam0 + margin), i.e. it compacts one scan earlier
  // than the fixing would.  Its sums are unchanged (dropped elements have
  // v < 0).  The margin covers a rounding-sized first step upwards.
  if (s.cap_first && s.fixing && !s.lam0_given) {
    s.cmd.capture = 1;
    s.cmd.compact = 1;
    s.cmd.fix_hi = s.lam0 + 1e-9 * fmax(1.0, fabs(s.lam0));
  }
}

// Capture start (TMA engine, large n): pass 0 (sum w, max w) and the first
// scan share one pass.  The start lam0 = min((r - sum w)/n, r - max w) (or
// the formula alone) bounds the root from above and the iterates only
// decrease from it, so an element with w + lam0 < 0 is zero at every iterate
// (simplex.py:256-303).  A sample gives a threshold T <= -lam0 with
// certainty for the tight term (sample max w - r <= max w - r) and six
// standard errors for the formula term; the fused pass computes pass 0's sums
// exactly and captures every w >= T.  If T <= -lam0 holds for the exact
// lam0 (checked), the captured values are the whole working set; otherwise
// the first scan reads y as usual.
// The sample: tot 0 sum w, 1 sum w^2, 2 elements, 3 max w.
DEVI void s_after_sample(SpxState& s, const double* tot, double local_count) {
  s.elems_scan += (int64_t)local_count;  // 8 B per sampled element
  const double m = fmax(tot[2], 1.0), N = (double)s.n;
  const double mean = tot[0] / m, var = fmax(tot[1] / m - mean * mean, 0.0);
  const double t_formula = mean - 6.0 * sqrt(var / m) - s.r / N;
  const double t_tight = tot[3] - s.r;
  // lowered by a margin the check below keeps (a sample holding the max
  // makes the tight term exactly -lam0)
  const double t = (s.start ? fmax(t_formula, t_tight) : t_formula);
  const double tm = t - 4e-9 * fmax(1.0, fabs(t));
  s.cmd.edge = isfinite(tm) && s.fused != 2 ? tm : HUGE_VAL;  // (nothing captured: the check fails)
  s.cmd.phase = PH_FUSED;
}

// The fused pass: tot 0 sum w, 1 max w (pass 0's sums), 2 elements captured.
DEVI void s_after_fused(SpxState& s, const double* tot, const double* loc) {
  s.cap_local = (int64_t)loc[2];
  s.elems_written += s.cap_local;
  s_after_init(s, tot);
  s.cmd.side = 0;
  if (s.cmd.phase != PH_SCAN) return;  // l1: inside the ball
  s.cmd.capture = 0;  // (the fused pass captured already; its fallback scans everything)
  s.cmd.compact = 0;
  s.cmd.fix_hi = INFINITY;
  // every element with w + lam0 >= -margin was captured (the margin covers a
  // first step upwards from rounding when lam0 is the root to the last bits)
  if (s.cmd.edge <= -s.lam0 - 1e-9 * fmax(1.0, fabs(s.lam0))) {
    s.cmd.side = 1;
    s.fixed_removed += s.local_active - s.cap_local;  // zero at every iterate, fixed at the first scan
    s.phys_count = s.cap_local;
    // every other x is a (signed) zero: the final pass need not re-read y --
    // worth it while the scatter of the captured x (index, y and x, each a
    // random sector) stays small against the 8 B per element it saves
    if (tot[2] * 64.0 <= (double)s.n) {
      s.sparse_final = 1;
      s.cmd.sparse = 1;
    }
  }
}

constexpr int64_t kCaptureEveryMax = 1 << 20;  // working sets up to 8 MB capture at every scan

// tot: 0 value, 1 #(v>0), 2 #(v==0)   (simplex.py:207-215, 256-294)
DEVI void s_after_scan(SpxState& s, const double* tot, const double* loc, double* trace) {
  s.phi_evals += 1;
  s.cmd.side = 0;
  s.elems_scan += s.phys_count;
  if (s.cmd.compact) {
    // a capturing scan's survivors are counted by the scan itself (slot 3)
    const int64_t kept = s.cmd.capture ? (int64_t)loc[3] : s.pending_phys;
    s.elems_written += kept;
    s.fixed_removed += s.phys_count - kept;
    s.phys_count = kept;
    s.cmd.compact = 0;
    s.cmd.capture = 0;
  }
  const double lam = s.cmd.lam, value = tot[0], dminus = tot[1], dplus = tot[1] + tot[2];
  if (trace && s.trace_len < s.trace_cap) {
    double* row = trace + 4 * s.trace_len++;
    row[0] = lam; row[1] = value; row[2] = dminus; row[3] = dplus;
  }
  double deriv;
  if (s.iterations == 0) {
    if (value == s.r) { s_finish(s, lam); return; }
    deriv = value < s.r ? dplus : dminus;
  } else {
    if (value <= s.r) { s_finish(s, lam); return; }
    deriv = dminus;
  }
  if (value < s.r) s.lo = lam;
  else {
    s.hi = lam;
    const int64_t at_zero = s.active - (int64_t)tot[1];
    if (s.fixing && at_zero > 0) {
      const int64_t at_zero_local = s.local_active - (int64_t)loc[1];
      s.fixed_count += at_zero;
      s.active -= at_zero;
      s.fixed_local += at_zero_local;
      s.local_active -= at_zero_local;
      s.cmd.fix_hi = lam;
    }
  }
  if (deriv <= 0) { s.cmd.phase = PH_SNAP; return; }
  const double step = -(value - s.r) / deriv;
  double next = lam + step;
  if (fabs(step) < s.tau || next == lam) { s_finish(s, next); return; }
  if (isfinite(s.lo) && isfinite(s.hi)) {
    if (s.hi - s.lo < s.tau * fmax(fabs(s.hi), fabs(s.lo))) { s_finish(s, next); return; }
  }
  // start "auto": both the Newton iterate and the histogram bound lie above
  // the root when phi > r; take the smaller (the first scan only)
  if (s.cmd.hist) {
    if (value > s.r && isfinite(s.lam_hist) && s.lam_hist < next && s.lam_hist > s.lo) next = s.lam_hist;
    s.cmd.hist = 0;
    s.lam_hist = NAN;
  }
  s.cmd.lam = next;
  s.iterations += 1;
  if (s.iterations > s.max_iter) { s_finish(s, next); return; }
  s.cmd.phase = PH_SCAN;
  s.cmd.compact = 0;
  if (s.cap_first && s.fixing && !s.lam0_given && s.phys_count <= kCaptureEveryMax) {
    // a small working set captures at every scan: the iterates only decrease
    // (upper-bound start), so w + next < 0 is zero from here on -- dropped in
    // the scan at next itself, one scan before the fixing would (the latency
    // of a grid epoch outweighs rewriting a small set)
    s.cmd.capture = 1;
    s.cmd.compact = 1;
    s.cmd.fix_hi = next + 1e-9 * fmax(1.0, fabs(next));
  } else if (s.fixing) {
    const int64_t present = s.fixed_local - s.fixed_removed;
    if (present > 0 && (double)present >= s.compact_ratio * (double)s.phys_count) {
      s.cmd.compact = 1;
      s.pending_phys = s.phys_count - present;
    }
  }
}

// tot: 0 max(-w) over the free set, 1 count
DEVI void s_after_snap(SpxState& s, const double* tot) {
  s.elems_scan += s.phys_count;
  if (tot[1] <= 0) { s.status = ST_CONTRACT; s.cmd.phase = PH_DONE; return; }
  s.cmd.lam = tot[0];
  s.iterations += 1;
  s.cmd.phase = PH_SCAN;
}

template <typename T, bool L1>
DEVI T spx_w(T y) { return L1 ? (T)fabs((double)y) : y; }

template <typename T, bool L1, bool SRC_SCRATCH, int MODE>  // MODE 0 init, 1 scan, 2 snap
DEVI void spx_pass(const SpxParams<T>& p, const Cmd& c, bool fix, int64_t seg_lo, int64_t& m,
                   bool compact, double (&acc)[kMaxK]) {
  constexpr int E = Vec<T>::n * kUnrollY, CH = 32 * E;
  const int lane = threadIdx.x & 31;
  const T* src = (SRC_SCRATCH ? p.sy : p.y) + seg_lo;
  const T lam = (T)c.lam, fhi = (T)c.fix_hi;
  const unsigned lt = (1u << lane) - 1u;
  const T* const pf[1] = {src};
  prefetch_chunks<T, 1, kUnrollY>(pf, 0, c_prefetch[1], m, lane);
  int64_t out_m = 0;
  for (int64_t base = 0; base < m; base += CH) {
    prefetch_chunks<T, 1, kUnrollY>(pf, base / CH + c_prefetch[1], c_prefetch[1] > 0 ? 1 : 0, m, lane);
    const bool full = base + CH <= m;
    T Y[E];
    load_chunk<T, SRC_SCRATCH, kUnrollY>(src, base, m, lane, full, T(0), Y);
    bool keep[E];
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const bool valid = full || chunk_index<T, kUnrollY>(base, lane, j) < m;
      // scratch already holds w = |y| for l1
      const T w = SRC_SCRATCH ? Y[j] : spx_w<T, L1>(Y[j]);
      Y[j] = w;
      keep[j] = false;
      if (!valid) continue;
      if (MODE == 0) {
        acc[0] += (double)w;
        acc[1] = fmax(acc[1], (double)w);
        continue;
      }
      const T v = add_rn(w, lam);
      if (fix && !(v > T(0)) && !(add_rn(w, fhi) > T(0))) continue;  // dropped
      keep[j] = true;
      if (MODE == 1) {
        if (v > T(0)) { acc[0] += (double)v; acc[1] += 1.0; }
        else if (v == T(0)) acc[2] += 1.0;
      } else {
        acc[0] = fmax(acc[0], -(double)w);
        acc[1] += 1.0;
      }
    }
    if (MODE == 1 && compact) {
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const unsigned mask = __ballot_sync(0xffffffffu, keep[j]);
        if (keep[j]) p.sy[seg_lo + out_m + __popc(mask & lt)] = Y[j];
        out_m += __popc(mask);
      }
    }
  }
  if (MODE == 1 && compact) m = out_m;
}

template <typename T, bool L1>
DEVI void spx_final(const SpxParams<T>& p, const Cmd& c, bool copy, int64_t seg_lo, int64_t m) {
  using V = typename Vec<T>::type;
  constexpr int VN = Vec<T>::n, E = VN * kUnrollY, CH = 32 * E;
  const int lane = threadIdx.x & 31;
  const T lam = (T)c.lam;
  T* x = p.x + seg_lo;
  const T* const pf[1] = {p.y + seg_lo};
  prefetch_chunks<T, 1, kUnrollY>(pf, 0, c_prefetch[1], m, lane);
  for (int64_t base = 0; base < m; base += CH) {
    prefetch_chunks<T, 1, kUnrollY>(pf, base / CH + c_prefetch[1], c_prefetch[1] > 0 ? 1 : 0, m, lane);
    const bool full = base + CH <= m;
    T Y[E], X[E];
    load_chunk<T, false, kUnrollY>(p.y + seg_lo, base, m, lane, full, T(0), Y);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      if (copy) { X[j] = Y[j]; continue; }
      const T w = spx_w<T, L1>(Y[j]);
      const T v = add_rn(w, lam);
      const T pos = v > T(0) ? v : T(0);  // np.maximum(0, w + lam)
      if (L1) {
        const T sg = Y[j] > T(0) ? T(1) : (Y[j] < T(0) ? T(-1) : T(0));
        X[j] = mul_rn(sg, pos);
      } else {
        X[j] = pos;
      }
    }
    if (full) {
#pragma unroll
      for (int u = 0; u < kUnrollY; ++u) {
        V v;
        T* vv = reinterpret_cast<T*>(&v);
#pragma unroll
        for (int q = 0; q < VN; ++q) vv[q] = X[u * VN + q];
        store_out(reinterpret_cast<V*>(x + base + (int64_t)u * 32 * VN + lane * VN), v);
      }
    } else {
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const int64_t e = chunk_index<T, kUnrollY>(base, lane, j);
        if (e < m) x[e] = X[j];
      }
    }
  }
}

template <typename T, bool L1>
__global__ void __launch_bounds__(kThreads, 1) spx_solve_kernel(SpxParams<T> p) {
  __shared__ double s_red[kWarps][kMaxK];
  __shared__ double s_tot[kMaxK];
  __shared__ Cmd s_cmd;
  __shared__ SpxState s_st;  // master (CTA 0) only
  __shared__ unsigned s_gen0;
  __shared__ int s_abort;
  const int warp = threadIdx.x >> 5;
  const bool master = blockIdx.x == 0;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp, W = (int64_t)gridDim.x * kWarps;
  int64_t seg_lo, seg_hi;
  warp_segment(p.n, gw, W, seg_lo, seg_hi);
  int64_t m = seg_hi - seg_lo;
  bool in_scratch = false;
  if (threadIdx.x == 0) {
    s_gen0 = ld_acquire(p.sync.gen);
    s_abort = 0;
    if (master) {
      s_st = p.init;
      s_cmd = s_st.cmd;
      tl_record(p.sync, 0, -1, p.n, 0);
    } else {
      s_cmd = p.init.cmd;
    }
  }
  __syncthreads();
  const bool fix = p.init.fixing != 0;
  for (unsigned epoch = 1;; ++epoch) {
    const Cmd c = s_cmd;
    if (c.phase == PH_DONE || s_abort) break;
    if (c.phase == PH_FINAL || c.phase == PH_COPY) {
      if (p.x) spx_final<T, L1>(p, c, c.phase == PH_COPY, seg_lo, seg_hi - seg_lo);
      break;
    }
    double acc[kMaxK];
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) acc[k] = 0.0;
    int ops[3] = {OP_SUM, OP_SUM, OP_SUM};
    int mode;
    if (c.phase == PH_LAMBDA0) {
      mode = 0;
      acc[1] = -HUGE_VAL;
      ops[1] = OP_MAX;
      int64_t m0 = seg_hi - seg_lo;
      spx_pass<T, L1, false, 0>(p, c, false, seg_lo, m0, false, acc);
    } else if (c.phase == PH_SCAN) {
      mode = 1;
      const bool compact = fix && c.compact;
      if (in_scratch) spx_pass<T, L1, true, 1>(p, c, fix, seg_lo, m, compact, acc);
      else spx_pass<T, L1, false, 1>(p, c, fix, seg_lo, m, compact, acc);
      if (compact) in_scratch = true;
    } else if (c.phase == PH_SNAP) {
      mode = 2;
      acc[0] = -HUGE_VAL;
      ops[0] = OP_MAX;
      if (in_scratch) spx_pass<T, L1, true, 2>(p, c, fix, seg_lo, m, false, acc);
      else spx_pass<T, L1, false, 2>(p, c, fix, seg_lo, m, false, acc);
    } else {
      break;
    }
    double a3[3] = {acc[0], acc[1], acc[2]};
    block_reduce<3>(a3, ops, s_red, s_tot);
    const bool is_master = grid_step<3>(p.partials, s_tot, ops, p.sync, s_red, s_tot, &s_abort, epoch);
    if (threadIdx.x == 0) {
      if (is_master) {
        tl_record(p.sync, epoch, c.phase, mode == 0 ? p.n : s_st.phys_count, s_st.cmd.compact);
        double loc[3] = {s_tot[0], s_tot[1], s_tot[2]}, glob[3];
        if (!exchange_totals_1(p.ex, epoch, 3, ops, loc, glob)) {
          raise_timeout(p.sync);
          s_st.status = ST_TIMEOUT;
          s_st.cmd.phase = PH_DONE;
        } else if (mode == 0) s_after_init(s_st, glob);
        else if (mode == 1) s_after_scan(s_st, glob, loc, p.trace);
        else s_after_snap(s_st, glob);
        const int ph = s_st.cmd.phase;
        if (ph == PH_FINAL || ph == PH_DONE || ph == PH_COPY) publish_state(p.out, s_st, p.sync);
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

// ------------------------------------------------------------ batched rows
// K8: one CTA per row (grid-stride over rows); the row lives in registers
// (EPT values per thread); every thread sees the same block totals so the
// Algorithm-4 decisions (simplex.py:256-294) are taken redundantly and
// identically -- no master, one __syncthreads per phi evaluation.
constexpr int kRowThreads = 256;

template <int EPT>
__global__ void __launch_bounds__(kRowThreads) spx_rows_kernel(
    const double* __restrict__ Y, double* __restrict__ X, double* __restrict__ lam_out,
    int32_t* __restrict__ it_out, int64_t rows, int cols, double r, double tau, int max_iter,
    int fixing, double lam0_given, int start) {
  __shared__ double s_part[2][kRowThreads / 32][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kRowThreads / 32;
  int buf = 0;
  auto reduce3 = [&](double v0, double v1, double v2, double& t0, double& t1, double& t2,
                     bool max1) {
    v0 = warp_sum(v0);
    v1 = max1 ? warp_max(v1) : warp_sum(v1);
    v2 = warp_sum(v2);
    if (lane == 0) { s_part[buf][warp][0] = v0; s_part[buf][warp][1] = v1; s_part[buf][warp][2] = v2; }
    __syncthreads();
    t0 = s_part[buf][0][0]; t1 = s_part[buf][0][1]; t2 = s_part[buf][0][2];
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      t0 += s_part[buf][w][0];
      t1 = max1 ? fmax(t1, s_part[buf][w][1]) : t1 + s_part[buf][w][1];
      t2 += s_part[buf][w][2];
    }
    buf ^= 1;  // double-buffered: the next write cannot race these reads
  };
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const double* y = Y + row * (int64_t)cols;
    double v[EPT];
    bool live[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int c = k * kRowThreads + threadIdx.x;
      live[k] = c < cols;
      v[k] = live[k] ? __ldcs(y + c) : 0.0;
    }
    double sum = 0.0, mx = -HUGE_VAL, unused;
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (live[k]) { sum += v[k]; mx = fmax(mx, v[k]); }
    double tsum, tmax;
    reduce3(sum, mx, 0.0, tsum, tmax, unused, true);
    const double formula = (r - tsum) / (double)cols, tight = r - tmax;
    double lam = !isnan(lam0_given) ? lam0_given : (start && tight < formula ? tight : formula);
    lam = lam >= -tmax ? lam : -tmax;
    double lo = -HUGE_VAL, hi = HUGE_VAL;
    int iterations = 0;
    bool drop[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) drop[k] = !live[k];
    for (;;) {
      double val = 0.0, npos = 0.0, nzero = 0.0;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        if (drop[k]) continue;
        const double t = __dadd_rn(v[k], lam);
        if (t > 0) { val += t; npos += 1.0; }
        else if (t == 0) nzero += 1.0;
      }
      double value, dminus, cz;
      reduce3(val, npos, nzero, value, dminus, cz, false);
      const double dplus = dminus + cz;
      double deriv;
      if (iterations == 0) {
        if (value == r) break;
        deriv = value < r ? dplus : dminus;
      } else {
        if (value <= r) break;
        deriv = dminus;
      }
      if (value < r) lo = lam;
      else {
        hi = lam;
        if (fixing) {
#pragma unroll
          for (int k = 0; k < EPT; ++k)
            if (!drop[k] && !(__dadd_rn(v[k], lam) > 0)) drop[k] = true;
        }
      }
      if (deriv <= 0) {
        double mneg = -HUGE_VAL;
#pragma unroll
        for (int k = 0; k < EPT; ++k)
          if (!drop[k]) mneg = fmax(mneg, -v[k]);
        double t0, t2;
        reduce3(0.0, mneg, 0.0, t0, mneg, t2, true);
        lam = mneg;
        ++iterations;
        continue;
      }
      const double step = -(value - r) / deriv;
      const double next = lam + step;
      if (fabs(step) < tau || next == lam) { lam = next; break; }
      if (isfinite(lo) && isfinite(hi) && hi - lo < tau * fmax(fabs(hi), fabs(lo))) {
        lam = next;
        break;
      }
      lam = next;
      ++iterations;
      if (iterations > max_iter) break;
    }
    double* x = X + row * (int64_t)cols;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int c = k * kRowThreads + threadIdx.x;
      if (live[k]) {
        const double t = __dadd_rn(v[k], lam);
        __stcs(x + c, t > 0 ? t : 0.0);
      }
    }
    if (threadIdx.x == 0) {
      if (lam_out) lam_out[row] = lam;
      if (it_out) it_out[row] = iterations;
    }
  }
}

// ------------------------------------------------------------ bulk-copy helpers
DEVI unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
DEVI void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
DEVI void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
DEVI void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
DEVI void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

// ------------------------------------------------------------ Algorithm 2
// The reference's Gauss-Seidel initializer (simplex.py:47-111) run per
// contiguous chunk -- par_simplex_init semantics (parallel.py:330-368): chunk
// k = [floor(k n/W), floor((k+1) n/W)) exactly as np.linspace(...).astype(int64)
// (parallel.py:82-85), one GPU thread per chunk replaying the sequential
// recurrence bit for bit, then a one-block merge in _tree_sum order
// (parallel.py:62-72).  Every zero proven inside a chunk is valid globally
// (the chunk's multiplier bounds the full problem's from above), so the free
// set that Algorithm 4 iterates on collapses to a tiny fraction of n.
struct Alg2Out {
  double lam0, sum_free, sum_abs;
  int64_t n_free;
  int32_t inside;  // l1: sum |y| <= r
  int32_t pad;
};

DEVI void chunk_bounds(int64_t n, int64_t W, int64_t k, int64_t& lo, int64_t& hi) {
  const double step = (double)n / (double)W;
  lo = (int64_t)((double)k * step);
  hi = k + 1 == W ? n : (int64_t)((double)(k + 1) * step);
}

template <bool L1>
__global__ void __launch_bounds__(256) alg2_chunks_kernel(
    const double* __restrict__ y, const int64_t* __restrict__ idx, int64_t p, double r,
    int64_t W, const double* __restrict__ xbar, int sharpened, int32_t* __restrict__ J,
    int32_t* __restrict__ Jt, uint8_t* __restrict__ fixed, double* __restrict__ sums,
    int64_t* __restrict__ cards, int64_t* __restrict__ jplus_out, double* __restrict__ sumabs,
    double* __restrict__ lams) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= W) return;
  int64_t lo, hi;
  chunk_bounds(p, W, k, lo, hi);
  auto w_of = [&](int64_t pos) -> double {
    const int64_t i = idx ? idx[pos] : pos;
    const double v = __ldg(y + i);
    return L1 ? fabs(v) : v;
  };
  auto orig = [&](int64_t pos) -> int64_t { return idx ? idx[pos] : pos; };
  const bool use_xbar = xbar != nullptr;
  int32_t* Jc = J + lo;
  int32_t* Jtc = Jt + lo;
  double sabs = 0.0;
  // simplex.py:58-111 with local offsets (pos - lo) in J / Jt.  Sharpened,
  // a chunk other than the first does not seed with a y <= 0: the sequential
  // recurrence only ever seeds with idx[0], every later y <= 0 is fixed
  // outright (simplex.py:74-76), so the chunk skips (fixes) its leading
  // nonpositive entries and seeds with its first positive one -- the union of
  // the fixed sets then matches the sequential one apart from zero proofs,
  // which hold for the restricted problem too.  (Chunk 0's seed idx[0] <= 0
  // is decided by the host: it runs the exact sequential recurrence.)
  int64_t first = lo;
  if (sharpened && k > 0 && !use_xbar) {
    while (first < hi && !(w_of(first) > 0.0)) {
      sabs += w_of(first);
      if (fixed) fixed[orig(first)] = 1;
      ++first;
    }
    if (first == hi) {  // nothing positive: the chunk joins no free set
      sums[k] = 0.0;
      cards[k] = 0;
      jplus_out[k] = 0;
      lams[k] = INFINITY;
      if (sumabs) sumabs[k] = sabs;
      return;
    }
  }
  const double y1 = w_of(first);
  sabs += y1;
  int64_t nJ = 1, nJt = 0, jplus = 0;
  Jc[0] = (int32_t)(first - lo);
  double sumJ = y1, lam = r - y1;
  if (!use_xbar || xbar[orig(first)] > 0.0) jplus = 1;
  for (int64_t pos = first + 1; pos < hi; ++pos) {
    const double yi = w_of(pos);
    sabs += yi;
    if (use_xbar && xbar[orig(pos)] <= 0.0) continue;
    bool ok = __dadd_rn(yi, lam) > 0.0;
    if (sharpened && yi <= 0.0) ok = false;
    if (!ok) {
      if (fixed) fixed[orig(pos)] = 1;
      continue;
    }
    const double cand = __ddiv_rn(__dsub_rn(__dsub_rn(r, sumJ), yi), (double)(nJ + 1));
    if (cand < __dsub_rn(r, yi)) {
      Jc[nJ++] = (int32_t)(pos - lo);
      sumJ = __dadd_rn(sumJ, yi);
      lam = cand;
    } else {
      for (int64_t q = 0; q < nJ; ++q) Jtc[nJt++] = Jc[q];
      Jc[0] = (int32_t)(pos - lo);
      nJ = 1;
      sumJ = yi;
      lam = __dsub_rn(r, yi);
      jplus = 0;
    }
    if (!use_xbar || xbar[orig(pos)] > 0.0) ++jplus;
  }
  for (int64_t q = 0; q < nJt; ++q) {
    const int64_t pos = lo + Jtc[q];
    const double yi = w_of(pos);
    bool ok = __dadd_rn(yi, lam) > 0.0;
    if (sharpened && yi <= 0.0) ok = false;
    if (!ok) {
      if (fixed) fixed[orig(pos)] = 1;
      continue;
    }
    lam = __ddiv_rn(__dsub_rn(__dsub_rn(r, sumJ), yi), (double)(nJ + 1));
    Jc[nJ++] = Jtc[q];
    sumJ = __dadd_rn(sumJ, yi);
    if (!use_xbar || xbar[orig(pos)] > 0.0) ++jplus;
  }
  sums[k] = sumJ;
  cards[k] = nJ;
  jplus_out[k] = jplus;
  lams[k] = lam;  // simplex_init_lambda returns the recurrence's own lam
  if (sumabs) sumabs[k] = sabs;
}

// One block: _tree_sum of the chunk sums (and of sum|y| for the l1 test) in
// the reference's pairwise order, and exclusive offsets of the chunk cards.
__global__ void __launch_bounds__(1024) alg2_merge_kernel(const double* __restrict__ sums,
                                                          const double* __restrict__ sumabs,
                                                          const int64_t* __restrict__ cards,
                                                          const double* __restrict__ lams,
                                                          int64_t W, double r, double* scratch,
                                                          int64_t* offsets, Alg2Out* out) {
  __shared__ int64_t s_part[1024];
  // exclusive scan of cards: contiguous ranges per thread
  const int64_t per = (W + blockDim.x - 1) / blockDim.x;
  const int64_t c0 = threadIdx.x * per, c1 = c0 + per < W ? c0 + per : W;
  int64_t loc = 0;
  for (int64_t c = c0; c < c1; ++c) loc += cards[c];
  s_part[threadIdx.x] = loc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const int64_t v = s_part[t];
      s_part[t] = run;
      run += v;
    }
    out->n_free = run;
  }
  __syncthreads();
  int64_t run = s_part[threadIdx.x];
  for (int64_t c = c0; c < c1; ++c) {
    offsets[c] = run;
    run += cards[c];
  }
  // _tree_sum: adjacent pairs level by level, odd tail carried (ping-pong)
  for (int pass = 0; pass < (sumabs ? 2 : 1); ++pass) {
    const double* src = pass == 0 ? sums : sumabs;
    double* bufA = scratch;
    double* bufB = scratch + W;
    for (int64_t i = threadIdx.x; i < W; i += blockDim.x) bufA[i] = src[i];
    __syncthreads();
    int64_t k = W;
    while (k > 1) {
      const int64_t half = k / 2;
      for (int64_t j = threadIdx.x; j < half; j += blockDim.x) bufB[j] = bufA[2 * j] + bufA[2 * j + 1];
      if ((k & 1) && threadIdx.x == 0) bufB[half] = bufA[k - 1];
      __syncthreads();
      k = half + (k & 1);
      double* t = bufA;
      bufA = bufB;
      bufB = t;
    }
    if (threadIdx.x == 0) {
      if (pass == 0) out->sum_free = bufA[0];
      else out->sum_abs = bufA[0];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // one chunk: simplex_init_lambda's lam (simplex.py:111); else the merge
    // of par_simplex_init (parallel.py:365)
    out->lam0 = W == 1 ? lams[0] : (r - out->sum_free) / (double)out->n_free;
    out->inside = sumabs ? out->sum_abs <= r : 0;
  }
}

// Gather the free set: values (w = y or |y|) and, optionally, global indices.
template <bool L1>
__global__ void __launch_bounds__(256) alg2_gather_kernel(
    const double* __restrict__ y, const int64_t* __restrict__ idx, int64_t p, int64_t W,
    const int32_t* __restrict__ J, const int64_t* __restrict__ cards,
    const int64_t* __restrict__ offsets, double* __restrict__ vals, int64_t* __restrict__ gidx) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= W) return;
  int64_t lo, hi;
  chunk_bounds(p, W, k, lo, hi);
  const int64_t c = cards[k], o = offsets[k];
  for (int64_t q = 0; q < c; ++q) {
    const int64_t pos = lo + J[lo + q];
    const int64_t i = idx ? idx[pos] : pos;
    if (vals) {
      const double v = y[i];
      vals[o + q] = L1 ? fabs(v) : v;
    }
    if (gidx) gidx[o + q] = i;
  }
}

// x = max(0, y + lam) (simplex.py:303) / sign(y) max(0, |y| + lam) (simplex.py:333)
template <bool L1>
__global__ void __launch_bounds__(256) spx_x_kernel(const double* __restrict__ y, int64_t n,
                                                    double lam, int copy, double* __restrict__ x) {
  const int64_t n2 = n / 2;
  const double2* y2 = reinterpret_cast<const double2*>(y);
  double2* x2 = reinterpret_cast<double2*>(x);
  const bool vec = (((uintptr_t)y | (uintptr_t)x) & 15) == 0;
  auto f = [&](double v) {
    if (copy) return v;
    const double w = L1 ? fabs(v) : v;
    const double t = __dadd_rn(w, lam);
    const double pos = t > 0 ? t : 0.0;
    if (!L1) return pos;
    const double sg = v > 0 ? 1.0 : (v < 0 ? -1.0 : 0.0);
    return __dmul_rn(sg, pos);
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
      double2 v = ld_stream(y2 + i);
      v.x = f(v.x);
      v.y = f(v.y);
      __stcs(x2 + i, v);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) x[n - 1] = f(y[n - 1]);
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) x[i] = f(y[i]);
  }
}

// Warm-started projections: the free set is every index the initializer did
// not prove zero (simplex.py:244, ~fixed_mask -- with xbar that is more than
// its running set J).  One CTA, chunks of 1024 in index order, warp-ballot
// block scan: deterministic, np.flatnonzero order.
template <bool L1>
__global__ void __launch_bounds__(1024) spx_gather_free_kernel(const double* __restrict__ y,
                                                               const uint8_t* __restrict__ fixed,
                                                               int64_t n, double* __restrict__ vals,
                                                               int64_t* __restrict__ count) {
  __shared__ int s_w[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t base_out = 0;
  for (int64_t c0 = 0; c0 < n; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    const bool keep = i < n && !fixed[i];
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_w[warp] = __popc(bal);
    __syncthreads();
    int pre = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      const int v = s_w[w];
      pre += w < warp ? v : 0;
      tot += v;
    }
    if (keep) {
      const double v = y[i];
      vals[base_out + pre + __popc(bal & ((1u << lane) - 1u))] = L1 ? fabs(v) : v;
    }
    base_out += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base_out;
}

// ------------------------------------------------------------ utilities
// Grid-stride kernels with per-block partials + a fixed-order finalize; used
// by the component-level entry points (eval_phi, eval_x, breakpoints,
// validate, initial_multiplier), optionally through an index list.
constexpr int kUtilThreads = 256;

template <typename T>
DEVI int64_t gat(const int64_t* idx, int64_t k) { return idx ? idx[k] : k; }

// slots: 0 value, 1 abs, 2 core, 3 tie_lo, 4 tie_hi
template <typename T>
__global__ void __launch_bounds__(kUtilThreads) phi_util_kernel(
    const T* d, const T* a, const T* b, const T* l, const T* u, const int64_t* idx, int64_t m,
    double lam_d, uint8_t* at_lo, uint8_t* at_hi, double* partials) {
  __shared__ double s_red[kUtilThreads / 32][kMaxK];
  __shared__ double s_tot[kMaxK];
  const T lam = (T)lam_d;
  double acc[kMaxK];
  for (int k = 0; k < kMaxK; ++k) acc[k] = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = gat<T>(idx, k);
    const T t = t_of(d[i], a[i], b[i], lam);
    if (at_lo) at_lo[k] = t <= l[i];
    if (at_hi) at_hi[k] = t >= u[i];
    elem_scan<T, false>(d[i], a[i], b[i], l[i], u[i], lam, lam, lam, false, false, acc);
  }
  const int ops[5] = {OP_SUM, OP_SUM, OP_SUM, OP_SUM, OP_SUM};
  double a5[5] = {acc[0], acc[1], acc[2], acc[3], acc[4]};
  block_reduce<5>(a5, ops, s_red, s_tot);
  if (threadIdx.x < 5) partials[blockIdx.x * kMaxK + threadIdx.x] = s_tot[threadIdx.x];
}

template <typename T>
__global__ void __launch_bounds__(kUtilThreads) evalx_util_kernel(
    const T* d, const T* a, const T* b, const T* l, const T* u, const int64_t* idx, int64_t m,
    double lam_d, T* x) {
  const T lam = (T)lam_d;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = gat<T>(idx, k);
    x[k] = clip(t_of(d[i], a[i], b[i], lam), l[i], u[i]);
  }
}

// slots: 0 best, 1 found
template <typename T>
__global__ void __launch_bounds__(kUtilThreads) bp_util_kernel(
    const T* d, const T* a, const T* b, const T* l, const T* u, const int64_t* idx, int64_t m,
    double edge, int right, double* partials) {
  __shared__ double s_red[kUtilThreads / 32][kMaxK];
  __shared__ double s_tot[kMaxK];
  double best = right ? HUGE_VAL : -HUGE_VAL, found = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = gat<T>(idx, k);
    elem_bp<T>(d[i], a[i], b[i], l[i], u[i], edge, right != 0, best, found);
  }
  const int ops[2] = {right ? OP_MIN : OP_MAX, OP_SUM};
  double a2[2] = {best, found};
  block_reduce<2>(a2, ops, s_red, s_tot);
  if (threadIdx.x < 2) partials[blockIdx.x * kMaxK + threadIdx.x] = s_tot[threadIdx.x];
}

// slots as the persistent lambda0 pass (0..4 sums, 5..14 validate mins)
template <typename T>
__global__ void __launch_bounds__(kUtilThreads) lambda0_util_kernel(
    const T* d, const T* a, const T* b, const T* l, const T* u, const T* xbar, int64_t n,
    int check, double* partials) {
  __shared__ double s_red[kUtilThreads / 32][kMaxK];
  __shared__ double s_tot[kMaxK];
  double acc[15];
  for (int k = 0; k < 15; ++k) acc[k] = k < kValidateSlot ? 0.0 : HUGE_VAL;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T di = d[i], ai = a[i], bi = b[i];
    const T y = rcp_nr(di);
    const double s = (double)mul_rn(bi, ai * y);
    const double q = (double)mul_rn(bi, bi * y);
    acc[0] += s;
    acc[1] += q;
    if (xbar) {
      const T xi = xbar[i];
      if (l[i] < xi && xi < u[i]) { acc[2] += s; acc[3] += q; acc[4] += 1.0; }
    }
    if (check) {
      const double gi = (double)i;
      const T li = l[i], ui = u[i];
      if (!isfinite((double)di)) acc[5] = fmin(acc[5], gi);
      if (!isfinite((double)ai)) acc[6] = fmin(acc[6], gi);
      if (!isfinite((double)bi)) acc[7] = fmin(acc[7], gi);
      if (isnan((double)li)) acc[8] = fmin(acc[8], gi);
      if (isnan((double)ui)) acc[9] = fmin(acc[9], gi);
      if (!(di > T(0))) acc[10] = fmin(acc[10], gi);
      if (!(bi > T(0))) acc[11] = fmin(acc[11], gi);
      if (!(li <= ui)) acc[12] = fmin(acc[12], gi);
      if ((double)li == HUGE_VAL) acc[13] = fmin(acc[13], gi);
      if ((double)ui == -HUGE_VAL) acc[14] = fmin(acc[14], gi);
    }
  }
  const int ops[15] = {OP_SUM, OP_SUM, OP_SUM, OP_SUM, OP_SUM, OP_MIN, OP_MIN, OP_MIN,
                       OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN, OP_MIN};
  block_reduce<15>(acc, ops, s_red, s_tot);
  if (threadIdx.x < 15) partials[blockIdx.x * kMaxK + threadIdx.x] = s_tot[threadIdx.x];
}

// one block: fixed-order reduction of `nblk` partial rows -> out[0..K)
__global__ void __launch_bounds__(kUtilThreads) finalize_kernel(const double* partials,
                                                                int nblk, int K, int opmask_min,
                                                                int opmask_max, double* out) {
  __shared__ double s_red[kUtilThreads / 32][kMaxK];
  __shared__ double s_tot[kMaxK];
  double acc[kMaxK];
  int ops[kMaxK];
  for (int k = 0; k < kMaxK; ++k) {
    ops[k] = (opmask_min >> k) & 1 ? OP_MIN : (opmask_max >> k) & 1 ? OP_MAX : OP_SUM;
    acc[k] = ops[k] == OP_SUM ? 0.0 : ops[k] == OP_MIN ? HUGE_VAL : -HUGE_VAL;
  }
  for (int c = threadIdx.x; c < nblk; c += blockDim.x)
    for (int k = 0; k < K; ++k) {
      const double v = partials[c * kMaxK + k];
      acc[k] = ops[k] == OP_SUM ? acc[k] + v : ops[k] == OP_MIN ? fmin(acc[k], v) : fmax(acc[k], v);
    }
  block_reduce<kMaxK>(acc, ops, s_red, s_tot);
  if (threadIdx.x < K) out[threadIdx.x] = s_tot[threadIdx.x];
}

// Division self-test: bitwise comparison of div_y (shared reciprocal) with
// __ddiv_rn over random operands (counter-based hash RNG); counts mismatches.
DEVI unsigned long long mix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void div_selftest_kernel(unsigned long long seed, long long count, int mode,
                                    unsigned long long* mismatches, double* example) {
  unsigned long long bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long h1 = mix64(seed ^ (2 * i)), h2 = mix64(seed ^ (2 * i + 1));
    double a, b;
    if (mode == 0) {  // random mantissas, exponents over [-500, 500]
      const long long ea = (long long)(h1 % 1001) - 500, eb = (long long)(h2 % 1001) - 500;
      a = __longlong_as_double((long long)((ea + 1023) << 52) | (long long)(mix64(h1) & 0xFFFFFFFFFFFFFull));
      b = __longlong_as_double((long long)((eb + 1023) << 52) | (long long)(mix64(h2) & 0xFFFFFFFFFFFFFull));
      if (h1 & (1ull << 63)) a = -a;
    } else if (mode == 1) {  // the solver's numerators/denominators: |a| < 1e4, d in [1, 64)
      a = ((double)(h1 >> 11) * 0x1p-53 - 0.5) * 2e4;
      b = 1.0 + (double)(h2 >> 11) * 0x1p-53 * 63.0;
    } else {  // quotients near representable midpoints: a = q*b +- tiny
      b = 1.0 + (double)(h2 >> 11) * 0x1p-53 * 63.0;
      const double q = 1.0 + (double)(h1 >> 11) * 0x1p-53;
      a = __dmul_rn(q, b);
      a = __longlong_as_double(__double_as_longlong(a) + (long long)(mix64(h1) % 5) - 2);
    }
    const double ref = __ddiv_rn(a, b);
    const double got = div_y(a, b, rcp_div(b));
    if (__double_as_longlong(ref) != __double_as_longlong(got)) {
      ++bad;
      if (example) { example[0] = a; example[1] = b; }
    }
  }
  if (bad) atomicAdd(mismatches, bad);
}

}  // namespace cqk

// cqk_abi.cu -- C-ABI implementation (include/cqk_b200.h).
//
// Owns: one stream, the persistent kernels' grid-sync words and master state,
// per-CTA partials, compaction scratch (grow-only) and host-mode staging.
// Every solve is ONE cooperative kernel launch; the small state struct goes
// H2D before and D2H after it.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/cqk_b200.h"
#include <cub/device/device_radix_sort.cuh>
#include "cqk_kernels.cuh"
#include "cqk_tma.cuh"
#include "cqk_tma_spx.cuh"
#include "cqk_diag.cuh"
#include "cqk_rows.cuh"

using namespace cqk;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return set_err(CQK_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kTraceCap = 1024;
constexpr int kUtilBlocksMax = 1184;

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// L2 bulk-prefetch distance (chunks) for the persistent kernels, set once per
// process at handle creation (a per-solve constant-bank update would
// serialise against kernels of other handles); CQK_PREFETCH="cqk,y" tunes it.
cudaError_t set_prefetch() {
  int pf[2] = {0, 2};
  if (const char* e = getenv("CQK_PREFETCH")) sscanf(e, "%d,%d", &pf[0], &pf[1]);
  int tf = 12;  // late, shallow speculation (cqk_tma.cuh)
  if (const char* e = getenv("CQK_TMA_FLAGS")) tf = atoi(e);
  cudaError_t err = cudaMemcpyToSymbol(c_tma_flags, &tf, sizeof tf);
  err = err ? err : cudaMemcpyToSymbol(c_tma_flags_w, &tf, sizeof tf);
  return err ? err : cudaMemcpyToSymbol(c_prefetch, pf, sizeof pf);
}

}  // namespace

struct cqk_handle {
  int device = 0;
  int sm_count = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int grid_cqk_fix = 0, grid_cqk_jac = 0, grid_spx = 0, grid_l1 = 0;
  int grid_cqk_fix32 = 0, grid_cqk_jac32 = 0, grid_spx32 = 0, grid_l1_32 = 0;  // float instances
  int grid_tma_fix = 0, grid_tma_jac = 0;  // TMA-pipelined CQK kernels (0: unavailable)
  int grid_tma_spx = 0, grid_tma_l1 = 0;    // TMA-pipelined simplex / l1 kernels
  bool use_tma = true;                     // CQK_ENGINE=seg selects the warp-segment kernel
  int engine = 0;                          // cqk_set_engine: 0 auto, 1 TMA, 2 warp segments
  int64_t tma_min_n = 65536;               // auto: CQK solves of >= this many elements per rank
  int fused_guess = 1;                     // fused start: direction guess + survivor list (CQK_FUSED_GUESS)
  int spx_capture = 1;                     // simplex / l1 capture start (CQK_SPX_CAPTURE)
  int64_t spx_capture_min_n = 4000000;     // ... from this many elements per rank (CQK_SPX_CAPTURE_MIN_N)
  static constexpr int64_t kGuessMinN = 8000000;  // ... from this many elements per rank
  int64_t fused_min_n = 4000000;           // fused start (sample + fused first pass) from this size
  double fused_width = 2e-3;               // ... its classification interval, relative half-width
  unsigned* sync = nullptr;  // [0] arrive, [1] gen, [2] error
  void* state = nullptr;     // CqkState / SpxState
  double* partials = nullptr;
  double* trace = nullptr;
  long long* timeline = nullptr;
  double* red = nullptr;     // utility partials
  double* out = nullptr;     // utility outputs (kMaxK doubles)
  Buf scratch, stage, idxbuf, flags, alg2, warm;
  Buf sparse_buf;                     // output="sparse": (index, value) pairs, counter, sort space
  struct SparseReq {                  // set by spx/l1_project_sparse_f64 for one call
    int64_t* idx;
    double* val;
    unsigned long long* cnt;
    int64_t cap;
  };
  const SparseReq* sparse_req = nullptr;
  // pageable host inputs / outputs: a ring of pinned chunk buffers filled /
  // drained by OpenMP memcpy while the copy engine moves the previous chunk
  static constexpr int kRing = 4;
  static constexpr size_t kRingBytes = 32u << 20;
  void* ring[kRing] = {};
  cudaEvent_t ring_ev[kRing] = {};
  int32_t* wcnt = nullptr;            // per-warp scratch counts (simplex tail mode)
  int32_t* hist = nullptr;            // first-scan bucket counts (simplex start "auto"), two halves
  int hist_flip = 0;                  // ... the half the next launch uses (arrives zero)
  double* ar_rows = nullptr;          // masterless grid step: [2][grid][kArStride] tagged partial rows
  unsigned* ar_count = nullptr;       // ... [2] arrival counters, alternating per launch
  unsigned long long ar_seq = 0;      // masterless launches so far
  int rows_flip = 0;                  // C5 row counter (ar_count[8 + flip]) of the next launch
  double* alg2_vals = nullptr;        // gathered free values of the last Algorithm-2 run
  int64_t* alg2_idx = nullptr;        // ... and their global indices
  int64_t* alg2_jplus = nullptr;
  int64_t alg2_w = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int trace_len = 0;
  int grid_limit = 0;                 // 0: full device (virtual ranks share a GPU)
  // A/B switches, read once at cqk_create (environment)
  bool master_step = false;           // CQK_MASTER_STEP: master + release grid step
  bool static_final = false;          // CQK_STATIC_FINAL: static final-pass tiles
  bool tail_mode = true;              // CQK_TAIL=0: no single-CTA simplex tail
  int64_t alg2_chunk = 256;           // CQK_ALG2_CHUNK: device Algorithm-2 chunk length
  void* host_state = nullptr;         // pinned + mapped: the kernels' final state (and Alg2Out)
  void* host_state_dev = nullptr;     // ... its device alias
  volatile int* host_err = nullptr;   // mapped word after the state: any CTA's spin timeout
  int* host_err_dev = nullptr;        // ... its device alias
  // multi-GPU communicator (one rank per GPU; mailboxes in device memory)
  int rank = 0, world = 1;
  double* mbox = nullptr;             // this rank's mailbox
  double* peers[kMaxRanks] = {};      // every rank's mailbox (IPC-mapped or local)
  bool ipc_opened[kMaxRanks] = {};
  unsigned long long seq = 0;         // sharded-solve sequence number
};

extern "C" {

int cqk_abi_version(void) { return CQK_ABI_VERSION; }

const char* cqk_last_error(void) { return g_err.c_str(); }

int cqk_create(cqk_handle** out, int device) {
  if (!out) return set_err(CQK_E_ARG, "null handle pointer");
  *out = nullptr;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_err(CQK_E_ARG, "bad device ordinal");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return set_err(CQK_E_CUDA, "this library is built for sm_100a (B200); found sm_" +
                                   std::to_string(prop.major * 10 + prop.minor));
  if (!prop.cooperativeLaunch) return set_err(CQK_E_CUDA, "device lacks cooperative launch");
  cqk_handle* h = new cqk_handle();
  h->device = device;
  h->sm_count = prop.multiProcessorCount;
  auto occ = [&](const void* fn) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, 0);
    return b < 1 ? 0 : b * h->sm_count;
  };
  h->grid_cqk_fix = occ((const void*)cqk_solve_kernel<double, true>);
  h->grid_cqk_jac = occ((const void*)cqk_solve_kernel<double, false>);
  h->grid_spx = occ((const void*)spx_solve_kernel<double, false>);
  h->grid_l1 = occ((const void*)spx_solve_kernel<double, true>);
  h->grid_cqk_fix32 = occ((const void*)cqk_solve_kernel<float, true>);
  h->grid_cqk_jac32 = occ((const void*)cqk_solve_kernel<float, false>);
  h->grid_spx32 = occ((const void*)spx_solve_kernel<float, false>);
  h->grid_l1_32 = occ((const void*)spx_solve_kernel<float, true>);
  {
    auto occ_tma = [&](const void* fn) {
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemC) !=
          cudaSuccess)
        return 0;
      int b = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kTmaThreads, kSmemC);
      return b < 1 ? 0 : h->sm_count;  // one CTA per SM (the pipeline owns the SM)
    };
    h->grid_tma_fix = occ_tma((const void*)cqk_tma_kernel<true>);
    h->grid_tma_jac = occ_tma((const void*)cqk_tma_kernel<false>);
    h->grid_tma_spx = occ_tma((const void*)spx_tma_kernel<false>);
    h->grid_tma_l1 = occ_tma((const void*)spx_tma_kernel<true>);
    cudaGetLastError();
    const char* eng = getenv("CQK_ENGINE");
    h->use_tma = !(eng && std::strcmp(eng, "seg") == 0) && h->grid_tma_fix > 0 &&
                 h->grid_tma_jac > 0 && h->grid_tma_spx > 0 && h->grid_tma_l1 > 0;
  }
  int gmax = h->grid_cqk_fix;
  gmax = gmax > h->grid_cqk_jac ? gmax : h->grid_cqk_jac;
  gmax = gmax > h->grid_spx ? gmax : h->grid_spx;
  gmax = gmax > h->grid_l1 ? gmax : h->grid_l1;
  for (int g32 : {h->grid_cqk_fix32, h->grid_cqk_jac32, h->grid_spx32, h->grid_l1_32})
    gmax = gmax > g32 ? gmax : g32;
  if (gmax == 0) {
    delete h;
    return set_err(CQK_E_CUDA, "persistent kernels do not fit on an SM");
  }
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
  e = e ? e : cudaMalloc(&h->sync, 64);
  e = e ? e : cudaMemset(h->sync, 0, 64);
  size_t st_bytes = sizeof(CqkState) > sizeof(SpxState) ? sizeof(CqkState) : sizeof(SpxState);
  e = e ? e : cudaMalloc(&h->state, st_bytes);
  e = e ? e : cudaMalloc(&h->partials, sizeof(double) * kMaxK * (gmax + kUtilBlocksMax));
  e = e ? e : cudaMalloc(&h->trace, sizeof(double) * 4 * kTraceCap);
  e = e ? e : cudaMalloc(&h->timeline, sizeof(long long) * kTimelineCols * kTimelineCap);
  e = e ? e : cudaMemset(h->timeline, 0, sizeof(long long) * kTimelineCols * kTimelineCap);
  e = e ? e : cudaMalloc(&h->red, sizeof(double) * kMaxK * kUtilBlocksMax);
  e = e ? e : cudaMalloc(&h->out, sizeof(double) * kMaxK);
  e = e ? e : cudaMalloc(&h->wcnt, sizeof(int32_t) * kConsW * (h->sm_count + 8));
  e = e ? e : cudaMalloc(&h->hist, sizeof(int32_t) * kHistB * (h->sm_count + 8));
  e = e ? e : cudaMemset(h->hist, 0, sizeof(int32_t) * kHistB * (h->sm_count + 8));
  e = e ? e : cudaMalloc(&h->ar_rows, sizeof(double) * 2 * kArStride * (h->sm_count + 8));
  e = e ? e : cudaMemset(h->ar_rows, 0, sizeof(double) * 2 * kArStride * (h->sm_count + 8));
  e = e ? e : cudaMalloc(&h->ar_count, 64);
  e = e ? e : cudaMemset(h->ar_count, 0, 64);
  const size_t st_pad = (st_bytes + 63) / 64 * 64;
  e = e ? e : cudaHostAlloc(&h->host_state, st_pad + 64, cudaHostAllocMapped | cudaHostAllocPortable);
  e = e ? e : cudaHostGetDevicePointer(&h->host_state_dev, h->host_state, 0);
  if (e == cudaSuccess) {
    h->host_err = (volatile int*)((char*)h->host_state + st_pad);
    h->host_err_dev = (int*)((char*)h->host_state_dev + st_pad);
    *h->host_err = 0;
  }
  e = e ? e : set_prefetch();
  e = e ? e : cudaEventCreate(&h->ev0);
  e = e ? e : cudaEventCreate(&h->ev1);
  e = e ? e : cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cqk_destroy(h);
    return set_err(CQK_E_CUDA, std::string("cqk_create: ") + cudaGetErrorString(e));
  }
  h->stream = h->own;
  if (const char* gl = getenv("CQK_GRID_LIMIT")) h->grid_limit = atoi(gl);  // shared-GPU runs
  if (const char* mn = getenv("CQK_TMA_MIN_N")) h->tma_min_n = atoll(mn);
  if (const char* fm = getenv("CQK_FUSED_MIN_N")) h->fused_min_n = atoll(fm);
  if (const char* fg = getenv("CQK_FUSED_GUESS")) h->fused_guess = atoi(fg);
  if (const char* sc = getenv("CQK_SPX_CAPTURE")) h->spx_capture = atoi(sc);
  if (const char* sm = getenv("CQK_SPX_CAPTURE_MIN_N")) h->spx_capture_min_n = atoll(sm);
  auto flag = [](const char* name) {
    const char* e = getenv(name);
    return e && e[0] && e[0] != '0';
  };
  h->master_step = flag("CQK_MASTER_STEP");
  h->static_final = flag("CQK_STATIC_FINAL");
  if (const char* te = getenv("CQK_TAIL")) h->tail_mode = te[0] != '0';
  if (const char* e = getenv("CQK_ALG2_CHUNK")) h->alg2_chunk = atoll(e) > 0 ? atoll(e) : 256;
  *out = h;
  return 0;
}

int cqk_destroy(cqk_handle* h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->scratch.release();
  h->stage.release();
  h->idxbuf.release();
  h->flags.release();
  h->alg2.release();
  h->warm.release();
  h->sparse_buf.release();
  for (int q = 0; q < kMaxRanks; ++q)
    if (h->ipc_opened[q] && h->peers[q]) cudaIpcCloseMemHandle(h->peers[q]);
  if (h->mbox) cudaFree(h->mbox);
  cudaFree(h->sync);
  cudaFree(h->state);
  cudaFree(h->partials);
  cudaFree(h->trace);
  cudaFree(h->timeline);
  cudaFree(h->red);
  cudaFree(h->out);
  if (h->wcnt) cudaFree(h->wcnt);
  if (h->hist) cudaFree(h->hist);
  if (h->ar_rows) cudaFree(h->ar_rows);
  if (h->ar_count) cudaFree(h->ar_count);
  for (int k = 0; k < cqk_handle::kRing; ++k) {
    if (h->ring[k]) cudaFreeHost(h->ring[k]);
    if (h->ring_ev[k]) cudaEventDestroy(h->ring_ev[k]);
  }
  if (h->host_state) cudaFreeHost(h->host_state);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->own) cudaStreamDestroy(h->own);
  delete h;
  return 0;
}

int cqk_set_stream(cqk_handle* h, void* stream) {
  if (!h) return set_err(CQK_E_ARG, "null handle");
  h->stream = stream ? (cudaStream_t)stream : h->own;
  return 0;
}

int cqk_device_info(cqk_handle* h, int32_t* sm_count, int32_t* ctas, int32_t* threads) {
  if (!h) return set_err(CQK_E_ARG, "null handle");
  if (sm_count) *sm_count = h->sm_count;
  if (ctas) *ctas = h->grid_cqk_fix;
  if (threads) *threads = kThreads;
  return 0;
}

int cqk_get_timeline(cqk_handle* h, long long* out, int32_t max_rows) {
  if (!h || !out) return set_err(CQK_E_ARG, "null argument");
  cudaSetDevice(h->device);
  int rows = max_rows < kTimelineCap ? max_rows : kTimelineCap;
  CUDA_TRY(cudaMemcpy(out, h->timeline, sizeof(long long) * kTimelineCols * rows,
                      cudaMemcpyDeviceToHost));
  return rows;
}

int cqk_get_trace(cqk_handle* h, double* out, int32_t max_rows) {
  if (!h || !out) return set_err(CQK_E_ARG, "null argument");
  cudaSetDevice(h->device);
  int rows = h->trace_len < max_rows ? h->trace_len : max_rows;
  if (rows > 0) CUDA_TRY(cudaMemcpy(out, h->trace, sizeof(double) * 4 * rows, cudaMemcpyDeviceToHost));
  return rows;
}

}  // extern "C"

// ------------------------------------------------------------ helpers
namespace {

double tau_of(const cqk_options* o, bool f32) {
  if (o && o->tolerance_scale > 0) return o->tolerance_scale;
  const double eps = f32 ? (double)std::numeric_limits<float>::epsilon()
                         : std::numeric_limits<double>::epsilon();
  return std::pow(eps, 0.75);
}

cqk_options default_opts() {
  cqk_options o;
  std::memset(&o, 0, sizeof o);
  o.variable_fixing = 1;
  o.max_iterations = 100;
  o.tolerance_scale = NAN;
  o.variant = CQK_VARIANT_SOLVE;
  o.check = 1;
  o.lambda0 = NAN;
  o.compact_ratio = NAN;
  o.simplex_start = 4;
  return o;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

int ensure_ring(cqk_handle* h) {
  for (int k = 0; k < cqk_handle::kRing; ++k) {
    if (!h->ring[k]) CUDA_TRY(cudaMallocHost(&h->ring[k], cqk_handle::kRingBytes));
    if (!h->ring_ev[k]) CUDA_TRY(cudaEventCreateWithFlags(&h->ring_ev[k], cudaEventDisableTiming));
  }
  return 0;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const int64_t nt = omp_get_max_threads() < 8 ? omp_get_max_threads() : 8;
  const size_t part = (bytes / nt + 63) / 64 * 64;
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t t = 0; t < nt; ++t) {
    const size_t o = (size_t)t * part;
    if (o < bytes) std::memcpy((char*)dst + o, (const char*)src + o, o + part < bytes ? part : bytes - o);
  }
}

// Pageable host -> device: memcpy chunks into the pinned ring (several host
// threads) while the copy engine moves the previous chunk (~3-4x the
// driver's own pageable path on this class of host).  Pinned memory goes
// straight to cudaMemcpyAsync.
int h2d(cqk_handle* h, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return 0;
  if (bytes < (1u << 20) || is_pinned(src)) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
    return 0;
  }
  int rc = ensure_ring(h);
  if (rc) return rc;
  for (size_t off = 0, k = 0; off < bytes; off += cqk_handle::kRingBytes, ++k) {
    const int s = (int)(k % cqk_handle::kRing);
    const size_t len = bytes - off < cqk_handle::kRingBytes ? bytes - off : cqk_handle::kRingBytes;
    CUDA_TRY(cudaEventSynchronize(h->ring_ev[s]));  // the slot's previous copy is done
    par_memcpy(h->ring[s], (const char*)src + off, len);
    CUDA_TRY(cudaMemcpyAsync((char*)dst + off, h->ring[s], len, cudaMemcpyHostToDevice, h->stream));
    CUDA_TRY(cudaEventRecord(h->ring_ev[s], h->stream));
  }
  return 0;
}

// Device -> pageable host, the mirror image (enqueued work on the stream
// completes first; the caller's buffer is complete on return).
int d2h(cqk_handle* h, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return 0;
  if (bytes < (1u << 20) || is_pinned(dst)) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
    return 0;
  }
  int rc = ensure_ring(h);
  if (rc) return rc;
  const size_t R = cqk_handle::kRingBytes;
  const size_t nchunks = (bytes + R - 1) / R;
  auto launch = [&](size_t k) -> int {
    const int s = (int)(k % cqk_handle::kRing);
    const size_t off = k * R, len = bytes - off < R ? bytes - off : R;
    CUDA_TRY(cudaMemcpyAsync(h->ring[s], (const char*)src + off, len, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaEventRecord(h->ring_ev[s], h->stream));
    return 0;
  };
  for (size_t k = 0; k < nchunks && k < (size_t)cqk_handle::kRing; ++k)
    if ((rc = launch(k))) return rc;
  for (size_t k = 0; k < nchunks; ++k) {
    const int s = (int)(k % cqk_handle::kRing);
    const size_t off = k * R, len = bytes - off < R ? bytes - off : R;
    CUDA_TRY(cudaEventSynchronize(h->ring_ev[s]));
    par_memcpy((char*)dst + off, h->ring[s], len);
    if (k + cqk_handle::kRing < nchunks && (rc = launch(k + cqk_handle::kRing))) return rc;
  }
  return 0;
}

// Host-mode staging: copy `count` host arrays of n T into one device slab.
template <typename T>
int stage_inputs(cqk_handle* h, int mem, int64_t n, const T* const* in, int count,
                 const T** dev, int extra_out, T** dev_out) {
  if (mem == CQK_MEM_DEVICE) {
    for (int i = 0; i < count; ++i) dev[i] = in[i];
    return 0;
  }
  const size_t per = ((size_t)n * sizeof(T) + 255) / 256 * 256;
  CUDA_TRY(h->stage.ensure(per * (count + extra_out)));
  char* base = (char*)h->stage.p;
  for (int i = 0; i < count; ++i) {
    if (!in[i]) { dev[i] = nullptr; continue; }
    T* d = (T*)(base + per * i);
    int rc = h2d(h, d, in[i], (size_t)n * sizeof(T));
    if (rc) return rc;
    dev[i] = d;
  }
  for (int j = 0; j < extra_out; ++j) dev_out[j] = (T*)(base + per * (count + j));
  return 0;
}

// Compact when the logically fixed, physically present elements reach this
// share of the working set (CQK_COMPACT_RATIO overrides).  Measured on the C3
// families (n = 1e8): with the TMA engine 0.5 streams 2-5% fewer bytes and is
// fastest (weak 3.99 -> 3.88 ms, corr 4.26 -> 3.88 ms); the warp-segment
// engine (small n) keeps 0.25.
// Once the direction guess's survivors are adopted the working set is
// already compacted once, and 0.4 compacts it once more (tools/policy_ab.py,
// 36 instances 5e6..1e8: 0.4 the best mean, 0.5 leaves C3 weak seed 1
// uncompacted at 3.36 ms against 3.23); without adoption 0.5 stays.
double default_compact_ratio(bool tma = false, bool adopted = false) {
  static double v = [] {
    const char* e = getenv("CQK_COMPACT_RATIO");
    return e ? atof(e) : -1.0;
  }();
  return v >= 0 ? v : (tma ? (adopted ? 0.4 : 0.5) : 0.25);
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }



int finish_sync(cqk_handle* h) {
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return set_err(CQK_E_CUDA, std::string("solve: ") + cudaGetErrorString(e));
  return 0;
}

// The barrier-timeout flag travels back inside the published state (no copy
// on the solve stream, no legacy-stream or device-wide synchronisation, so
// several handles can run concurrent persistent kernels, e.g. virtual ranks on
// one GPU).  A state still RUNNING was never published: the grid aborted.
int check_timeout(cqk_handle* h, int32_t status, int32_t err) {
  const bool any_cta = *h->host_err != 0;  // a CTA that timed out alone (its rows unwritten)
  *h->host_err = 0;
  if (status != ST_RUNNING && !err && !any_cta) return 0;
  cudaMemsetAsync(h->sync, 0, 64, h->stream);
  cudaMemsetAsync(h->ar_count, 0, 64, h->stream);
  cudaMemsetAsync(h->hist, 0, sizeof(int32_t) * 2 * kHistB, h->stream);  // may hold a partial scan
  cudaStreamSynchronize(h->stream);
  return set_err(CQK_E_TIMEOUT, "persistent kernel barrier timed out");
}

// The masterless grid step for a single-GPU persistent TMA launch of `grid`
// CTAs (one CTA per SM; the buffers hold sm_count + 8 rows).
GridAR masterless(cqk_handle* h, int grid, const Exchange& ex) {
  GridAR ar{nullptr, 0ull, nullptr, nullptr, 0};
  if (grid > h->sm_count + 8 || h->master_step) return ar;
  const int k = (int)(h->ar_seq++ & 1u);
  ar.tag = h->ar_seq << 32;  // unique per launch of this handle (rows carry it)
  ar.rows = h->ar_rows;
  ar.tiles = h->ar_count + 2 + k;
  ar.tiles_next = h->ar_count + 2 + (k ^ 1);
  ar.dyn_final = !h->static_final;
  return ar;
}

int map_status(int32_t st) {
  switch (st) {
    case ST_SOLVED: return CQK_SOLVED;
    case ST_INFEASIBLE: return CQK_INFEASIBLE;
    case ST_DOMAIN: return CQK_E_DOMAIN;
    case ST_MAXITER: return CQK_E_MAXITER;
    case ST_CONTRACT: return CQK_E_CONTRACT;
    default: return CQK_E_CUDA;
  }
}

int util_blocks(cqk_handle* h, int64_t m) {
  int64_t b = (m + kUtilThreads - 1) / kUtilThreads;
  int64_t cap = (int64_t)h->sm_count * 8;
  if (cap > kUtilBlocksMax) cap = kUtilBlocksMax;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

// Copy an optional index list to the device.
int stage_idx(cqk_handle* h, int mem, const int64_t* idx, int64_t m, const int64_t** out) {
  if (!idx || mem == CQK_MEM_DEVICE) { *out = idx; return 0; }
  CUDA_TRY(h->idxbuf.ensure(sizeof(int64_t) * (m ? m : 1)));
  CUDA_TRY(cudaMemcpyAsync(h->idxbuf.p, idx, sizeof(int64_t) * m, cudaMemcpyHostToDevice, h->stream));
  *out = (const int64_t*)h->idxbuf.p;
  return 0;
}

}  // namespace

// ------------------------------------------------------------ communicator
namespace {
int limit_grid(const cqk_handle* h, int grid) {
  return h->grid_limit > 0 && h->grid_limit < grid ? h->grid_limit : grid;
}
Exchange make_exchange(cqk_handle* h, bool sharded) {
  Exchange ex;
  std::memset(&ex, 0, sizeof ex);
  ex.world = sharded ? h->world : 1;
  ex.rank = sharded ? h->rank : 0;
  ex.mbox = h->mbox;
  for (int q = 0; q < kMaxRanks; ++q) ex.peer[q] = h->peers[q];
  if (sharded) ex.seq = ++h->seq;
  return ex;
}
}  // namespace

extern "C" int cqk_reserve(cqk_handle* h, int64_t n) {
  if (!h || n < 0) return set_err(CQK_E_ARG, "bad reserve");
  CUDA_TRY(cudaSetDevice(h->device));
  const size_t per = ((size_t)tma_scratch_elems(n) * sizeof(double) + 255) / 256 * 256;
  CUDA_TRY(h->scratch.ensure(per * 10));  // compaction + side-list scratch (fused start)
  CUDA_TRY(cudaDeviceSynchronize());
  return 0;
}

extern "C" int cqk_reserve_host(cqk_handle* h, int64_t n) {
  if (!h || n < 0) return set_err(CQK_E_ARG, "bad reserve");
  CUDA_TRY(cudaSetDevice(h->device));
  const size_t per = ((size_t)n * sizeof(double) + 255) / 256 * 256;
  CUDA_TRY(h->stage.ensure(per * 7));  // d, a, b, l, u, xbar + x
  if (int rc = ensure_ring(h)) return rc;
  CUDA_TRY(cudaDeviceSynchronize());
  return 0;
}

extern "C" int cqk_set_engine(cqk_handle* h, int mode) {
  if (!h || mode < 0 || mode > 2) return set_err(CQK_E_ARG, "engine: 0 auto, 1 tma, 2 segments");
  h->engine = mode;
  return 0;
}

extern "C" int cqk_set_fused(cqk_handle* h, int64_t min_n, double half_width) {
  if (!h || !(half_width >= 0.0)) return set_err(CQK_E_ARG, "fused start: half_width >= 0");
  h->fused_min_n = min_n;
  h->fused_width = half_width;
  return 0;
}

extern "C" int cqk_set_fused_guess(cqk_handle* h, int mode) {
  if (!h || mode < 0 || mode > 3) return set_err(CQK_E_ARG, "fused guess: mode 0..3");
  h->fused_guess = mode;
  return 0;
}

extern "C" int cqk_set_switches(cqk_handle* h, int flags) {
  if (!h) return set_err(CQK_E_ARG, "null handle");
  h->master_step = (flags & 1) != 0;
  h->static_final = (flags & 2) != 0;
  h->tail_mode = (flags & 4) == 0;
  h->spx_capture = (flags & 8) ? 0 : ((flags & 16) ? 2 : 1);
  return 0;
}

extern "C" int cqk_set_grid_limit(cqk_handle* h, int max_ctas) {
  if (!h) return set_err(CQK_E_ARG, "null handle");
  h->grid_limit = max_ctas;
  return 0;
}

extern "C" int cqk_comm_create(cqk_handle* h, int rank, int world, void* ipc_handle_out) {
  if (!h || world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    return set_err(CQK_E_ARG, "need 0 <= rank < world <= 8");
  CUDA_TRY(cudaSetDevice(h->device));
  if (!h->mbox) CUDA_TRY(cudaMalloc(&h->mbox, sizeof(double) * kMboxDoubles));
  // a fresh group restarts its solve sequence at 1: no flag of an earlier
  // group (e.g. one abandoned after a timeout) may survive to match it
  CUDA_TRY(cudaMemset(h->mbox, 0, sizeof(double) * kMboxDoubles));
  h->rank = rank;
  h->world = world;
  h->seq = 0;
  h->peers[rank] = h->mbox;
  if (ipc_handle_out) {
    cudaIpcMemHandle_t ih;
    CUDA_TRY(cudaIpcGetMemHandle(&ih, h->mbox));
    std::memcpy(ipc_handle_out, &ih, sizeof ih);
  }
  CUDA_TRY(cudaDeviceSynchronize());
  return 0;
}

extern "C" int cqk_comm_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

extern "C" int cqk_comm_connect(cqk_handle* h, const void* handles) {
  if (!h || !handles || !h->mbox) return set_err(CQK_E_ARG, "cqk_comm_create first");
  CUDA_TRY(cudaSetDevice(h->device));
  const char* hb = (const char*)handles;
  for (int q = 0; q < h->world; ++q) {
    if (q == h->rank) continue;
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, hb + q * sizeof(cudaIpcMemHandle_t), sizeof ih);
    void* ptr = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess));
    h->peers[q] = (double*)ptr;
    h->ipc_opened[q] = true;
  }
  return 0;
}

extern "C" int cqk_comm_connect_local(cqk_handle* h, cqk_handle* const* ranks, int world) {
  if (!h || !ranks || world != h->world) return set_err(CQK_E_ARG, "bad local rank table");
  for (int q = 0; q < world; ++q)
    if (!ranks[q] || !ranks[q]->mbox) return set_err(CQK_E_ARG, "peer without mailbox");
  // this rank's kernel stores into every peer's mailbox: a peer on another
  // device must be reachable (NVLink P2P) and mapped into this device's
  // address space before any solve
  CUDA_TRY(cudaSetDevice(h->device));
  for (int q = 0; q < world; ++q) {
    const int pd = ranks[q]->device;
    if (pd == h->device) continue;
    int can = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&can, h->device, pd));
    if (!can)
      return set_err(CQK_E_ARG, "device " + std::to_string(h->device) + " cannot access device " +
                                    std::to_string(pd) + " (no P2P): local groups need peer access");
    cudaError_t e = cudaDeviceEnablePeerAccess(pd, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return set_err(CQK_E_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
  }
  for (int q = 0; q < world; ++q) h->peers[q] = ranks[q]->mbox;
  return 0;
}

// ------------------------------------------------------------ CQK solve
template <typename T>
static int solve_impl(cqk_handle* h, int mem, const T* d, const T* a, const T* b, const T* l,
                      const T* u, int64_t n, int64_t offset, int64_t n_total, double r,
                      const cqk_options* opts_in, const T* xbar, T* x, cqk_result* res,
                      bool sharded);

extern "C" int cqk_solve_f64(cqk_handle* h, int mem, const double* d, const double* a,
                             const double* b, const double* l, const double* u, int64_t n,
                             double r, const cqk_options* opts_in, const double* xbar, double* x,
                             cqk_result* res) {
  return solve_impl(h, mem, d, a, b, l, u, n, 0, n, r, opts_in, xbar, x, res, false);
}

extern "C" int cqk_solve_sharded_f64(cqk_handle* h, int mem, const double* d, const double* a,
                                     const double* b, const double* l, const double* u,
                                     int64_t n_local, int64_t offset, int64_t n_total, double r,
                                     const cqk_options* opts, const double* xbar, double* x,
                                     cqk_result* res) {
  if (!h || h->world < 1 || !h->mbox) return set_err(CQK_E_ARG, "communicator not set up");
  return solve_impl(h, mem, d, a, b, l, u, n_local, offset, n_total, r, opts, xbar, x, res, true);
}

extern "C" int cqk_solve_f32(cqk_handle* h, int mem, const float* d, const float* a,
                             const float* b, const float* l, const float* u, int64_t n, double r,
                             const cqk_options* opts_in, const float* xbar, float* x,
                             cqk_result* res) {
  return solve_impl<float>(h, mem, d, a, b, l, u, n, 0, n, r, opts_in, xbar, x, res, false);
}

// T = double: the TMA engine (n >= tma_min_n) or the warp-segment kernel;
// T = float: the warp-segment kernel with the element math in float (the
// reference computes t, x, b x of a float32 instance in float32, core.py:195-200)
// and fp64 accumulation.
template <typename T>
static int solve_impl(cqk_handle* h, int mem, const T* d, const T* a, const T* b, const T* l,
                      const T* u, int64_t n, int64_t offset, int64_t n_total, double r,
                      const cqk_options* opts_in, const T* xbar, T* x, cqk_result* res,
                      bool sharded) {
  constexpr bool F64 = std::is_same<T, double>::value;
  if (!h || !d || !a || !b || !l || !u || !res) return set_err(CQK_E_ARG, "null argument");
  std::memset(res, 0, sizeof *res);
  res->domain_index = -1;
  res->lam = NAN;
  cqk_options opts = opts_in ? *opts_in : default_opts();
  CUDA_TRY(cudaSetDevice(h->device));
  if (n_total < 1 || (!sharded && n < 1)) {  // validate(): at least one variable
    if (opts.check) {
      res->status = CQK_E_DOMAIN;
      res->domain_field = CQK_F_D;
      return CQK_E_DOMAIN;
    }
    return set_err(CQK_E_ARG, "n must be >= 1");
  }
  const bool jacobi = opts.variant == CQK_VARIANT_JACOBI;
  const bool fixing = !jacobi && opts.variable_fixing;
  const T* dv[6];
  T* xo = x;
  T* xdev = nullptr;
  {
    const T* in[6] = {d, a, b, l, u, xbar};
    int rc = stage_inputs<T>(h, mem, n, in, 6, dv, (mem == CQK_MEM_HOST && x) ? 1 : 0, &xdev);
    if (rc) return rc;
    if (mem == CQK_MEM_HOST) xo = x ? xdev : nullptr;
  }
  for (int i = 0; i < 5; ++i)
    if (!aligned16(dv[i])) return set_err(CQK_E_ARG, "device arrays must be 16-byte aligned");
  if (xbar && !aligned16(dv[5])) return set_err(CQK_E_ARG, "xbar must be 16-byte aligned");
  if (xo && !aligned16(xo)) return set_err(CQK_E_ARG, "x must be 16-byte aligned");

  CqkState s;
  std::memset(&s, 0, sizeof s);
  const bool lam0_given = !std::isnan(opts.lambda0);
  s.cmd.lam = lam0_given ? opts.lambda0 : 0.0;
  s.cmd.fix_hi = INFINITY;
  s.cmd.fix_lo = -INFINITY;
  s.cmd.phase = (opts.check || !lam0_given) ? PH_LAMBDA0 : PH_SCAN;
  s.lo = -INFINITY;
  s.hi = INFINITY;
  s.r_res = r;
  s.r_orig = r;
  s.tau = tau_of(&opts, !F64);
  s.lam0 = s.cmd.lam;
  s.fhi_phys = INFINITY;  // the original arrays: nothing removed yet
  s.flo_phys = -INFINITY;
  s.max_iter = opts.max_iterations;
  s.n = n_total;
  s.phys_count = n;
  s.fixing = fixing;
  s.variant = opts.variant;
  s.status = ST_RUNNING;
  s.has_xbar = xbar != nullptr;
  s.check = opts.check;
  s.domain_index = -1;
  s.trace_cap = opts.record_trace ? kTraceCap : 0;
  s.lam0_given = lam0_given;
  // engine: the TMA pipeline wins at every measured size since the producer
  // warp left the reduction shuffles and the grid step lost its master
  // (tools/crossover.py: 70 vs 72 us at 5e4 ... 0.65 vs 0.82 ms at 1.6e7);
  // below 64Ki elements the two tie, and the warp-segment kernel's summation
  // order reproduces the reference's iterate counts on tiny inputs more often
  const bool tma = F64 && h->use_tma && (h->engine == 1 || (h->engine == 0 && n >= h->tma_min_n));
  // fused start (cqk_tma.cuh): lambda0 and the first scan share one pass
  // (a per-rank size every rank derives alike: the phases must match across ranks)
  const int64_t per_rank = sharded ? n_total / std::max(h->world, 1) : n;
  const bool fused = tma && !lam0_given && !xbar && per_rank >= h->fused_min_n;
  // the direction guess's extra sample epoch (~12 us) pays from ~1e7 elements
  // per rank (tools/policy_ab.py: 1e7 -1.7% mean, 1e8 -4.2%; 5e6 +1.5%);
  // the forced modes (tests) apply at any size
  const int guess = !(fused && fixing) ? 0
                    : (h->fused_guess >= 2 || per_rank >= cqk_handle::kGuessMinN) ? h->fused_guess : 0;
  s.compact_ratio = std::isnan(opts.compact_ratio) ? default_compact_ratio(tma) : opts.compact_ratio;
  s.compact_ratio_adopt =
      std::isnan(opts.compact_ratio) ? default_compact_ratio(tma, true) : opts.compact_ratio;
  if (fused) {
    s.fused = 1;
    s.fused_guess = guess;
    s.fused_width = h->fused_width;
    s.cmd.phase = PH_SAMPLE;
  }
  // scratch: n per array (warp segments) or whole tile slots (TMA engine)
  const size_t per = ((size_t)(tma ? tma_scratch_elems(n) : n) * sizeof(T) + 255) / 256 * 256;
  // fused start: the side list gets its own five arrays behind the compaction
  // scratch (the fused pass also writes its guessed survivors into the latter)
  if (fixing || fused) CUDA_TRY(h->scratch.ensure(per * (fused ? 10 : 5)));
  std::memcpy(h->host_state, &s, sizeof s);  // status RUNNING until the master publishes
  CqkParams<T> p;
  std::memset(&p, 0, sizeof p);
  p.init = s;
  p.out = (CqkState*)h->host_state_dev;
  p.d = dv[0]; p.a = dv[1]; p.b = dv[2]; p.l = dv[3]; p.u = dv[4]; p.xbar = xbar ? dv[5] : nullptr;
  if (fixing) {
    char* sb = (char*)h->scratch.p;
    p.sd = (T*)(sb); p.sa = (T*)(sb + per); p.sb = (T*)(sb + 2 * per);
    p.sl = (T*)(sb + 3 * per); p.su = (T*)(sb + 4 * per);
  }
  if (fused) {
    char* sb = (char*)h->scratch.p + 5 * per;
    p.vd = (T*)(sb); p.va = (T*)(sb + per); p.vb = (T*)(sb + 2 * per);
    p.vl = (T*)(sb + 3 * per); p.vu = (T*)(sb + 4 * per);
  }
  p.x = xo;
  p.trace = h->trace;
  p.n = n;
  p.offset = offset;
  p.r = r;
  p.st = (CqkState*)h->state;
  p.ex = make_exchange(h, sharded);
  p.partials = h->partials;
  p.sync.arrive = h->sync;
  p.sync.gen = h->sync + 1;
  p.sync.error = (int*)(h->sync + 2);
  p.sync.timeline = h->timeline;
  p.sync.herr = h->host_err_dev;
  void* args[] = {&p};
  int grid;
  const void* fn;
  if constexpr (F64) {
    if (tma) {
      grid = limit_grid(h, fixing ? h->grid_tma_fix : h->grid_tma_jac);
      fn = fixing ? (const void*)cqk_tma_kernel<true> : (const void*)cqk_tma_kernel<false>;
      p.ar = masterless(h, grid, p.ex);
    } else {
      grid = limit_grid(h, fixing ? h->grid_cqk_fix : h->grid_cqk_jac);
      fn = fixing ? (const void*)cqk_solve_kernel<double, true>
                  : (const void*)cqk_solve_kernel<double, false>;
    }
  } else {
    grid = limit_grid(h, fixing ? h->grid_cqk_fix32 : h->grid_cqk_jac32);
    fn = fixing ? (const void*)cqk_solve_kernel<float, true> : (const void*)cqk_solve_kernel<float, false>;
  }
  CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
  CUDA_TRY(cudaLaunchCooperativeKernel(fn, grid, tma ? kTmaThreads : kThreads, args,
                                       tma ? kSmemC : 0, h->stream));
  CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
  if (mem == CQK_MEM_HOST && x && xo)
  {
    int rc_ = d2h(h, x, xo, sizeof(T) * n);
    if (rc_) return rc_;
  }
  int rc = finish_sync(h);
  if (rc) return rc;
  std::memcpy(&s, h->host_state, sizeof s);
  rc = check_timeout(h, s.status, s.err);
  if (rc) return rc;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  h->trace_len = s.trace_len;
  res->status = map_status(s.status);
  res->domain_field = s.domain_field;
  res->domain_index = s.domain_index;
  res->lam = s.status == ST_SOLVED ? s.cmd.lam : (s.status == ST_MAXITER ? s.cmd.lam : NAN);
  res->lam0 = s.lam0;
  res->iterations = s.iterations;
  res->phi_evals = s.phi_evals;
  res->fixed_count = s.fixed_count;
  res->bracket_lo = s.lo;
  res->bracket_hi = s.hi;
  // fused start: no pass 0; the sample reads 24 B per sampled element
  const int64_t pass0 = s.fused ? s.elems_sample : ((opts.check || !lam0_given) ? n : 0);
  constexpr int64_t E = sizeof(T);         // bytes per array element
  const int64_t bytes0 = xbar ? 6 * E : 3 * E;  // l, u are validated on the first scan
  const int64_t fin = (s.status == ST_SOLVED && xo) ? n : 0;
  res->elems_read = pass0 + s.elems_scan + s.elems_bp + fin;
  res->elems_written = s.elems_written + fin;
  res->bytes_model = pass0 * bytes0 + 5 * E * (s.elems_scan + s.elems_bp + s.elems_written) + 6 * E * fin;
  res->device_ms = ms;
  res->launches = 1;
  res->trace_len = s.trace_len;
  return res->status;
}

// ------------------------------------------------------------ simplex / l1
namespace {

// Enqueue one persistent simplex / l1 solve (state H2D, launch, state and
// timeout flag D2H) on the handle's stream; the caller synchronises.
template <typename T>
int launch_spx(cqk_handle* h, SpxState& s, const T* yv, int64_t n, T* xo, bool l1, bool sharded) {
  constexpr bool F64 = std::is_same<T, double>::value;
  const bool tma = F64 && h->use_tma;
  // scratch: working values; with the capture start also the captured
  // elements' indices and (l1) the sign bits of y
  const size_t per_y = ((size_t)(tma ? tma_scratch_elems_y(n) : n) * sizeof(T) + 255) / 256 * 256;
  const size_t per_i = s.fused ? ((size_t)tma_scratch_elems_y(n) * 8 + 255) / 256 * 256 : 0;
  // (the sign bits serve the dense sparse-final only)
  const size_t per_s = s.fused && l1 && !h->sparse_req ? ((size_t)tma_scratch_elems_y(n) / 8 + 255) / 256 * 256 : 0;
  if (s.fixing) CUDA_TRY(h->scratch.ensure(per_y + per_i + per_s));
  std::memcpy(h->host_state, &s, sizeof s);  // status RUNNING until the master publishes
  SpxParams<T> p;
  std::memset(&p, 0, sizeof p);
  p.init = s;
  p.out = (SpxState*)h->host_state_dev;
  p.y = yv;
  p.sy = s.fixing ? (T*)h->scratch.p : nullptr;
  p.sidx = per_i ? (int64_t*)((char*)h->scratch.p + per_y) : nullptr;
  p.signs = per_s ? (uint32_t*)((char*)h->scratch.p + per_y + per_i) : nullptr;
  if (h->sparse_req) {
    p.out_idx = h->sparse_req->idx;
    p.out_val = h->sparse_req->val;
    p.out_cnt = h->sparse_req->cnt;
    p.out_cap = h->sparse_req->cap;
  }
  p.x = xo;
  p.trace = h->trace;
  p.n = n;
  p.st = (SpxState*)h->state;
  p.ex = make_exchange(h, sharded);
  p.partials = h->partials;
  p.sync.arrive = h->sync;
  p.sync.gen = h->sync + 1;
  p.sync.error = (int*)(h->sync + 2);
  p.sync.timeline = h->timeline;
  p.sync.herr = h->host_err_dev;
  {
    p.wcnt = (tma && !sharded && h->tail_mode) ? h->wcnt : nullptr;
    if (tma && !sharded && s.hist_ok) {  // the halves alternate: this one is zero
      p.hist = h->hist + h->hist_flip * kHistB;
      p.hist_next = h->hist + (h->hist_flip ^ 1) * kHistB;
      h->hist_flip ^= 1;
    }
  }
  void* args[] = {&p};
  int grid;
  const void* fn;
  if constexpr (F64) {
    if (tma) {
      grid = limit_grid(h, l1 ? h->grid_tma_l1 : h->grid_tma_spx);
      fn = l1 ? (const void*)spx_tma_kernel<true> : (const void*)spx_tma_kernel<false>;
      p.ar = masterless(h, grid, p.ex);
    } else {
      grid = limit_grid(h, l1 ? h->grid_l1 : h->grid_spx);
      fn = l1 ? (const void*)spx_solve_kernel<double, true> : (const void*)spx_solve_kernel<double, false>;
    }
  } else {
    grid = limit_grid(h, l1 ? h->grid_l1_32 : h->grid_spx32);
    fn = l1 ? (const void*)spx_solve_kernel<float, true> : (const void*)spx_solve_kernel<float, false>;
  }
  CUDA_TRY(cudaLaunchCooperativeKernel(fn, grid, tma ? kTmaThreads : kThreads, args,
                                       tma ? kSmemC : 0, h->stream));
  return 0;
}

// Chunked Algorithm 2 (par_simplex_init semantics) on the device: W chunks,
// merged lambda0, gathered free set.  Results stay in h->alg2; `out` is the
// merged summary (copied back, stream synchronised).
int run_alg2(cqk_handle* h, const double* yv, const int64_t* idx, int64_t p, double r, int64_t W,
             const double* xbar, int sharpened, bool l1, bool want_vals, bool want_idx,
             uint8_t* fixed_dev, Alg2Out* out) {
  if (W < 1) {  // auto: chunks of >= 256 elements (a chunk must be long enough
                // for its multiplier to prove zeros), at most one per GPU thread
    W = p / h->alg2_chunk;
    if (W > (int64_t)h->sm_count * 1024) W = (int64_t)h->sm_count * 1024;
    if (W < 1) W = 1;
  }
  if (W > p) W = p;
  const size_t nb = ((size_t)p * 4 + 255) / 256 * 256, wb = ((size_t)W * 8 + 255) / 256 * 256;
  const size_t vb = ((size_t)p * 8 + 255) / 256 * 256;
  const size_t total = 2 * nb + 8 * wb + (want_vals ? vb : 0) + (want_idx ? vb : 0) + 256;
  CUDA_TRY(h->alg2.ensure(total));
  char* base = (char*)h->alg2.p;
  int32_t* J = (int32_t*)base;
  int32_t* Jt = (int32_t*)(base + nb);
  double* sums = (double*)(base + 2 * nb);
  double* sumabs = (double*)(base + 2 * nb + wb);
  double* scratch = (double*)(base + 2 * nb + 2 * wb);  // 2 W doubles
  int64_t* cards = (int64_t*)(base + 2 * nb + 4 * wb);
  int64_t* jplus = (int64_t*)(base + 2 * nb + 5 * wb);
  int64_t* offsets = (int64_t*)(base + 2 * nb + 6 * wb);
  double* lams = (double*)(base + 2 * nb + 7 * wb);
  char* tail = base + 2 * nb + 8 * wb;
  double* vals = want_vals ? (double*)tail : nullptr;
  if (want_vals) tail += vb;
  int64_t* gidx = want_idx ? (int64_t*)tail : nullptr;
  if (want_idx) tail += vb;
  Alg2Out* dout = (Alg2Out*)tail;
  h->alg2_vals = vals;
  h->alg2_idx = gidx;
  const int blocks = (int)((W + 255) / 256);
  if (l1)
    alg2_chunks_kernel<true><<<blocks, 256, 0, h->stream>>>(yv, idx, p, r, W, xbar, sharpened, J,
                                                            Jt, fixed_dev, sums, cards, jplus, sumabs, lams);
  else
    alg2_chunks_kernel<false><<<blocks, 256, 0, h->stream>>>(yv, idx, p, r, W, xbar, sharpened, J,
                                                             Jt, fixed_dev, sums, cards, jplus, sumabs,
                                                             lams);
  alg2_merge_kernel<<<1, 1024, 0, h->stream>>>(sums, l1 ? sumabs : nullptr, cards, lams, W, r,
                                               scratch, offsets, dout);
  if (want_vals || want_idx) {
    if (l1)
      alg2_gather_kernel<true><<<blocks, 256, 0, h->stream>>>(yv, idx, p, W, J, cards, offsets,
                                                              vals, gidx);
    else
      alg2_gather_kernel<false><<<blocks, 256, 0, h->stream>>>(yv, idx, p, W, J, cards, offsets,
                                                               vals, gidx);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(h->host_state, dout, sizeof(Alg2Out), cudaMemcpyDeviceToHost, h->stream));
  // total jplus (for the xbar fallback of simplex_init_lambda) into host_state tail
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  std::memcpy(out, h->host_state, sizeof(Alg2Out));
  h->alg2_w = W;
  h->alg2_jplus = jplus;
  return 0;
}

// T = float: the warp-segment kernel with y + lam in float (simplex.py:207-215)
// and the formula / tight starts (the device Algorithm 2 is fp64-only).
template <typename T>
int spx_common(cqk_handle* h, int mem, const T* y, int64_t n, int64_t n_total, double r,
               const cqk_options* opts_in, T* x, cqk_result* res, bool l1, bool sharded,
               const T* xbar = nullptr, int sharpened = -1) {
  constexpr bool F64 = std::is_same<T, double>::value;
  if (!h || !y || !res) return set_err(CQK_E_ARG, "null argument");
  std::memset(res, 0, sizeof *res);
  res->domain_index = -1;
  res->lam = NAN;
  cqk_options opts = opts_in ? *opts_in : default_opts();
  CUDA_TRY(cudaSetDevice(h->device));
  if (!(r > 0)) {  // simplex.py:234-235, 322-323
    res->status = CQK_E_DOMAIN;
    res->domain_field = CQK_F_R;
    return CQK_E_DOMAIN;
  }
  if (n_total < 1 || (!sharded && n < 1)) return set_err(CQK_E_ARG, "n must be >= 1");
  const T* yv;
  const T* xbv = nullptr;
  T* xdev = nullptr;
  T* xo = x;
  {
    const T* in[2] = {y, xbar};
    const T* dv[2] = {nullptr, nullptr};
    int rc = stage_inputs<T>(h, mem, n, in, 2, dv, (mem == CQK_MEM_HOST && x) ? 1 : 0, &xdev);
    if (rc) return rc;
    yv = dv[0];
    xbv = xbar ? dv[1] : nullptr;
    if (mem == CQK_MEM_HOST) xo = x ? xdev : nullptr;
  }
  if (!aligned16(yv) || (xo && !aligned16(xo)))
    return set_err(CQK_E_ARG, "device arrays must be 16-byte aligned");
  const bool fixing = opts.variable_fixing != 0;
  // the Algorithm-2 route: start "alg2", or a warm start (xbar, simplex.py:65-109)
  const bool alg2 = F64 && (opts.simplex_start == 2 || xbv) && !sharded && std::isnan(opts.lambda0);
  SpxState s;
  std::memset(&s, 0, sizeof s);
  s.cmd.fix_hi = INFINITY;
  s.cmd.fix_lo = -INFINITY;
  s.cmd.phase = PH_LAMBDA0;
  s.lo = -INFINITY;
  s.hi = INFINITY;
  s.r = r;
  s.tau = tau_of(&opts, !F64);
  s.n = n_total;
  s.active = n_total;
  s.local_active = n;
  s.phys_count = n;
  s.max_iter = opts.max_iterations;
  s.fixing = fixing;
  s.status = ST_RUNNING;
  s.l1 = l1;
  s.lam0_given = !std::isnan(opts.lambda0);
  s.lam0_value = opts.lambda0;
  s.trace_cap = opts.record_trace ? kTraceCap : 0;
  s.compact_ratio = std::isnan(opts.compact_ratio) ? default_compact_ratio() : opts.compact_ratio;
  s.start = (!F64 && opts.simplex_start == 2) ? 1 : opts.simplex_start;  // float: alg2 -> tight
  // start "auto": the histogram scan costs ~10% of one pass and saves grid
  // epochs; it pays while epochs dominate (measured: u01 1e6 139 -> 81 us; at
  // 1e9 the tail mode already makes the late epochs cheap and it costs 2%)
  s.hist_ok = F64 && h->use_tma && !sharded && n <= 30000000;
  s.lam_hist = NAN;
  s.cap_first = F64 && h->use_tma && h->spx_capture;  // the first scan captures (s_after_init)
  // capture start (cqk_kernels.cuh s_after_sample / s_after_fused): pass 0 and
  // the first scan share one pass that captures the possible support; for an
  // upper-bound start (formula / tight / auto) on the TMA engine, with fixing
  {
    const int64_t per_rank = sharded ? n_total / std::max(h->world, 1) : n;
    const bool ub_start = s.start == 0 || s.start == 1 || s.start == 4;
    if (F64 && h->use_tma && !alg2 && !s.lam0_given && fixing && ub_start && h->spx_capture &&
        per_rank >= h->spx_capture_min_n) {
      s.fused = h->spx_capture;  // 2: an impossible threshold (tests the fallback)
      s.cmd.phase = PH_SAMPLE;
      // ("auto": the histogram rides on the first scan over the captured
      // list; a list small enough for the tail mode iterates without it)
    }
  }
  int launches = 1;
  int64_t extra_read = 0;
  CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
  if constexpr (!F64) {
    int rc = launch_spx<T>(h, s, yv, n, xo, l1, sharded);
    if (rc) return rc;
  } else if (alg2) {
    // simplex.py:243-245 with the chunked initializer: Algorithm 4 then runs
    // on the gathered free set (values only) and x is one dense pass.
    Alg2Out a2;
    const int sharp = sharpened >= 0 ? sharpened : (l1 ? 1 : 0);
    // chunks without a warm start (every chunk multiplier bounds the root,
    // par_simplex_init); with xbar the sequential recurrence exactly as
    // simplex_init_lambda runs it (its no-support fallback is global), and
    // the free set is ~fixed_mask (wider than the initializer's set J)
    uint8_t* mask = nullptr;
    double* wvals = nullptr;
    int64_t* wcount = nullptr;
    if (xbv) {
      const size_t mb = ((size_t)n + 255) / 256 * 256, vb = ((size_t)n * 8 + 255) / 256 * 256;
      CUDA_TRY(h->warm.ensure(mb + vb + 256));
      mask = (uint8_t*)h->warm.p;
      wvals = (double*)((char*)h->warm.p + mb);
      wcount = (int64_t*)((char*)h->warm.p + mb + vb);
      CUDA_TRY(cudaMemsetAsync(mask, 0, n, h->stream));
    }
    int64_t W = xbv ? 1 : 0;
    if (sharp && !l1 && !xbv) {
      // sharpened with y[0] <= 0: whether the sequential recurrence later
      // fixes its seed depends on the whole pass, so run it exactly (one chunk)
      double y0 = 0.0;
      CUDA_TRY(cudaMemcpyAsync(&y0, yv, sizeof y0, cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(cudaStreamSynchronize(h->stream));
      if (!(y0 > 0.0)) W = 1;
    }
    int rc = run_alg2(h, yv, nullptr, n, r, W, xbv, sharp, l1, !xbv, false, mask, &a2);
    if (rc) return rc;
    if (xbv) {
      if (l1) spx_gather_free_kernel<true><<<1, 1024, 0, h->stream>>>(yv, mask, n, wvals, wcount);
      else spx_gather_free_kernel<false><<<1, 1024, 0, h->stream>>>(yv, mask, n, wvals, wcount);
      CUDA_TRY(cudaGetLastError());
      int64_t m = 0;
      CUDA_TRY(cudaMemcpyAsync(&m, wcount, sizeof m, cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(cudaStreamSynchronize(h->stream));
      a2.n_free = m;
      h->alg2_vals = wvals;
    }
    if (xbv) {  // simplex.py:151-152: no positive xbar component contributed
      int64_t jp = 0;
      CUDA_TRY(cudaMemcpy(&jp, h->alg2_jplus, sizeof jp, cudaMemcpyDeviceToHost));
      if (jp == 0) {
        double y0 = 0.0;
        CUDA_TRY(cudaMemcpy(&y0, yv, sizeof y0, cudaMemcpyDeviceToHost));
        if (l1) y0 = std::fabs(y0);
        a2.lam0 = std::max(r / (double)n, -y0);
      }
    }
    launches = 5;
    extra_read = n;
    if (l1 && a2.inside) {
      if (xo) spx_x_kernel<false><<<h->sm_count * 4, 256, 0, h->stream>>>(yv, n, 0.0, 1, xo);
      s.status = ST_SOLVED;
      s.iterations = -1;
      s.cmd.phase = PH_COPY;
    } else {
      const int64_t m = a2.n_free;
      s.cmd.phase = PH_LAMBDA0;  // one pass over the free set: r - max(w) tightens the start
      s.lam0_given = 1;
      s.lam0_value = a2.lam0;
      s.start = xbv ? 2 : 3;  // warm: the initializer's multiplier as is (simplex.py:243-245)
      s.n = m;
      s.active = m;
      s.local_active = m;
      s.phys_count = m;
      s.fixed_count = n - m;  // proven zero by the initializer (simplex.py:251)
      s.fixed_local = n - m;
      s.fixed_removed = n - m;
      rc = launch_spx<double>(h, s, h->alg2_vals, m, nullptr, false, false);
      if (rc) return rc;
      if (xo) {
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        std::memcpy(&s, h->host_state, sizeof s);
        if (l1) spx_x_kernel<true><<<h->sm_count * 4, 256, 0, h->stream>>>(yv, n, s.cmd.lam, 0, xo);
        else spx_x_kernel<false><<<h->sm_count * 4, 256, 0, h->stream>>>(yv, n, s.cmd.lam, 0, xo);
        CUDA_TRY(cudaGetLastError());
      }
    }
  } else {
    int rc = launch_spx(h, s, yv, n, xo, l1, sharded);
    if (rc) return rc;
  }
  CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
  if (mem == CQK_MEM_HOST && x && xo)
  {
    int rc_ = d2h(h, x, xo, sizeof(T) * n);
    if (rc_) return rc_;
  }
  int rc = finish_sync(h);
  if (rc) return rc;
  if (!(alg2 && s.iterations < 0)) std::memcpy(&s, h->host_state, sizeof s);
  rc = check_timeout(h, s.status, s.err);
  if (rc) return rc;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  h->trace_len = s.trace_len;
  res->status = map_status(s.status);
  res->lam = s.iterations < 0 ? NAN : s.cmd.lam;
  res->lam0 = s.lam0;
  res->iterations = s.iterations;
  res->phi_evals = s.phi_evals;
  res->fixed_count = s.fixed_count;
  res->bracket_lo = s.lo;
  res->bracket_hi = s.hi;
  const int64_t fin = (s.status == ST_SOLVED && xo) ? n : 0;
  const int64_t pass0 = alg2 ? extra_read : n;
  res->elems_read = pass0 + s.elems_scan + fin;
  res->elems_written = s.elems_written + fin;
  res->bytes_model = (int64_t)sizeof(T) * (pass0 + s.elems_scan + s.elems_written + 2 * fin);
  if (s.sparse_final && fin) {
    // x is written (8 B) without re-reading y; l1 writes and reads one sign
    // bit per element; each captured element: its index written by the fused
    // pass, then index + y read and x written by the scatter
    res->elems_read = pass0 + s.elems_scan + 2 * s.cap_local;
    res->bytes_model = (int64_t)sizeof(T) * (pass0 + s.elems_scan + s.elems_written + fin) +
                       (l1 ? 2 * ((n + 7) / 8) : 0) + 32 * s.cap_local;
  }
  res->device_ms = ms;
  res->launches = launches;
  res->trace_len = s.trace_len;
  return res->status;
}

}  // namespace

extern "C" int spx_project_f64(cqk_handle* h, int mem, const double* y, int64_t n, double r,
                               const cqk_options* opts, double* x, cqk_result* res) {
  return spx_common(h, mem, y, n, n, r, opts, x, res, false, false);
}

extern "C" int spx_project_f32(cqk_handle* h, int mem, const float* y, int64_t n, double r,
                               const cqk_options* opts, float* x, cqk_result* res) {
  return spx_common<float>(h, mem, y, n, n, r, opts, x, res, false, false);
}

extern "C" int l1_project_f32(cqk_handle* h, int mem, const float* y, int64_t n, double r,
                              const cqk_options* opts, float* x, cqk_result* res) {
  return spx_common<float>(h, mem, y, n, n, r, opts, x, res, true, false);
}

extern "C" int spx_project_sharded_f64(cqk_handle* h, int mem, const double* y, int64_t n_local,
                                       int64_t n_total, double r, const cqk_options* opts,
                                       double* x, cqk_result* res) {
  if (!h || !h->mbox) return set_err(CQK_E_ARG, "communicator not set up");
  return spx_common(h, mem, y, n_local, n_total, r, opts, x, res, false, true);
}

extern "C" int l1_project_sharded_f64(cqk_handle* h, int mem, const double* y, int64_t n_local,
                                      int64_t n_total, double r, const cqk_options* opts,
                                      double* x, cqk_result* res) {
  if (!h || !h->mbox) return set_err(CQK_E_ARG, "communicator not set up");
  return spx_common(h, mem, y, n_local, n_total, r, opts, x, res, true, true);
}

// Warm-started projections (simplex.py:218 / 311 with xbar): the Algorithm-2
// initializer seeded by the support of xbar (device chunks, par_simplex_init
// merge), Algorithm 4 on its free set.  xbar may be NULL (sharpened only).
extern "C" int spx_project_warm_f64(cqk_handle* h, int mem, const double* y, int64_t n, double r,
                                    const cqk_options* opts, const double* xbar, int sharpened,
                                    double* x, cqk_result* res) {
  cqk_options o = opts ? *opts : default_opts();
  o.simplex_start = 2;
  return spx_common(h, mem, y, n, n, r, &o, x, res, false, false, xbar, sharpened);
}

extern "C" int l1_project_warm_f64(cqk_handle* h, int mem, const double* y, int64_t n, double r,
                                   const cqk_options* opts, const double* xbar, double* x,
                                   cqk_result* res) {
  cqk_options o = opts ? *opts : default_opts();
  o.simplex_start = 2;
  return spx_common(h, mem, y, n, n, r, &o, x, res, true, false, xbar, 1);
}

extern "C" int l1_project_f64(cqk_handle* h, int mem, const double* y, int64_t n, double r,
                              const cqk_options* opts, double* x, cqk_result* res) {
  return spx_common(h, mem, y, n, n, r, opts, x, res, true, false);
}

// ------------------------------------------------------------ sparse output
// output="sparse" of newton_project_simplex / project_l1 (simplex.py:296-300,
// 328-331): the capture start's list holds every nonzero x, so the solve
// writes no dense x -- the kernel appends (index, value) pairs, which are
// sorted by index here (the reference's order).  Returns CQK_SPARSE_DENSE
// when the route does not apply (no adopted capture: small n, a large
// support, l1 inside the ball) and CQK_SPARSE_OVERFLOW (with *count) when
// more than cap entries are nonzero; the caller then takes the dense route.
extern "C" int spx_project_sparse_f64(cqk_handle* h, int mem, const double* y, int64_t n, double r,
                                      const cqk_options* opts, int l1, int64_t* idx_out,
                                      double* val_out, int64_t cap, int64_t* count,
                                      cqk_result* res) {
  if (!h || !y || !idx_out || !val_out || !count || !res || cap < 1)
    return set_err(CQK_E_ARG, "null argument or cap < 1");
  CUDA_TRY(cudaSetDevice(h->device));
  int end_bit = 1;
  while (end_bit < 63 && ((int64_t)1 << end_bit) < n) ++end_bit;
  size_t sort_bytes = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const int64_t*)nullptr, (int64_t*)nullptr,
                                           (const double*)nullptr, (double*)nullptr, (int)cap, 0, end_bit,
                                           h->stream));
  const size_t pb = ((size_t)cap * 8 + 255) / 256 * 256;
  CUDA_TRY(h->sparse_buf.ensure(256 + 4 * pb + sort_bytes));
  char* b = (char*)h->sparse_buf.p;
  auto* cnt = (unsigned long long*)b;
  auto* idx_a = (int64_t*)(b + 256);
  auto* val_a = (double*)(b + 256 + pb);
  auto* idx_b = (int64_t*)(b + 256 + 2 * pb);
  auto* val_b = (double*)(b + 256 + 3 * pb);
  void* tmp = b + 256 + 4 * pb;
  CUDA_TRY(cudaMemsetAsync(cnt, 0, 8, h->stream));
  const cqk_handle::SparseReq req{idx_a, val_a, cnt, cap};
  h->sparse_req = &req;
  int rc = spx_common(h, mem, y, n, n, r, opts, (double*)nullptr, res, l1 != 0, false);
  h->sparse_req = nullptr;
  if (rc != 0) return rc;
  if (res->iterations < 0) return CQK_SPARSE_DENSE;  // l1 inside the ball: x = y
  unsigned long long got = 0;
  CUDA_TRY(cudaMemcpyAsync(&got, cnt, 8, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  *count = (int64_t)got;
  if (got == 0) return CQK_SPARSE_DENSE;  // the kernel took the dense route (r > 0: x != 0)
  if ((int64_t)got > cap) return CQK_SPARSE_OVERFLOW;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, idx_a, idx_b, val_a, val_b, (int)got, 0,
                                           end_bit, h->stream));
  const cudaMemcpyKind k = mem == CQK_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  CUDA_TRY(cudaMemcpyAsync(idx_out, idx_b, sizeof(int64_t) * got, k, h->stream));
  CUDA_TRY(cudaMemcpyAsync(val_out, val_b, sizeof(double) * got, k, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return 0;
}

// ------------------------------------------------------------ batched rows
namespace {
template <int EPT>
cudaError_t launch_rows(cqk_handle* h, const double* Y, double* X, double* lam, int32_t* it,
                        int64_t rows, int cols, double r, double tau, int max_iter, int fixing,
                        double lam0, int start) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spx_rows_kernel<EPT>, kRowThreads, 0);
  int64_t grid = (int64_t)(occ > 0 ? occ : 1) * h->sm_count;
  if (grid > rows) grid = rows;
  spx_rows_kernel<EPT><<<(unsigned)grid, kRowThreads, 0, h->stream>>>(Y, X, lam, it, rows, cols, r,
                                                                       tau, max_iter, fixing, lam0,
                                                                       start);
  return cudaGetLastError();
}
}  // namespace

extern "C" int spx_project_batched_f64(cqk_handle* h, int mem, const double* Y, int64_t rows,
                                       int64_t cols, double r, const cqk_options* opts_in,
                                       double* X, double* lam, int32_t* iters, cqk_result* res) {
  if (!h || !Y || !X || !res) return set_err(CQK_E_ARG, "null argument");
  std::memset(res, 0, sizeof *res);
  res->domain_index = -1;
  cqk_options opts = opts_in ? *opts_in : default_opts();
  CUDA_TRY(cudaSetDevice(h->device));
  if (!(r > 0)) {
    res->status = CQK_E_DOMAIN;
    res->domain_field = CQK_F_R;
    return CQK_E_DOMAIN;
  }
  if (rows < 1 || cols < 1 || cols > 32 * kRowThreads)
    return set_err(CQK_E_ARG, "rows >= 1 and 1 <= cols <= 8192 required");
  const double* Yd = Y;
  double *Xd = X, *Ld = lam;
  int32_t* Id = iters;
  const int64_t tot = rows * cols;
  if (mem == CQK_MEM_HOST) {
    const size_t per = ((size_t)tot * 8 + 255) / 256 * 256;
    const size_t rb = ((size_t)rows * 8 + 255) / 256 * 256;
    CUDA_TRY(h->stage.ensure(2 * per + 2 * rb));
    char* base = (char*)h->stage.p;
    {
      int rc_ = h2d(h, base, Y, (size_t)tot * 8);
      if (rc_) return rc_;
    }
    Yd = (const double*)base;
    Xd = (double*)(base + per);
    Ld = lam ? (double*)(base + 2 * per) : nullptr;
    Id = iters ? (int32_t*)(base + 2 * per + rb) : nullptr;
  }
  const double tau = tau_of(&opts, false);
  const int fixing = opts.variable_fixing != 0;
  const int c = (int)cols;
  CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
  cudaError_t e;
  // aligned rows of even length: one warp per row fed by per-warp bulk-copy
  // rings, rows handed out by a grid counter (cqk_rows.cuh); otherwise the
  // CTA-per-row register kernel
  const bool aligned_rows = (c % 2) == 0 && aligned16(Yd) && aligned16(Xd);
  if (aligned_rows) {
    auto kern = spx_rows_tma_kernel<kRsU, kRsStages, kRsWarps>;
    constexpr size_t sm = rs_tma_warp_bytes<kRsU, kRsStages>() * kRsWarps;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kRsWarps, sm);
    int64_t grid = (int64_t)(occ > 0 ? occ : 1) * h->sm_count;
    const int64_t need = (rows + kRsWarps - 1) / kRsWarps;
    if (grid > need) grid = need;
    // two row counters alternate between launches; each launch zeroes the other
    unsigned* ctr = h->ar_count + 8 + h->rows_flip;
    unsigned* nxt = h->ar_count + 8 + (h->rows_flip ^ 1);
    h->rows_flip ^= 1;
    kern<<<(unsigned)grid, 32 * kRsWarps, sm, h->stream>>>(Yd, Xd, Ld, Id, rows, c, r, tau,
                                                           opts.max_iterations, fixing,
                                                           opts.lambda0, opts.simplex_start, ctr, nxt);
    e = cudaGetLastError();
  } else if (c <= kRowThreads) e = launch_rows<1>(h, Yd, Xd, Ld, Id, rows, c, r, tau, opts.max_iterations, fixing, opts.lambda0, opts.simplex_start);
  else if (c <= 2 * kRowThreads) e = launch_rows<2>(h, Yd, Xd, Ld, Id, rows, c, r, tau, opts.max_iterations, fixing, opts.lambda0, opts.simplex_start);
  else if (c <= 4 * kRowThreads) e = launch_rows<4>(h, Yd, Xd, Ld, Id, rows, c, r, tau, opts.max_iterations, fixing, opts.lambda0, opts.simplex_start);
  else if (c <= 8 * kRowThreads) e = launch_rows<8>(h, Yd, Xd, Ld, Id, rows, c, r, tau, opts.max_iterations, fixing, opts.lambda0, opts.simplex_start);
  else if (c <= 16 * kRowThreads) e = launch_rows<16>(h, Yd, Xd, Ld, Id, rows, c, r, tau, opts.max_iterations, fixing, opts.lambda0, opts.simplex_start);
  else e = launch_rows<32>(h, Yd, Xd, Ld, Id, rows, c, r, tau, opts.max_iterations, fixing, opts.lambda0, opts.simplex_start);
  if (e != cudaSuccess) return set_err(CQK_E_CUDA, std::string("rows kernel: ") + cudaGetErrorString(e));
  CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
  if (mem == CQK_MEM_HOST) {
    {
      int rc_ = d2h(h, X, Xd, (size_t)tot * 8);
      if (rc_) return rc_;
    }
    if (lam) CUDA_TRY(cudaMemcpyAsync(lam, Ld, (size_t)rows * 8, cudaMemcpyDeviceToHost, h->stream));
    if (iters) CUDA_TRY(cudaMemcpyAsync(iters, Id, (size_t)rows * 4, cudaMemcpyDeviceToHost, h->stream));
  }
  int rc = finish_sync(h);
  if (rc) return rc;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  res->status = CQK_SOLVED;
  res->elems_read = tot;
  res->elems_written = tot;
  res->bytes_model = 16 * tot;
  res->device_ms = ms;
  res->launches = 1;
  return 0;
}

// C5 across GPUs ("batched rows: replicas only"): contiguous
// row blocks, one per handle, solved concurrently -- one host thread per
// handle drives its own device, stream, staging ring and kernel; no
// communication.  Each block is an ordinary spx_project_batched_f64 call, so
// a row's result does not depend on the split.
extern "C" int spx_project_batched_multi_f64(cqk_handle* const* hs, int nh, const double* Y,
                                             int64_t rows, int64_t cols, double r,
                                             const cqk_options* opts, double* X, double* lam,
                                             int32_t* iters, cqk_result* res) {
  if (!hs || nh < 1 || !Y || !X || !res) return set_err(CQK_E_ARG, "null argument");
  for (int q = 0; q < nh; ++q)
    if (!hs[q]) return set_err(CQK_E_ARG, "null handle in the device list");
  std::memset(res, 0, sizeof *res);
  res->domain_index = -1;
  if (rows < 1) return set_err(CQK_E_ARG, "rows >= 1 required");
  std::vector<cqk_result> part((size_t)nh);
  std::vector<int> rc((size_t)nh, 0);
  std::vector<std::string> err((size_t)nh);
  std::vector<std::thread> th;
  for (int q = 0; q < nh; ++q) {
    const int64_t lo = rows * q / nh, hi = rows * (q + 1) / nh;
    if (hi == lo) continue;
    th.emplace_back([&, q, lo, hi] {
      rc[q] = spx_project_batched_f64(hs[q], CQK_MEM_HOST, Y + lo * cols, hi - lo, cols, r, opts,
                                      X + lo * cols, lam ? lam + lo : nullptr,
                                      iters ? iters + lo : nullptr, &part[q]);
      if (rc[q] != 0) err[q] = g_err;  // thread_local: carry it to the caller's thread
    });
  }
  for (auto& t : th) t.join();
  for (int q = 0; q < nh; ++q) {
    if (rc[q] != 0) {
      *res = part[q];
      return set_err(rc[q], "device list entry " + std::to_string(q) + ": " + err[q]);
    }
  }
  res->status = CQK_SOLVED;
  for (int q = 0; q < nh; ++q) {
    res->elems_read += part[q].elems_read;
    res->elems_written += part[q].elems_written;
    res->bytes_model += part[q].bytes_model;
    res->device_ms = std::max(res->device_ms, part[q].device_ms);  // concurrent: the slowest
    res->launches += part[q].launches;
  }
  return 0;
}

// ------------------------------------------------------------ device groups
// One process driving several GPUs (the GPU analogue of the reference's
// worker pool, parallel.py:52-59): one handle and one rank per listed device,
// mailboxes wired with cqk_comm_connect_local (peer access enabled), n cut
// into contiguous shards (_chunk_ranges, parallel.py:82-85), one host thread
// per rank calling the sharded entry point, so every rank's persistent kernel
// is in flight at once.  A device listed k times hosts k ranks on 1/k of its
// SMs each (a one-GPU stand-in for k GPUs).
struct cqk_group {
  std::vector<cqk_handle*> h;
  int64_t reserved = -1;  // the largest shard the scratch and staging hold
};

extern "C" int cqk_group_create(cqk_group** out, const int* devices, int ndev) {
  if (!out || !devices || ndev < 1 || ndev > kMaxRanks)
    return set_err(CQK_E_ARG, "need 1..8 devices");
  auto* g = new cqk_group;
  auto fail = [&](int rc) {
    for (auto* x : g->h) cqk_destroy(x);
    delete g;
    return rc;
  };
  for (int q = 0; q < ndev; ++q) {
    cqk_handle* x = nullptr;
    if (int rc = cqk_create(&x, devices[q])) return fail(rc);
    g->h.push_back(x);
  }
  for (int q = 0; q < ndev; ++q) {
    int mult = 0;
    for (int k = 0; k < ndev; ++k) mult += devices[k] == devices[q];
    if (mult > 1) g->h[q]->grid_limit = g->h[q]->sm_count / mult;
    if (int rc = cqk_comm_create(g->h[q], q, ndev, nullptr)) return fail(rc);
  }
  for (int q = 0; q < ndev; ++q)
    if (int rc = cqk_comm_connect_local(g->h[q], g->h.data(), ndev)) return fail(rc);
  *out = g;
  return 0;
}

extern "C" int cqk_group_destroy(cqk_group* g) {
  if (!g) return 0;
  for (auto* x : g->h) cqk_destroy(x);
  delete g;
  return 0;
}

extern "C" int cqk_group_size(const cqk_group* g) { return g ? (int)g->h.size() : 0; }

namespace {

// Allocate every rank's scratch and host staging for shards of up to
// n / W + 1 elements before any kernel starts: an allocation while a peer's
// kernel waits in the exchange could synchronise a shared device.
int group_reserve(cqk_group* g, int64_t n) {
  const int64_t W = (int64_t)g->h.size();
  const int64_t per = n / W + 1;
  if (per <= g->reserved) return 0;
  for (auto* x : g->h) {
    if (int rc = cqk_reserve(x, per)) return rc;
    if (int rc = cqk_reserve_host(x, per)) return rc;
  }
  g->reserved = per;
  return 0;
}

// Run f(q, lo, hi, &res_q) on one thread per rank; combine the outcomes
// (identical on every rank except the per-rank byte counters).
template <class F>
int group_run(cqk_group* g, int64_t n, cqk_result* res, F&& f) {
  const int W = (int)g->h.size();
  std::vector<cqk_result> part((size_t)W);
  std::vector<int> rc((size_t)W, 0);
  std::vector<std::string> err((size_t)W);
  std::vector<std::thread> th;
  for (int q = 0; q < W; ++q) {
    const int64_t lo = n * q / W, hi = n * (q + 1) / W;
    th.emplace_back([&, q, lo, hi] {
      rc[q] = f(q, lo, hi, &part[q]);
      if (rc[q] < 0) err[q] = g_err;  // thread_local: carry it to the caller's thread
    });
  }
  for (auto& t : th) t.join();
  *res = part[0];
  for (int q = 0; q < W; ++q)
    if (rc[q] < 0 && rc[q] != CQK_E_DOMAIN && rc[q] != CQK_E_MAXITER && rc[q] != CQK_E_CONTRACT)
      return set_err(rc[q], "group rank " + std::to_string(q) + ": " + err[q]);
  for (int q = 1; q < W; ++q) {
    const cqk_result& o = part[q];
    if (o.status != res->status || o.iterations != res->iterations ||
        !(o.lam == res->lam || (std::isnan(o.lam) && std::isnan(res->lam))))
      return set_err(CQK_E_CUDA, "group ranks disagree on the outcome (rank " + std::to_string(q) + ")");
    if (o.domain_index >= 0 && (res->domain_index < 0 || o.domain_index < res->domain_index)) {
      res->domain_field = o.domain_field;
      res->domain_index = o.domain_index;
    }
    res->elems_read += o.elems_read;
    res->elems_written += o.elems_written;
    res->bytes_model += o.bytes_model;
    res->device_ms = std::max(res->device_ms, o.device_ms);  // concurrent: the slowest
    res->launches += o.launches;
  }
  return rc[0];
}

}  // namespace

extern "C" int cqk_solve_group_f64(cqk_group* g, const double* d, const double* a,
                                   const double* b, const double* l, const double* u, int64_t n,
                                   double r, const cqk_options* opts, const double* xbar,
                                   double* x, cqk_result* res) {
  if (!g || !d || !a || !b || !l || !u || !res) return set_err(CQK_E_ARG, "null argument");
  const int W = (int)g->h.size();
  if (n < W) return cqk_solve_f64(g->h[0], CQK_MEM_HOST, d, a, b, l, u, n, r, opts, xbar, x, res);
  if (int rc = group_reserve(g, n)) return rc;
  return group_run(g, n, res, [&](int q, int64_t lo, int64_t hi, cqk_result* rq) {
    return cqk_solve_sharded_f64(g->h[q], CQK_MEM_HOST, d + lo, a + lo, b + lo, l + lo, u + lo,
                                 hi - lo, lo, n, r, opts, xbar ? xbar + lo : nullptr,
                                 x ? x + lo : nullptr, rq);
  });
}

static int spx_group(cqk_group* g, const double* y, int64_t n, double r, const cqk_options* opts,
                     double* x, cqk_result* res, bool l1) {
  if (!g || !y || !res) return set_err(CQK_E_ARG, "null argument");
  const int W = (int)g->h.size();
  if (n < W) return spx_common(g->h[0], CQK_MEM_HOST, y, n, n, r, opts, x, res, l1, false);
  if (int rc = group_reserve(g, n)) return rc;
  return group_run(g, n, res, [&](int q, int64_t lo, int64_t hi, cqk_result* rq) {
    return spx_common(g->h[q], CQK_MEM_HOST, y + lo, hi - lo, n, r, opts, x ? x + lo : nullptr, rq,
                      l1, true);
  });
}

extern "C" int spx_project_group_f64(cqk_group* g, const double* y, int64_t n, double r,
                                     const cqk_options* opts, double* x, cqk_result* res) {
  return spx_group(g, y, n, r, opts, x, res, false);
}

extern "C" int l1_project_group_f64(cqk_group* g, const double* y, int64_t n, double r,
                                    const cqk_options* opts, double* x, cqk_result* res) {
  return spx_group(g, y, n, r, opts, x, res, true);
}

// ------------------------------------------------------------ components
extern "C" int cqk_phi_f64(cqk_handle* h, int mem, const double* d, const double* a,
                           const double* b, const double* l, const double* u, int64_t n,
                           const int64_t* idx, int64_t m, double lam, double* out4,
                           uint8_t* at_lower, uint8_t* at_upper) {
  if (!h || !d || !a || !b || !l || !u || !out4) return set_err(CQK_E_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  if (!idx) m = n;
  const double* dv[5];
  {
    const double* in[5] = {d, a, b, l, u};
    int rc = stage_inputs<double>(h, mem, n, in, 5, dv, 0, nullptr);
    if (rc) return rc;
  }
  const int64_t* ix;
  int rc = stage_idx(h, mem, idx, m, &ix);
  if (rc) return rc;
  uint8_t *flo = at_lower, *fhi = at_upper;
  if (mem == CQK_MEM_HOST && (at_lower || at_upper)) {
    CUDA_TRY(h->flags.ensure(2 * (size_t)(m ? m : 1)));
    flo = at_lower ? (uint8_t*)h->flags.p : nullptr;
    fhi = at_upper ? (uint8_t*)h->flags.p + m : nullptr;
  }
  const int nb = util_blocks(h, m);
  phi_util_kernel<double><<<nb, kUtilThreads, 0, h->stream>>>(dv[0], dv[1], dv[2], dv[3], dv[4],
                                                             ix, m, lam, flo, fhi, h->red);
  finalize_kernel<<<1, kUtilThreads, 0, h->stream>>>(h->red, nb, 5, 0, 0, h->out);
  CUDA_TRY(cudaGetLastError());
  double t[kMaxK];
  CUDA_TRY(cudaMemcpyAsync(t, h->out, sizeof(double) * 5, cudaMemcpyDeviceToHost, h->stream));
  if (mem == CQK_MEM_HOST) {
    if (at_lower) CUDA_TRY(cudaMemcpyAsync(at_lower, flo, m, cudaMemcpyDeviceToHost, h->stream));
    if (at_upper) CUDA_TRY(cudaMemcpyAsync(at_upper, fhi, m, cudaMemcpyDeviceToHost, h->stream));
  }
  rc = finish_sync(h);
  if (rc) return rc;
  out4[0] = t[0];
  out4[1] = t[2] + t[4];  // dminus = core + tie_hi
  out4[2] = t[2] + t[3];  // dplus  = core + tie_lo
  out4[3] = t[1];
  return 0;
}

extern "C" int cqk_eval_x_f64(cqk_handle* h, int mem, const double* d, const double* a,
                              const double* b, const double* l, const double* u, int64_t n,
                              const int64_t* idx, int64_t m, double lam, double* x) {
  if (!h || !d || !a || !b || !l || !u || !x) return set_err(CQK_E_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  if (!idx) m = n;
  const double* dv[5];
  double* xd = x;
  {
    const double* in[5] = {d, a, b, l, u};
    int rc = stage_inputs<double>(h, mem, n, in, 5, dv, mem == CQK_MEM_HOST ? 1 : 0, &xd);
    if (rc) return rc;
  }
  const int64_t* ix;
  int rc = stage_idx(h, mem, idx, m, &ix);
  if (rc) return rc;
  evalx_util_kernel<double><<<util_blocks(h, m), kUtilThreads, 0, h->stream>>>(
      dv[0], dv[1], dv[2], dv[3], dv[4], ix, m, lam, xd);
  CUDA_TRY(cudaGetLastError());
  if (mem == CQK_MEM_HOST) CUDA_TRY(cudaMemcpyAsync(x, xd, sizeof(double) * m, cudaMemcpyDeviceToHost, h->stream));
  return finish_sync(h);
}

extern "C" int cqk_nearest_breakpoint_f64(cqk_handle* h, int mem, const double* d,
                                          const double* a, const double* b, const double* l,
                                          const double* u, int64_t n, const int64_t* idx,
                                          int64_t m, double edge, int right, double* bp,
                                          int32_t* found) {
  if (!h || !d || !a || !b || !l || !u || !bp || !found) return set_err(CQK_E_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  if (!idx) m = n;
  const double* dv[5];
  {
    const double* in[5] = {d, a, b, l, u};
    int rc = stage_inputs<double>(h, mem, n, in, 5, dv, 0, nullptr);
    if (rc) return rc;
  }
  const int64_t* ix;
  int rc = stage_idx(h, mem, idx, m, &ix);
  if (rc) return rc;
  const int nb = util_blocks(h, m);
  bp_util_kernel<double><<<nb, kUtilThreads, 0, h->stream>>>(dv[0], dv[1], dv[2], dv[3], dv[4], ix,
                                                            m, edge, right, h->red);
  finalize_kernel<<<1, kUtilThreads, 0, h->stream>>>(h->red, nb, 2, right ? 1 : 0, right ? 0 : 1,
                                                     h->out);
  CUDA_TRY(cudaGetLastError());
  double t[2];
  CUDA_TRY(cudaMemcpyAsync(t, h->out, sizeof t, cudaMemcpyDeviceToHost, h->stream));
  rc = finish_sync(h);
  if (rc) return rc;
  *found = t[1] > 0;
  *bp = t[1] > 0 ? t[0] : NAN;
  return 0;
}

namespace {
int lambda0_util(cqk_handle* h, int mem, const double* d, const double* a, const double* b,
                 const double* l, const double* u, int64_t n, const double* xbar, int check,
                 double* t15) {
  const double* dv[6];
  {
    const double* in[6] = {d, a, b, l, u, xbar};
    int rc = stage_inputs<double>(h, mem, n, in, 6, dv, 0, nullptr);
    if (rc) return rc;
  }
  const int nb = util_blocks(h, n);
  lambda0_util_kernel<double><<<nb, kUtilThreads, 0, h->stream>>>(
      dv[0], dv[1], dv[2], dv[3], dv[4], xbar ? dv[5] : nullptr, n, check, h->red);
  finalize_kernel<<<1, kUtilThreads, 0, h->stream>>>(h->red, nb, 15, 0x7fe0, 0, h->out);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(t15, h->out, sizeof(double) * 15, cudaMemcpyDeviceToHost, h->stream));
  return finish_sync(h);
}
}  // namespace

extern "C" int cqk_initial_multiplier_f64(cqk_handle* h, int mem, const double* d,
                                          const double* a, const double* b, const double* l,
                                          const double* u, int64_t n, double r,
                                          const double* xbar, double* lam0) {
  if (!h || !d || !a || !b || !l || !u || !lam0) return set_err(CQK_E_ARG, "null argument");
  if (n < 1) return set_err(CQK_E_ARG, "n must be >= 1");
  CUDA_TRY(cudaSetDevice(h->device));
  double t[15];
  int rc = lambda0_util(h, mem, d, a, b, l, u, n, xbar, 0, t);
  if (rc) return rc;
  *lam0 = (xbar && t[4] > 0) ? (r - t[2]) / t[3] : (r - t[0]) / t[1];
  return 0;
}

extern "C" int cqk_validate_f64(cqk_handle* h, int mem, const double* d, const double* a,
                                const double* b, const double* l, const double* u, int64_t n,
                                double r, cqk_result* res) {
  if (!h || !res) return set_err(CQK_E_ARG, "null argument");
  std::memset(res, 0, sizeof *res);
  res->domain_index = -1;
  if (n < 1) {
    res->status = CQK_E_DOMAIN;
    res->domain_field = CQK_F_D;
    return CQK_E_DOMAIN;
  }
  if (!d || !a || !b || !l || !u) return set_err(CQK_E_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  double t[15];
  int rc = lambda0_util(h, mem, d, a, b, l, u, n, nullptr, 1, t);
  if (rc) return rc;
  const int32_t field_of[10] = {CQK_F_D, CQK_F_A, CQK_F_B, CQK_F_L, CQK_F_U,
                                CQK_F_D, CQK_F_B, CQK_F_BOUNDS, CQK_F_L, CQK_F_U};
  for (int c = 0; c < 10; ++c) {
    if (c == 5 && !std::isfinite(r)) {
      res->status = CQK_E_DOMAIN;
      res->domain_field = CQK_F_R;
      return CQK_E_DOMAIN;
    }
    if (t[kValidateSlot + c] < (double)n) {
      res->status = CQK_E_DOMAIN;
      res->domain_field = field_of[c];
      res->domain_index = (int64_t)t[kValidateSlot + c];
      return CQK_E_DOMAIN;
    }
  }
  return 0;
}

// ------------------------------------------------------------ self-test
extern "C" int cqk_selftest_division(cqk_handle* h, uint64_t seed, int64_t count, int mode,
                                     uint64_t* mismatches, double* example2) {
  if (!h || !mismatches) return set_err(CQK_E_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  unsigned long long* dm = nullptr;
  double* dex = nullptr;
  CUDA_TRY(cudaMalloc(&dm, sizeof(unsigned long long) + 2 * sizeof(double)));
  dex = (double*)(dm + 1);
  cudaMemsetAsync(dm, 0, sizeof(unsigned long long) + 2 * sizeof(double), h->stream);
  div_selftest_kernel<<<h->sm_count * 8, 256, 0, h->stream>>>(seed, count, mode, dm, dex);
  unsigned long long m = 0;
  double ex[2] = {0, 0};
  cudaMemcpyAsync(&m, dm, sizeof m, cudaMemcpyDeviceToHost, h->stream);
  cudaMemcpyAsync(ex, dex, sizeof ex, cudaMemcpyDeviceToHost, h->stream);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  cudaFree(dm);
  if (e != cudaSuccess) return set_err(CQK_E_CUDA, cudaGetErrorString(e));
  *mismatches = m;
  if (example2) { example2[0] = ex[0]; example2[1] = ex[1]; }
  return 0;
}

// ------------------------------------------------------------ read-only peak
extern "C" int cqk_read_peak_f64(cqk_handle* h, const double* const* arrays, int narr, int64_t n,
                                 int reps, double* gbs_best, double* ms_best) {
  if (!h || !arrays || narr < 1 || narr > kPeakMaxArr || n < kPeakTile || reps < 1 || !gbs_best)
    return set_err(CQK_E_ARG, "read peak: 1..5 device arrays of >= 2048 doubles");
  CUDA_TRY(cudaSetDevice(h->device));
  PeakArgs a;
  std::memset(&a, 0, sizeof a);
  for (int k = 0; k < narr; ++k) {
    if (!arrays[k] || !aligned16(arrays[k])) return set_err(CQK_E_ARG, "read peak: bad array");
    a.arr[k] = arrays[k];
  }
  a.narr = narr;
  a.n = n;
  a.sink = h->out;
  const size_t smem = read_peak_smem();
  CUDA_TRY(cudaFuncSetAttribute(read_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  float best = 1e30f;
  for (int r = 0; r <= reps; ++r) {  // the first launch warms up
    CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    read_peak_kernel<<<h->sm_count, kPeakThreads, smem, h->stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
    CUDA_TRY(cudaEventSynchronize(h->ev1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (r > 0 && ms < best) best = ms;
  }
  const double bytes = (double)narr * (double)(n / kPeakTile * kPeakTile) * 8.0;
  *gbs_best = bytes / (best * 1e-3) / 1e9;
  if (ms_best) *ms_best = best;
  return 0;
}

// ------------------------------------------------------------ Algorithm 2
extern "C" int spx_init_alg2_f64(cqk_handle* h, int mem, const double* y, int64_t n, double r,
                                 const int64_t* idx, int64_t p, int64_t workers,
                                 const double* xbar, int sharpened, double* lam0, int64_t* nfree,
                                 int64_t* free_idx, uint8_t* fixed_mask, double* sum_free,
                                 int64_t* jplus) {
  if (!h || !y || !lam0 || !nfree) return set_err(CQK_E_ARG, "null argument");
  CUDA_TRY(cudaSetDevice(h->device));
  if (!idx) p = n;
  if (p < 1) return set_err(CQK_E_EMPTY, "initializer needs at least one candidate index");
  const double* dv[2];
  {
    const double* in[2] = {y, xbar};
    int rc = stage_inputs<double>(h, mem, n, in, 2, dv, 0, nullptr);
    if (rc) return rc;
  }
  const int64_t* ix;
  int rc = stage_idx(h, mem, idx, p, &ix);
  if (rc) return rc;
  uint8_t* fdev = nullptr;
  if (fixed_mask) {
    if (mem == CQK_MEM_DEVICE) fdev = fixed_mask;
    else {
      CUDA_TRY(h->flags.ensure(n));
      fdev = (uint8_t*)h->flags.p;
    }
    CUDA_TRY(cudaMemsetAsync(fdev, 0, n, h->stream));
  }
  Alg2Out a2;
  rc = run_alg2(h, dv[0], ix, p, r, workers < 1 ? 0 : workers, xbar ? dv[1] : nullptr, sharpened,
                false, false, free_idx != nullptr, fdev, &a2);
  if (rc) return rc;
  *lam0 = a2.lam0;
  *nfree = a2.n_free;
  if (sum_free) *sum_free = a2.sum_free;
  if (free_idx)
    CUDA_TRY(cudaMemcpyAsync(free_idx, h->alg2_idx, sizeof(int64_t) * a2.n_free,
                             mem == CQK_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                             h->stream));
  if (fixed_mask && mem == CQK_MEM_HOST)
    CUDA_TRY(cudaMemcpyAsync(fixed_mask, fdev, n, cudaMemcpyDeviceToHost, h->stream));
  if (jplus) {
    std::vector<int64_t> jp(h->alg2_w);
    CUDA_TRY(cudaMemcpyAsync(jp.data(), h->alg2_jplus, sizeof(int64_t) * h->alg2_w,
                             cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    int64_t t = 0;
    for (int64_t v : jp) t += v;
    *jplus = t;
  }
  return finish_sync(h);
}

// ------------------------------------------------------------ device generators
#include "gen_kernels.cuh"
extern "C" {
#include "xoshiro_jump.h"
}

namespace {
// per-thread states of a stream of `count` tuples of `per_elem` draws from `base`
int upload_states(cqk_handle* h, uint64_t seed, uint64_t base, int64_t per, int64_t per_elem,
                  int64_t T, XoState* dst) {
  std::vector<xo_state> st((size_t)T);
  xo_jump_states(seed, base, (uint64_t)(per * per_elem), T, st.data());
  CUDA_TRY(cudaMemcpyAsync(dst, st.data(), sizeof(XoState) * T, cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));  // st is pageable and dies here
  return 0;
}
}  // namespace

extern "C" int cqk_gen_cqk_device_range(cqk_handle* h, int family, int64_t n, uint64_t seed,
                                        int64_t lo, int64_t hi, double* d, double* a, double* b,
                                        double* l, double* u, double* bl, double* bu) {
  if (!h || !d || !a || !b || !l || !u || n < 1 || family < 0 || family > 2 || lo < 0 ||
      hi > n || lo >= hi)
    return set_err(CQK_E_ARG, "bad generator arguments");
  CUDA_TRY(cudaSetDevice(h->device));
  const int64_t m = hi - lo;
  const int64_t T = m < 16384 ? m : 16384;
  const int64_t per = (m + T - 1) / T;
  const int64_t Tn = (m + per - 1) / per;
  CUDA_TRY(h->idxbuf.ensure(sizeof(XoState) * 2 * Tn));
  XoState* st1 = (XoState*)h->idxbuf.p;
  XoState* st2 = st1 + Tn;
  const int64_t tup = family == 2 ? 1 : 3;
  const uint64_t off = (uint64_t)tup * (uint64_t)n;
  int rc = upload_states(h, seed, (uint64_t)tup * lo, per, tup, Tn, st1);
  if (rc) return rc;
  rc = upload_states(h, seed, off + 2 * (uint64_t)lo, per, 2, Tn, st2);
  if (rc) return rc;
  gen_cqk_kernel<<<(unsigned)((Tn + 255) / 256), 256, 0, h->stream>>>(family, m, per, st1, st2, d,
                                                                      a, b, l, u);
  const int nb = util_blocks(h, m);
  dot_bl_bu_kernel<<<nb, 256, 0, h->stream>>>(b, l, u, m, h->red);
  finalize_kernel<<<1, kUtilThreads, 0, h->stream>>>(h->red, nb, 2, 0, 0, h->out);
  CUDA_TRY(cudaGetLastError());
  double t[2];
  CUDA_TRY(cudaMemcpyAsync(t, h->out, sizeof t, cudaMemcpyDeviceToHost, h->stream));
  rc = finish_sync(h);
  if (rc) return rc;
  if (bl) *bl = t[0];
  if (bu) *bu = t[1];
  return 0;
}

static double gen_cqk_r(int family, int64_t n, uint64_t seed, double bl, double bu) {
  const uint64_t off = (uint64_t)(family == 2 ? 1 : 3) * (uint64_t)n;
  xo_state s = xo_jump(xo_seed(seed), off + 2 * (uint64_t)n);  // instances.py:66
  const double ur = (double)(xo_next(&s) >> 11) * 0x1p-53;
  return bl + ur * (bu - bl);
}

extern "C" int cqk_gen_cqk_device(cqk_handle* h, int family, int64_t n, uint64_t seed, double* d,
                                  double* a, double* b, double* l, double* u, double* r_out) {
  if (!r_out) return set_err(CQK_E_ARG, "null r");
  double bl, bu;
  int rc = cqk_gen_cqk_device_range(h, family, n, seed, 0, n, d, a, b, l, u, &bl, &bu);
  if (rc) return rc;
  *r_out = gen_cqk_r(family, n, seed, bl, bu);
  return 0;
}

extern "C" int cqk_gen_simplex_u01_device(cqk_handle* h, int64_t n, uint64_t seed, double* y) {
  if (!h || !y || n < 1) return set_err(CQK_E_ARG, "bad generator arguments");
  CUDA_TRY(cudaSetDevice(h->device));
  const int64_t T = n < 16384 ? n : 16384;
  const int64_t per = (n + T - 1) / T;
  const int64_t Tn = (n + per - 1) / per;
  CUDA_TRY(h->idxbuf.ensure(sizeof(XoState) * Tn + 64));
  XoState* st = (XoState*)h->idxbuf.p;
  unsigned long long* zeros = (unsigned long long*)(st + Tn);
  for (uint64_t attempt = 0;; ++attempt) {  // instances.py:78-86: redraw while any zero
    int rc = upload_states(h, seed, attempt * (uint64_t)n, per, 1, Tn, st);
    if (rc) return rc;
    CUDA_TRY(cudaMemsetAsync(zeros, 0, 8, h->stream));
    gen_u01_kernel<<<(unsigned)((Tn + 255) / 256), 256, 0, h->stream>>>(n, per, st, y, zeros);
    CUDA_TRY(cudaGetLastError());
    unsigned long long z = 0;
    CUDA_TRY(cudaMemcpyAsync(&z, zeros, 8, cudaMemcpyDeviceToHost, h->stream));
    rc = finish_sync(h);
    if (rc) return rc;
    if (!z) return 0;
  }
}

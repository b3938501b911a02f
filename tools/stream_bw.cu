// Read-only HBM streaming ceiling on B200 (perf-iteration aid, not product).
// Streams NARR fp64 arrays of n elements and reduces them; reports GB/s for
// several launch shapes so the scan passes have a realistic denominator.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw stream_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int NARR, int UNR>
__global__ void rd(const double* const* arr, long long n, double* out) {
  double acc = 0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n2 = n / 2;
  for (long long i = tid; i < n2; i += stride * UNR) {
    double2 v[NARR][UNR];
#pragma unroll
    for (int k = 0; k < NARR; ++k)
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        long long j = i + u * stride;
        v[k][u] = j < n2 ? __ldcs(reinterpret_cast<const double2*>(arr[k]) + j) : make_double2(0, 0);
      }
#pragma unroll
    for (int k = 0; k < NARR; ++k)
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc += v[k][u].x + v[k][u].y;
  }
  if (acc == 1.2345) out[0] = acc;
}

// warp-segment streaming (like the solver): warp w owns [w*n/W, (w+1)*n/W)
template <int NARR, int UNR>
__global__ void seg(const double* const* arr, long long n, double* out) {
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  long long lo = n * gw / W / 64 * 64, hi = n * (gw + 1) / W / 64 * 64;
  if (gw == W - 1) hi = n;
  double acc = 0;
  constexpr int CH = 64 * UNR;
  for (long long b = lo; b + CH <= hi; b += CH) {
    double2 v[NARR][UNR];
#pragma unroll
    for (int k = 0; k < NARR; ++k)
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        v[k][u] = __ldcs(reinterpret_cast<const double2*>(arr[k] + b + u * 64) + lane);
#pragma unroll
    for (int k = 0; k < NARR; ++k)
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc += v[k][u].x + v[k][u].y;
  }
  if (acc == 1.2345) out[0] = acc;
}


// warp-chunk-strided (warp w owns chunks w, w+W, ...): grid-wide contiguous window
template <int NARR, int UNR>
__global__ void wstride(const double* const* arr, long long n, double* out) {
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  constexpr int CH = 64 * UNR;
  double acc = 0;
  for (long long b = gw * CH; b + CH <= n; b += W * CH) {
    double2 v[NARR][UNR];
#pragma unroll
    for (int k = 0; k < NARR; ++k)
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        v[k][u] = __ldcs(reinterpret_cast<const double2*>(arr[k] + b + u * 64) + lane);
#pragma unroll
    for (int k = 0; k < NARR; ++k)
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc += v[k][u].x + v[k][u].y;
  }
  if (acc == 1.2345) out[0] = acc;
}

// TMA bulk pipeline: CTA c owns tiles c, c+G, ...; one producer thread keeps
// STAGES tiles (NARR arrays x TILE doubles) in flight into shared memory.
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int NARR, int TILE, int STAGES>
__global__ void tmapipe(const double* const* arr, long long n, double* out) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* buf = reinterpret_cast<double*>(smraw);
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  const int nw = blockDim.x / 32 - 1;  // consumer warps
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(nw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ntiles = n / TILE;
  double acc = 0;
  if (warp == nw) {
    if (lane == 0) {
      int j = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const int s = j % STAGES;
        if (j >= STAGES) {
          const unsigned ph = ((j / STAGES) - 1) & 1;
          asm volatile("{\n.reg .pred p;\nW1_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W1_%=;\n}" ::"r"(su32(&empty[s])), "r"(ph) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(NARR * TILE * 8) : "memory");
        for (int k = 0; k < NARR; ++k)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(buf + ((size_t)s * NARR + k) * TILE)), "l"(arr[k] + t * TILE), "r"(TILE * 8), "r"(su32(&full[s])) : "memory");
      }
    }
  } else {
    int j = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const int s = j % STAGES;
      const unsigned ph = (j / STAGES) & 1;
      asm volatile("{\n.reg .pred p;\nW2_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2_%=;\n}" ::"r"(su32(&full[s])), "r"(ph) : "memory");
      for (int k = 0; k < NARR; ++k) {
        const double2* q = reinterpret_cast<const double2*>(buf + ((size_t)s * NARR + k) * TILE);
        for (int i = warp * 32 + lane; i < TILE / 2; i += nw * 32) { double2 v = q[i]; acc += v.x + v.y; }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
  }
  if (acc == 1.2345) out[0] = acc;
}

static size_t g_smem = 0;
template <typename K>
float timeit(K k, int grid, int block, const double* const* arr, long long n, double* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<grid, block, g_smem>>>(arr, n, out);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<<<grid, block, g_smem>>>(arr, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  long long n = argc > 1 ? atoll(argv[1]) : 100000000LL;
  double* bufs[5];
  for (int k = 0; k < 5; ++k) {
    cudaMalloc(&bufs[k], n * 8);
    cudaMemset(bufs[k], 0, n * 8);
  }
  double** darr;
  cudaMalloc(&darr, sizeof bufs);
  cudaMemcpy(darr, bufs, sizeof bufs, cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double GB1 = n * 8.0 / 1e9;
#define RUN(NAME, KER, NARR, GRID, BLOCK)                                                   \
  {                                                                                         \
    float ms = timeit(KER, GRID, BLOCK, darr, n, out);                                      \
    printf("%-28s grid %5d block %4d : %7.1f GB/s (%.3f ms)\n", NAME, GRID, BLOCK,          \
           NARR * GB1 / ms * 1e3, ms);                                                      \
  }
  RUN("gridstride 1arr unr4", (rd<1, 4>), 1, sms * 4, 512);
  RUN("gridstride 1arr unr8", (rd<1, 8>), 1, sms * 4, 512);
  RUN("gridstride 5arr unr2", (rd<5, 2>), 5, sms * 4, 512);
  RUN("gridstride 5arr unr2 1cta", (rd<5, 2>), 5, sms, 512);
  RUN("gridstride 5arr unr1 2k", (rd<5, 1>), 5, sms, 1024);
  RUN("gridstride 3arr unr2", (rd<3, 2>), 3, sms * 4, 512);
  RUN("segment 5arr unr2 512", (seg<5, 2>), 5, sms, 512);
  RUN("segment 5arr unr2 1024", (seg<5, 2>), 5, sms, 1024);
  RUN("segment 5arr unr2 2x1024", (seg<5, 2>), 5, sms * 2, 1024);
  RUN("segment 5arr unr4 512", (seg<5, 4>), 5, sms, 512);
  RUN("segment 1arr unr8 512", (seg<1, 8>), 1, sms, 512);
  RUN("segment 1arr unr8 2x1024", (seg<1, 8>), 1, sms * 2, 1024);
  RUN("wstride 5arr unr2 512", (wstride<5, 2>), 5, sms, 512);
  RUN("wstride 5arr unr2 1024", (wstride<5, 2>), 5, sms, 1024);
  RUN("wstride 1arr unr8 512", (wstride<1, 8>), 1, sms, 512);
#define TP(NARR, TILE, ST, THR)                                                              \
  {                                                                                        \
    g_smem = (size_t)NARR * TILE * ST * 8;                                                 \
    cudaFuncSetAttribute(tmapipe<NARR, TILE, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g_smem); \
    RUN("tma " #NARR "arr tile" #TILE " st" #ST " thr" #THR, (tmapipe<NARR, TILE, ST>), NARR, sms, THR); \
    g_smem = 0;                                                                            \
  }
  TP(5, 1024, 4, 288);
  TP(5, 512, 8, 288);
  TP(5, 1024, 5, 544);
  TP(5, 2048, 2, 544);
  TP(5, 512, 10, 544);
  TP(1, 4096, 6, 288);
  TP(1, 2048, 12, 288);
  TP(1, 8192, 3, 288);
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}

// Write-only stream bandwidth on one GPU (the simplex / l1 sparse final is a
// zero fill): per-thread 16-byte streaming stores vs 32-byte stores vs bulk
// shared->global copies from a zeroed buffer.  Perf-iteration aid, not
// product code.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_bw write_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void st16(double* x, int64_t n, int cs) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
    if (cs) __stcs(reinterpret_cast<double2*>(x + i), make_double2(0.0, 0.0));
    else *reinterpret_cast<double2*>(x + i) = make_double2(0.0, 0.0);
  }
}

__global__ void st32(double* x, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(x + i), "d"(0.0) : "memory");
  }
}

// one elected thread per CTA issues bulk stores of CH bytes from a zeroed
// shared buffer; CTA c owns chunks c, c + G, ...
template <int CH>
__global__ void bulk(double* x, int64_t n) {
  extern __shared__ __align__(128) double z[];
  for (int i = threadIdx.x; i < CH / 8; i += blockDim.x) z[i] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int64_t per = CH / 8;
  const unsigned src = (unsigned)__cvta_generic_to_shared(z);
  int inflight = 0;
  for (int64_t c = blockIdx.x; c * per < n; c += gridDim.x) {
    const int64_t left = n - c * per;
    const unsigned bytes = (unsigned)((left < per ? left : per) * 8);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(x + c * per), "r"(src),
                 "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++inflight >= 8) asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the sparse final's pattern (cqk_tma_spx.cuh spx_sparse_final): tiles of
// 3840 doubles, warp w (of NW writers) owns a 256-double sub-segment, lane l
// writes elements 64u + 2l, +1; CTA c takes tiles t0 + kG, k < GRP, t0 = c, c + GRP G, ...
template <int GRP, int NW>
__global__ void tiled(double* x, int64_t n) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= NW) return;
  const int64_t G = gridDim.x, ntiles = (n + 3839) / 3840;
  constexpr int SEG = 3840 / NW;
  for (int64_t t0 = blockIdx.x; t0 < ntiles; t0 += GRP * G) {
#pragma unroll
    for (int k = 0; k < GRP; ++k) {
      const int64_t t = t0 + k * G;
      if (t >= ntiles) continue;
      const int64_t gbase = t * 3840 + (int64_t)SEG * warp;
      const int64_t left = n - gbase;
      const int wcnt = left <= 0 ? 0 : (left < SEG ? (int)left : SEG);
#pragma unroll
      for (int u = 0; u < SEG / 64; ++u) {
        const int e = 64 * u + 2 * lane;
        if (e + 1 < wcnt) __stcs(reinterpret_cast<double2*>(x + gbase + e), make_double2(0.0, -0.0));
      }
    }
  }
}

__global__ void rd(const double* y, int64_t n, double* sink) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
    const double2 v = __ldcs(reinterpret_cast<const double2*>(y + i));
    acc += v.x + v.y;
  }
  if (acc == 12345.678) *sink = acc;
}

int main(int argc, char** argv) {
  const bool cold = argc > 1;  // read a second n-element buffer before every timed write
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int64_t n : {(int64_t)100000000, (int64_t)1000000000}) {
    double *x, *y = nullptr;
    cudaMalloc(&x, n * 8);
    if (cold) { cudaMalloc(&y, n * 8); cudaMemset(y, 0, n * 8); }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
      float best = 1e30f;
      for (int r = 0; r < 6; ++r) {
        if (cold) rd<<<sms * 2, 512>>>(y, n, x);
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
      }
      printf("{\"n\": %lld, \"cold\": %d, \"variant\": \"%s\", \"ms\": %.4f, \"GBps\": %.0f, \"err\": \"%s\"}\n", (long long)n, (int)cold, name,
             best, n * 8.0 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int b : {1, 2, 4})
      for (int t : {512, 1024}) {
        char nm[64];
        snprintf(nm, sizeof nm, "st16_cs g=%dx%d", b, t);
        run(nm, [&] { st16<<<sms * b, t>>>(x, n, 1); });
        snprintf(nm, sizeof nm, "st16 g=%dx%d", b, t);
        run(nm, [&] { st16<<<sms * b, t>>>(x, n, 0); });
        snprintf(nm, sizeof nm, "st32_cs g=%dx%d", b, t);
        run(nm, [&] { st32<<<sms * b, t>>>(x, n); });
      }
    run("tiled grp4 nw15", [&] { tiled<4, 15><<<sms, 512>>>(x, n); });
    run("tiled grp1 nw15", [&] { tiled<1, 15><<<sms, 512>>>(x, n); });
    run("tiled grp8 nw15", [&] { tiled<8, 15><<<sms, 512>>>(x, n); });
    run("tiled grp4 nw16", [&] { tiled<4, 16><<<sms, 512>>>(x, n); });
    run("tiled grp4 nw15 2cta", [&] { tiled<4, 15><<<sms * 2, 512>>>(x, n); });
    cudaFuncSetAttribute(bulk<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaFuncSetAttribute(bulk<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    cudaFuncSetAttribute(bulk<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int b : {1, 2, 4}) {
      char nm[64];
      snprintf(nm, sizeof nm, "bulk16K g=%dx", b);
      run(nm, [&] { bulk<16384><<<sms * b, 128, 16384>>>(x, n); });
      snprintf(nm, sizeof nm, "bulk32K g=%dx", b);
      run(nm, [&] { bulk<32768><<<sms * b, 128, 32768>>>(x, n); });
      snprintf(nm, sizeof nm, "bulk64K g=%dx", b);
      run(nm, [&] { bulk<65536><<<sms * b, 128, 65536>>>(x, n); });
    }
    cudaFree(x);
    if (y) cudaFree(y);
  }
  return 0;
}

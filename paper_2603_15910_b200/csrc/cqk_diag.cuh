// cqk_diag.cuh -- measurement aids exported through the C-ABI.
//
// read_peak_kernel: the read-only HBM streaming ceiling for the roofline's
// second denominator (the phi passes are ~100% reads, the
// driver's copy peak is 50/50).  Same engine shape as the solver's passes --
// one producer lane per CTA keeping STAGES tiles of every array in flight with
// cp.async.bulk into shared memory, the other warps consuming -- but with no
// arithmetic beyond a sum, so it bounds what any streaming pass can reach.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cqk {

constexpr int kPeakTile = 2048;   // doubles per array per tile (16 KB)
constexpr int kPeakStages = 10;   // stages of one array; narr arrays use 10 / narr stages:
                                  // 160 KB in flight per SM whatever the array count
constexpr int kPeakThreads = 544; // 16 consumer warps + the producer warp
constexpr int kPeakMaxArr = 5;

struct PeakArgs {
  const double* arr[kPeakMaxArr];
  int narr;
  long long n;
  double* sink;
};

__device__ __forceinline__ unsigned peak_su32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(kPeakThreads, 1) read_peak_kernel(PeakArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double* buf = reinterpret_cast<double*>(smraw);
  __shared__ __align__(8) unsigned long long full[kPeakStages], empty[kPeakStages];
  const int nw = blockDim.x / 32 - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPeakStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(peak_su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(peak_su32(&empty[s])), "r"(nw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ntiles = a.n / kPeakTile;
  const int S = kPeakStages / a.narr;  // stages in flight (each holds narr tiles)
  double acc = 0;
  if (warp == nw) {
    if (lane == 0) {
      int j = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const int s = j % S;
        if (j >= S) {
          const unsigned ph = ((j / S) - 1) & 1;
          asm volatile(
              "{\n.reg .pred p;\nPW1_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
              "@!p bra PW1_%=;\n}" ::"r"(peak_su32(&empty[s])), "r"(ph) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(peak_su32(&full[s])),
                     "r"(a.narr * kPeakTile * 8) : "memory");
        for (int k = 0; k < a.narr; ++k)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  peak_su32(buf + ((size_t)s * a.narr + k) * kPeakTile)),
              "l"(a.arr[k] + t * kPeakTile), "r"(kPeakTile * 8), "r"(peak_su32(&full[s]))
              : "memory");
      }
    }
  } else {
    int j = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const int s = j % S;
      const unsigned ph = (j / S) & 1;
      asm volatile(
          "{\n.reg .pred p;\nPW2_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra PW2_%=;\n}" ::"r"(peak_su32(&full[s])), "r"(ph) : "memory");
      for (int k = 0; k < a.narr; ++k) {
        const double2* q = reinterpret_cast<const double2*>(buf + ((size_t)s * a.narr + k) * kPeakTile);
        for (int i = warp * 32 + lane; i < kPeakTile / 2; i += nw * 32) {
          const double2 v = q[i];
          acc += v.x + v.y;
        }
      }
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(peak_su32(&empty[s])) : "memory");
    }
  }
  if (acc == 1.2345) a.sink[0] = acc;  // keeps the loads live
}

inline size_t read_peak_smem() { return (size_t)kPeakTile * kPeakStages * sizeof(double); }

}  // namespace cqk

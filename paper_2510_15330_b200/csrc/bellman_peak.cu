// bellman_peak.cu — integer issue / lane-throughput microbenchmark for the
// roofline of the tick kernel (R_issue and R_lane, "L_int =
// INT32 lanes/clk/SM, measure with a microbenchmark").  Measurement only: it
// shares nothing with the simulator and computes nothing of the method.
//
// Each warp runs 8 independent dependency chains of 32-bit integer ops whose
// pipe is fixed by the opcode (B200 guide: IADD3/LOP3/SHF on the alu pipe,
// IMAD on the fma pipe, both latency 4 and one warp-instruction per 2 clk per
// SM sub-partition).  Every SM holds 32 warps, so dependencies are hidden and
// the pipes (or the 1 warp-instruction/clk issue port) bind.  Cycles come from
// %clock64 per warp: per SM, (max end - min start) over its warps.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bellman_peak.h"

namespace {

constexpr int kIters = 1024;
constexpr int kUnroll = 16;  // 8 chains x 16 = 128 ops per loop trip (+3 loop instructions)
constexpr int kWarpsPerSm = 32;

__device__ __forceinline__ void alu_add(uint32_t &x, uint32_t k) { asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(k)); }
__device__ __forceinline__ void alu_xor(uint32_t &x, uint32_t k) { asm volatile("xor.b32 %0, %0, %1;" : "+r"(x) : "r"(k)); }
__device__ __forceinline__ void alu_mad(uint32_t &x, uint32_t k) {
  asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(x) : "r"(k));
}

// MODE 0: alu pipe only (add / xor);  1: fma pipe only (mad.lo);  2: both, alternating
template <int MODE>
__global__ void __launch_bounds__(256) peak_kernel(uint32_t seed, uint32_t *sink, unsigned long long *cyc) {
  uint32_t a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = (seed + threadIdx.x) * (2u * c + 1u) ^ (0x9E3779B9u * c);
  const uint32_t k = seed | 1u;
  __syncthreads();
  const unsigned long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        // alu chains alternate add / xor per step: ptxas cannot fuse an add
        // into a LOP3 or a xor into an IADD3, so every op stays one instruction
        const bool fma = MODE == 1 || (MODE == 2 && (c & 1));
        if (fma) alu_mad(a[c], k);
        else if (u & 1) alu_xor(a[c], k);
        else alu_add(a[c], k);
      }
    }
  }
  const unsigned long long t1 = clock64();
  const uint32_t x = a[0] ^ a[1] ^ a[2] ^ a[3] ^ a[4] ^ a[5] ^ a[6] ^ a[7];
  if (x == 0x12345678u) sink[0] = x;  // keeps the chains live
  if ((threadIdx.x & 31u) == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    atomicMin(&cyc[3 * smid], t0);
    atomicMax(&cyc[3 * smid + 1], t1);
    atomicAdd(&cyc[3 * smid + 2], 1ull);  // warps run on this SM
  }
}

template <int MODE>
int run_mode(int nsm, double *inst_per_clk, double *lanes_per_clk) {
  constexpr int kMaxSm = 1024;
  uint32_t *sink = nullptr;
  unsigned long long *cyc = nullptr;
  static unsigned long long init[3 * kMaxSm], out[3 * kMaxSm];
  if (nsm > kMaxSm) return 1;
  if (cudaMalloc(&sink, 4) != cudaSuccess) return 1;
  if (cudaMalloc(&cyc, sizeof(init)) != cudaSuccess) return 1;
  for (int i = 0; i < kMaxSm; ++i) {
    init[3 * i] = ~0ull;
    init[3 * i + 1] = 0ull;
    init[3 * i + 2] = 0ull;
  }
  const int threads = 256, blocks = nsm * kWarpsPerSm * 32 / threads;
  double best = 0.0;
  int rc = 0;
  for (int rep = 0; rep < 3 && !rc; ++rep) {
    cudaMemcpy(cyc, init, sizeof(init), cudaMemcpyHostToDevice);
    peak_kernel<MODE><<<blocks, threads>>>(0x2545F491u + rep, sink, cyc);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      rc = 2;
      break;
    }
    cudaMemcpy(out, cyc, sizeof(out), cudaMemcpyDeviceToHost);
    // per SM: warp-instructions it issued / its cycles; the minimum over SMs
    // (a throughput every SM sustained)
    double lo = 0.0;
    int used = 0;
    for (int s = 0; s < kMaxSm; ++s)
      if (out[3 * s + 2] > 0 && out[3 * s + 1] > out[3 * s]) {
        const double inst = (double)out[3 * s + 2] * kIters * kUnroll * 8;  // ops (loop overhead excluded)
        const double r = inst / (double)(out[3 * s + 1] - out[3 * s]);
        lo = used++ ? (r < lo ? r : lo) : r;
      }
    if (used == 0) rc = 3;
    else if (lo > best) best = lo;
  }
  cudaFree(sink);
  cudaFree(cyc);
  *inst_per_clk = best;
  *lanes_per_clk = best * 32.0;
  return rc;
}

}  // namespace

extern "C" int bellman_peak_int(int device, double out[6]) {
  if (!out) return 1;
  if (cudaSetDevice(device) != cudaSuccess) return 4;
  int nsm = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || nsm <= 0) return 4;
  int rc = run_mode<0>(nsm, &out[0], &out[1]);
  if (!rc) rc = run_mode<1>(nsm, &out[2], &out[3]);
  if (!rc) rc = run_mode<2>(nsm, &out[4], &out[5]);
  return rc;
}

/* bellman_peak.h — integer-throughput microbenchmark behind the tick kernel's
 * roofline (R_issue = 148 x issue/clk x f / A_tick and
 * R_lane = 148 x L_int x f / A_tick, "L_int = INT32 lanes/clk/SM, measure with
 * a microbenchmark").  Measurement only: not part of the simulator's path.
 *
 * int bellman_peak_int(int device, double out[6])
 *   Runs three kernels on `device` (32 resident warps per SM, 8 independent
 *   32-bit chains per thread, 2^17 ops per thread in 128-op loop trips) and writes, per SM and per
 *   SM clock cycle (%clock64; the minimum over SMs of the best of 3 runs):
 *     out[0], out[1]  alu pipe only (add.u32 / xor.b32 -> IADD3 / LOP3):
 *                     warp-instructions/clk, integer lanes/clk (= 32 x out[0])
 *     out[2], out[3]  fma pipe only (mad.lo.u32 -> IMAD)
 *     out[4], out[5]  both pipes, alternating (the issue-port bound)
 *   `out` is caller-owned host memory.  Synchronous (device-wide sync).
 *   Returns 0 on success; 1 bad argument / allocation failure, 2 kernel
 *   failure, 3 no SM reported, 4 bad device.
 */
#ifndef BELLMAN_PEAK_H
#define BELLMAN_PEAK_H
#ifdef __cplusplus
extern "C" {
#endif

int bellman_peak_int(int device, double out[6]);

#ifdef __cplusplus
}
#endif
#endif

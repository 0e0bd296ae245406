// Product-internal device layout of the beLLMan simulator (not part of the ABI).
// DESIGN.md section 4 documents the HBM layout; section 2 names steps a1..a10.
#pragma once
#include <cstdint>

#include "../../include/bellman_sim.h"
#include "bellman_lane.cuh"

namespace bellman {

constexpr uint32_t kSeedHi = 0xB311A000u;  // Philox key word 1 (reading R32)
constexpr uint64_t kUs = 1000000ull;
// Two warps (two scenarios) per CTA, 8 CTAs per SM: measured faster than one
// warp per CTA (whose per-warp shared-memory addresses are compile-time
// constants) on the bench launches — C5 subset -0.95 %, C2 -2.4 %, A/B in one
// process; 4 warps per CTA exceed the 48 KB static shared memory.
#ifndef BELLMAN_WPB
#define BELLMAN_WPB 2
#endif
constexpr uint32_t kWarpsPerBlock = BELLMAN_WPB;
constexpr uint32_t kSegWords = BELLMAN_SEG_HIST_WORDS;

// One non-empty thinning segment of a trace, precomputed on the host (a2):
// [ta, tb) with endpoint rates la, lb, lmax = max(la, lb) > 0 and the
// exponential scale M = floor(2^32 * 1e9 / lmax) (µs per unit rate, Q32).
struct DevSeg {
  uint64_t ta, tb, span, M;
  uint32_t la, lb, lmax, _pad;
};
static_assert(sizeof(DevSeg) == 48, "DevSeg layout");

struct DevTrace {
  uint32_t seg_off, n_seg, cap, kind;  // kind 1 (replay): seg_off/n_seg index Params::arrivals
};

// Per-warp shared-memory histograms (a9, NEXT-2): 10,848 bytes.
struct alignas(16) WarpHist {
  uint32_t e2e[BELLMAN_HIST_LAT];
  uint32_t ttft[BELLMAN_HIST_LAT];
  uint32_t r[BELLMAN_HIST_R];
  uint32_t qa[204];  // similarity, active (BELLMAN_HIST_Q bins used)
  uint32_t qi[204];  // similarity, inactive
};
static_assert(sizeof(WarpHist) % 16 == 0, "WarpHist is zeroed with 16-byte stores");

// NEXT-4 preemption scratch of one CTA (one warp, one scenario at a time), in
// global memory: it is touched only by preempting profiles, at admissions,
// prefill ends, joins and preemptions.  Slot s = lane + 32 k.
struct PreEnt {   // a preempted request waiting at the queue front
  uint64_t a;     // arrival (absolute µs)
  uint64_t lt;    // its last word (absolute µs)
  uint64_t enq;   // start of this queue stay
  uint32_t in, R, em, _pad;  // input words, realized length, words emitted
};
struct PreScratch {
  uint64_t lt[64];   // last word of a re-admitted request (absolute µs)
  uint32_t seq[64];  // admission order
  uint32_t em[64];   // words emitted before the current phase (prefill: before it; ready: so far)
  PreEnt stk[64];    // preempted requests, top = stk[n - 1] (the queue front)
};
constexpr uint32_t kMaxPreCtas = 4096;  // CTAs of one launch (B200: 148 x 16)

struct Params {
  const bellman_scenario *sc;
  const DevTrace *traces;
  const DevSeg *segs;
  const bellman_profile *profs;
  const bellman_ctrl *ctrls;
  const int32_t *tabL, *tabI, *tabF, *tabN, *tabC, *tabQ;  // 4096 each
  const uint2 *log2tab;                             // (T[i], T[i+1]-T[i]), i < 4096
  int64_t poly0, poly1, poly2;
  uint32_t poly_fast;  // |poly(N) * Fcomp| < 2^63 for every N < 2^17: the rewrite fits int64
  uint32_t q_inactive, q_active, q_floor, q_safe, q_end;  // quality model (NEXT-2)
  uint32_t class_cum0, class_cum1, class_cum2;            // request classes (NEXT-3)
  const uint32_t *series_slot;  // [n_scenarios] slot or NONE
  const uint64_t *series_off;   // [n_slots] word offset into series
  const uint32_t *series_cap;   // [n_slots]
  uint32_t *series_n;           // [n_slots] samples written
  uint32_t *series;             // sample storage
  uint32_t *calib;              // [n_slots][4]: t1, t2, status, n
  const uint32_t *dbg_slot;     // [n_scenarios] debug-record slot or NONE (NEXT-1)
  const uint64_t *dbg_off;      // [n_dbg] row offset
  const uint32_t *dbg_cap;      // [n_dbg] rows (= controller-log rows) capacity
  uint32_t *dbg_n;              // [n_dbg][2]: rows, controller-log rows written
  bellman_second_row *dbg_rows;
  bellman_ctrl_row *dbg_ctrl;
  const bellman_arrival *arrivals;  // replay lists (NEXT-4)
  bellman_scenario_stats *stats;
  bellman_scenario_stats *peer[BELLMAN_MAX_PEERS];  // fused exchange: every rank's record array
  uint32_t n_peer;                                  // 0: off
  unsigned long long *seg_hist;  // [n_segments][kSegWords]
  unsigned int *counter;         // work counter of this launch
  const uint32_t *order;         // heavy-first scenario order of a whole-set run, else NULL
  PreScratch *pre;               // [kMaxPreCtas] NEXT-4 preemption scratch (preempting profiles only)
  uint64_t first, count, stride;
  uint32_t pass;  // 1: non-calibrated scenarios, 2: calibrated scenarios
  uint32_t lane_on;    // 1: kind-0 scenarios within K2L's bounds run in K2L (scenario_kind_of)
  uint32_t *lane_hist; // K2L per-thread histograms [kLaneMaxThreads][kLaneHistWords], all-zero between scenarios
  uint2 *lane_fifo;    // K2L per-thread arrival FIFOs [kLaneMaxThreads][32 entries x 3 uint2]
  const uint64_t *cost_magic;  // K2L: [n_profiles][65] ceil(2^63 / cost(B)) of the kv-free cost law (0: unused)
};

// K2L's leap divides by the kv-free iteration cost c(B) = t0 + slope max(0, B - knee)
// through a per-profile reciprocal table (cost_magic_build): floor(n / c) =
// floor(M n / 2^63) with M = ceil(2^63 / c), exact for n < 2^32 and 1 <= c < 2^31
// (M c - 2^63 = e < c, so e n < 2^63 keeps the error below one quotient step).
constexpr uint32_t kCostMagicB = 65;  // B = 0 .. 64

}  // namespace bellman

// launchers (bellman_kernels.cu, bellman_lane.cu)
// one persistent launch over the run's scenarios of one kernel: dbg (debug-recorded
// or not) x kind (0 TBT-specialised, 1 generic, 2 multi-replica; scenario_kind)
cudaError_t bellman_launch_tick(const bellman::Params &p, int grid, bool dbg, int kind, cudaStream_t stream);
// K2L (kind 3: kv = 0, kind 4: kv > 0), one CTA per SM
cudaError_t bellman_launch_lane(const bellman::Params &p, int grid, int kind, cudaStream_t stream);
int bellman_lane_grid(int device);
cudaError_t bellman_launch_calibrate(const bellman::Params &p, uint32_t n_slots, cudaStream_t stream);
int bellman_tick_grid(int device);

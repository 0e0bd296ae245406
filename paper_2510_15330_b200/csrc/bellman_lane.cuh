// Which engine runs a scenario, and the layout constants of K2L (the
// lane-per-scenario kernel, bellman_lane.cu).  Product-internal.
#pragma once
#include <cstdint>

#include "../../include/bellman_sim.h"

namespace bellman {

// K2L per-warp shared memory: slot fields [field][64 slots][32 lanes] (u32),
// then the decode heap (64 one-byte slot indices per lane, [16][32] words).
// Fields: prefill end (then the completion iteration), arrival, R (+ input
// words with a KV term).
template <bool KV0>
constexpr uint32_t kFields = KV0 ? 3u : 4u;
#ifdef BELLMAN_AB_NOSENT
template <bool KV0>
constexpr uint32_t kLaneWarpWords = (kFields<KV0> * 64u + 17u) * 32u;  // A/B only: no sentinel (heap: 67 bytes)
#else
// + one sentinel word per lane after the last field (the key kInf of the
// sentinel slot index 64 that fills every heap position >= the heap's size);
// the heap spans 22 words: positions 0 .. 84, the children of every node of
// depth <= 2 (a 4-ary heap of <= 64 slots has depth <= 3)
template <bool KV0>
constexpr uint32_t kLaneWarpWords = (kFields<KV0> * 64u + 23u) * 32u;  // 27.5 KB / 35.7 KB
#endif
// one CTA per SM: 8 x 27.5 KB (kv = 0) or 6 x 35.7 KB of the 227 KB per CTA
#ifndef BELLMAN_LANE_WARPS0
#define BELLMAN_LANE_WARPS0 8
#endif
template <bool KV0>
constexpr uint32_t kLaneWarps = KV0 ? BELLMAN_LANE_WARPS0 : 6u;
constexpr uint32_t kLaneMaxCtas = 160;  // >= SM count (B200: 148)
// per-thread histograms in global memory (u32): e2e, ttft, r, similarity
// active / inactive (224 = 7 groups of 32 bins each for the 201 similarity bins)
constexpr uint32_t kHistE2E = 0, kHistTTFT = BELLMAN_HIST_LAT, kHistR = 2 * BELLMAN_HIST_LAT,
                   kHistQA = kHistR + BELLMAN_HIST_R, kHistQI = kHistQA + 224u, kHistRing = kHistQI + 224u,
                   kLaneHistWords = kHistRing + 8u;  // + the controller window's samples (8 words)
static_assert(kLaneHistWords % 4 == 0, "16-byte aligned per-thread histograms");
constexpr uint64_t kLaneMaxThreads = (uint64_t)kLaneMaxCtas * 32u * 8u;

// Which kernel runs a scenario: 0 the TBT-specialised warp engine (K2 <0>), 1
// the generic warp engine, 2 the multi-replica warp engine, 3 / 4 the
// lane-per-scenario engine K2L (kv = 0 / kv > 0).  K2L takes the scenarios of
// kind 0 on a Poisson trace whose instants fit 31 bits (horizon < 2^31 µs) and
// (so iteration indices stay below 2^31: t0 >= 1), unless lane_on is 0.
__host__ __device__ __forceinline__ uint32_t scenario_kind_of(const bellman_scenario &sc, const bellman_ctrl &cc,
                                                              const bellman_profile &pf, uint32_t trace_kind,
                                                              uint32_t lane_on) {
  if (pf.replicas > 1u) return 2u;
  if ((sc.record & BELLMAN_RECORD_SECONDS) != 0) return 1u;
  const bool tbto = cc.signal == BELLMAN_SIG_TBT && pf.prefill_mode == BELLMAN_PREFILL_NONBLOCKING &&
                    pf.kv_cap_words == 0 && pf.tpw_q16 == 0u && cc.law < BELLMAN_LAW_MPC;
  if (!tbto) return 1u;
  if (lane_on && trace_kind == 0u && sc.horizon_us < (1ll << 31))  // t0 >= 1: fewer than 2^31 iterations
    return pf.kv_ns_per_word == 0 ? 3u : 4u;
  return 0u;
}

}  // namespace bellman

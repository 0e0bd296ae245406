// bellman_kernels.cu — sm_100a kernels of the beLLMan scenario simulator.
//
// K2 bellman_tick_kernel: persistent; one warp simulates one scenario (a1-a9)
//    and fetches the next scenario id from a global counter when done.
// K5 bellman_calibrate_kernel: nearest-rank p50/p75 of recorded series (a10).
//
// Warp organisation:
//  * warp-uniform scalar state in registers: simulated clock, iteration,
//    batch size B and context K, controller, per-second accumulator, counters;
//  * lane-parallel request slots: slot s of lane l is batch slot l + 32 s
//    (max_batch <= 64 -> 2 slots per lane); admission ranks free slots with
//    ballot/popc, completions and prefill ends are ballot masks;
//  * lane-parallel arrival generator: 32 Philox candidates per refill, a warp
//    prefix sum of the exponential gaps, thinning by ballot, compaction by
//    __fns into a 32-entry register buffer that is the head of the FIFO queue;
//  * shared-memory latency histograms per warp, reduced to nearest-rank
//    percentiles by a warp scan and merged into segment histograms with
//    integer atomics (order-independent, hence bit-exact).
// No floating point except the final fp64 energy (IEEE _rn intrinsics, no FMA).
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "bellman_internal.cuh"

#ifdef BELLMAN_PROFILE_COUNTERS
// Development-only event counters (separate build, never the product .so).
__device__ unsigned long long g_prof[24];
// per-scenario [start, end) of run_one in %globaltimer ns (scenario ids < 2^16)
__device__ unsigned long long g_span[2 << 16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROF(i) (prof_[i]++)
// cycles spent in a handler (clock64 deltas; a profiling build only)
#define PROFC(i, stmt)                               \
  do {                                               \
    const long long c0_ = clock64();                 \
    stmt;                                            \
    prof_[i] += (uint32_t)(clock64() - c0_);         \
  } while (0)
#else
#define PROF(i) ((void)0)
#define PROFC(i, stmt) stmt
#endif
#ifdef BELLMAN_PROFILE_COUNTERS
#define PROF_MARK(v) const long long v = clock64()
#define PROF_ACC(i, v) (prof[i] += (uint32_t)(clock64() - v))
#else
#define PROF_MARK(v) ((void)0)
#define PROF_ACC(i, v) ((void)0)
#endif

namespace bellman {

constexpr unsigned FULL = 0xffffffffu;
// The event loop keeps instants as 32-bit offsets from a per-scenario epoch E
// (absolute time = E + offset, µs).  INF32: no such event; FAR32: an instant
// beyond the window.  advance() moves E to T once T >= kRebaseAt; idle jumps
// and leaps stop at kJumpCap, so every derived instant (T + d, d < 2^31; T +
// prefill < 2^31) stays below FAR32.
constexpr uint32_t INF32 = 0xffffffffu, FAR32 = 0xfffffffeu;
constexpr uint32_t kRebaseAt = 1u << 30, kJumpCap = 1u << 30;
// PH_PENDING: admitted under contending prefill (NEXT-4), prefill not started
constexpr uint32_t PH_EMPTY = 0, PH_PREFILL = 1, PH_READY = 2, PH_DEC = 3, PH_OFF = 4, PH_PENDING = 5;
constexpr uint64_t kLn2Q32 = 2977044472ull;  // round(ln 2 * 2^32)

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11) — counter (c0..c3), key (k0, k1).
__device__ __noinline__ uint4 philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                                        uint32_t c3) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// -ln(U), U = (2u+1)/2^33, in Q32 (reading R33): log2 by table + interpolation.
__device__ __forceinline__ uint64_t neglog_q32(uint32_t u, const uint2 *__restrict__ tab) {
  uint32_t e, x;
  if (u >= 0x80000000u) {  // v = 2u+1 >= 2^32: leading one at bit 32
    e = 32;
    x = 2u * u + 1u;  // v - 2^32 (mod 2^32)
  } else {
    const uint32_t v = 2u * u + 1u;
    e = 31u - __clz(v);
    x = (uint32_t)(((uint64_t)(v - (1u << e))) << (32u - e));
  }
  const uint2 t = __ldg(&tab[x >> 20]);
  const uint64_t f = x & 0xFFFFFu;
  const uint64_t log2v = ((uint64_t)e << 32) + t.x + (((uint64_t)t.y * f) >> 20);
  const uint64_t neg = (33ull << 32) - log2v;
  const uint64_t lo = neg * kLn2Q32, hi = __umul64hi(neg, kLn2Q32);
  return (hi << 32) | (lo >> 32);
}

// latency bin of a value in ms (a9): exact below 32, then 32 per octave.
__device__ __forceinline__ uint32_t lat_bin(uint64_t ms) {
  if (ms < 32) return (uint32_t)ms;
  const uint32_t e = 63u - (uint32_t)__clzll((long long)ms);
  if (e > 31) return BELLMAN_HIST_LAT - 1;
  return 32u * (e - 4u) + ((uint32_t)(ms >> (e - 5u)) & 31u);
}
// out of line: latencies of 2^32 µs (71 min) and more are rare
__device__ __noinline__ uint32_t lat_bin_wide(uint64_t us) { return lat_bin(us / 1000u); }
// latency bin of a value in µs: floor(us / 1000) ms, in 32 bits when it fits
__device__ __forceinline__ uint32_t lat_bin_us(uint64_t us) {
  if ((us >> 32) == 0) {
    const uint32_t ms = (uint32_t)us / 1000u;
    if (ms < 32) return ms;
    const uint32_t e = 31u - (uint32_t)__clz(ms);
    return 32u * (e - 4u) + ((ms >> (e - 5u)) & 31u);
  }
  return lat_bin_wide(us);
}
__device__ __forceinline__ uint32_t lat_edge(uint32_t b) {
  if (b < 32) return b;
  const uint32_t e = b / 32u + 4u, s = b % 32u;
  return (32u + s) << (e - 5u);
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// Warp sum of per-lane values < 2^48 with two REDUX.SUM (no 64-bit shuffles):
// low 22 bits and the rest are summed separately (each total < 2^32 for <= 64 terms).
__device__ __forceinline__ uint64_t warp_sum_split(uint64_t x) {
  const uint32_t lo = __reduce_add_sync(FULL, (uint32_t)(x & 0x3FFFFFu));
  const uint32_t hi = __reduce_add_sync(FULL, (uint32_t)(x >> 22));
  return ((uint64_t)hi << 22) + lo;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
// The lane index read once into a register the compiler cannot re-derive
// (it would otherwise rematerialize threadIdx.x & 31 with a slow S2R at each
// use on the event loop's critical path).
__device__ __forceinline__ uint32_t lane_pinned() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}
// this warp's index in its CTA (a constant 0 with one warp per CTA)
__device__ __forceinline__ uint32_t warp_in_block() { return kWarpsPerBlock == 1 ? 0u : threadIdx.x >> 5; }

// One queued request in the arrival lookahead buffer (32 bytes).
struct alignas(16) QEnt {
  uint64_t a;    // arrival time (absolute µs)
  uint32_t in;   // input words | request class << 16 (NEXT-3) | bypass rule holds << 31
  uint32_t U;    // realized unbounded length | similarity bin if not rewritten << 24
  uint32_t P;    // predicted length
  uint32_t fcq;  // compliance factor Q16 (bits 0-19) | similarity noise + 2048 (bits 20-31)
  uint32_t pf;   // prefill duration max(1, floor(prefill_ns * input / 1000)) µs
  uint32_t j;    // candidate index
};

// Cold per-scenario state: touched at events (admissions, completions,
// ingests, refills), not per iteration.  Lives in shared memory, one per warp,
// so the event loop keeps its hot state in registers without spilling.
// one entry written as two 16-byte stores (lanes write entries 32 bytes apart)
static_assert(sizeof(QEnt) == 32 && offsetof(QEnt, in) == 8 && offsetof(QEnt, P) == 16, "QEnt layout");

struct alignas(16) Cold {
  // a6 controller state, in 16-byte groups read with one LDS.128 each (g0..g4)
  uint64_t ringA;                                       // g0: window sum A,
  uint32_t ring_n, ring_pos;                            //     samples k, ring position
  uint32_t rung, active, activations, active_ingests;   // g1
  uint32_t first_act, last_deact, law, window;          // g2
  uint32_t t1, t2, rmin, rmax;                          // g3
  uint32_t *series;                                     // g4: recorded series (a10) or NULL,
  uint32_t series_n, series_cap;                        //     samples written, capacity
  uint32_t ring[8];   // last `window` per-second samples (a6)
  uint32_t rungs[8];  // word-limit ladder (R5)
  uint32_t nrungs, flags, dbg_cap, dbg_nctrl;
  const DevSeg *segs;
  uint64_t gen_tau;
  uint64_t w0, w1;
  uint64_t H;  // horizon (absolute µs)
  bellman_ctrl_row *dbg_ctrl;
  uint32_t n_seg, gen_seg, gen_fresh, gen_j, gen_acc, gen_cap, gen_done;
  uint32_t replay;  // NEXT-4: the trace is an explicit arrival list (segs unused)
  uint32_t rep_off;
  uint32_t k0, wid_lo, wid_hi;
  uint32_t bypass_mask, min_words, bypassed;  // NEXT-3
  uint32_t kv_cap;                            // NEXT-4 KV capacity in context words (0 = none)
  uint32_t pf_ns;                             // prefill ns per input word (token, tpw != 0)
  // KV-free cost law: floor((2^32 - 1) / cost(B)) for B = 0..max_batch, filled
  // lane-parallel at scenario start; the leap divides by cost(B) with it
  uint32_t cbm_tab[68];
  // a2/a3: the next <= 32 accepted arrivals (the head of the FIFO queue),
  // entry i written by lane i at refill, read whole (two 16-byte broadcasts)
  // by every lane at admission
  QEnt q[32];
  // round 2 additions, after the hot fields (their offsets unchanged)
  uint32_t tpw;                               // NEXT-4 tokens per word Q16, 0 = words (R44)
  // NEXT-3 MPC / BBR / PCC parameters and state (ingest_ext only)
  uint32_t hz, wlat, wq, wosc, step;          // horizon s, cost weights, step / delta bp
  uint32_t rt_min, phase, rbase;              // BBR RTprop; PCC phase and r_base
  uint64_t cost_a;                            // PCC: cost of the pair's first experiment
  uint32_t wring[8];                          // BBR: decode words of the window's seconds
};
static_assert(offsetof(Cold, ringA) == 0 && offsetof(Cold, rung) == 16 && offsetof(Cold, first_act) == 32 &&
                  offsetof(Cold, t1) == 48 && offsetof(Cold, series) == 64 && offsetof(Cold, ring) == 80,
              "controller state groups g0..g4 of Cold");

// At refill, per request and independent of r: whether a bypass rule (NEXT-3,
// S:267) holds, and the similarity bin it scores if not rewritten
// (NEXT-2: the inactive base plus its noise, clamped, in 0.5-point bins).
__device__ __forceinline__ void store_qent(QEnt &q, uint64_t a, uint32_t in, uint32_t U, uint32_t P, uint32_t fcq,
                                           uint32_t pf, uint32_t j, const Cold &c, uint32_t q_inactive) {
  const uint32_t byp = (((c.bypass_mask >> (in >> 16)) & 1u) || P < c.min_words) ? 1u : 0u;
  int32_t sc = (int32_t)q_inactive + (int32_t)(fcq >> 20) - 2048;
  sc = sc < 0 ? 0 : (sc > 10000 ? 10000 : sc);
  uint4 *w = reinterpret_cast<uint4 *>(&q);
  w[0] = make_uint4((uint32_t)a, (uint32_t)(a >> 32), in | (byp << 31), U | (((uint32_t)sc / 50u) << 24));
  w[1] = make_uint4(P, fcq, pf, j);
}


// a7 rewrite (R11): realized length of a request whose
// predicted length is P and compliance factor in fcq under r > 0:
// N = round(P (1 - r)), realized = clamp(round(poly(N) Fcomp), 1, 2^24).
// Out of line (one copy): it runs once per rewritten admission.
__device__ __noinline__ uint32_t rewrite_len(int64_t poly0, int64_t poly1, int64_t poly2, uint32_t fast, uint32_t P,
                                             uint32_t fcq, uint32_t ra) {
  uint32_t N = (P * (10000u - ra) + 5000u) / 10000u;  // P < 2^17: no overflow
  if (N < 1u) N = 1u;
  const int32_t fc = (int32_t)(fcq & 0xFFFFFu);
  if (fast) {  // host-checked coefficient bound: |poly(N) * fc| < 2^63, int64 suffices
    const int64_t n = N;
    const int64_t poly = poly0 + poly1 * n + poly2 * n * n;
    int64_t x = (poly * fc + (1ll << 31)) >> 32;  // floor (arithmetic shift)
    x = x < 1 ? 1 : (x > (1 << 24) ? (1 << 24) : x);
    return (uint32_t)x;
  }
  const __int128 poly = (__int128)poly0 + (__int128)poly1 * N + (__int128)poly2 * N * N;
  __int128 x = (poly * fc + ((__int128)1 << 31)) >> 32;  // floor (arithmetic shift)
  if (x < 1) x = 1;
  if (x > (1 << 24)) x = 1 << 24;
  return (uint32_t)x;
}

__device__ __forceinline__ uint32_t realized_len(const Params &p, uint32_t U, uint32_t P, uint32_t fcq, uint32_t ra) {
  if (ra == 0) return U;
  if (p.poly_fast) {  // the int64 path of rewrite_len, inline (one call site)
    uint32_t N = (P * (10000u - ra) + 5000u) / 10000u;
    if (N < 1u) N = 1u;
    const int64_t n = N;
    const int64_t poly = p.poly0 + p.poly1 * n + p.poly2 * n * n;
    int64_t x = (poly * (int32_t)(fcq & 0xFFFFFu) + (1ll << 31)) >> 32;
    x = x < 1 ? 1 : (x > (1 << 24) ? (1 << 24) : x);
    return (uint32_t)x;
  }
  return rewrite_len(p.poly0, p.poly1, p.poly2, p.poly_fast, P, fcq, ra);
}

// NEXT-2 similarity decay between the safe window and decay_end:
// q_active - floor((q_active - q_floor) X / D), 0 < X < D < 2^32, float
// estimate with an exact integer fix-up.  Out of line (rare branch).
__device__ __noinline__ int32_t sim_decay(uint32_t q_active, uint32_t q_floor, uint64_t X, uint64_t D) {
  const uint64_t aX = (uint64_t)(q_active - q_floor) * X;
  uint32_t q = (uint32_t)__fmul_rz((float)aX, __frcp_rn((float)D));
  while (q && (uint64_t)q * D > aX) q--;
  while ((uint64_t)(q + 1u) * D <= aX) q++;
  return (int32_t)q_active - (int32_t)q;
}

// a4/a5 leap, long runs: iterations of the batch with K growing by B each,
// 32 per step.  Lane j takes iteration n + j, whose gap is c + floor(kv (K +
// j B) / 1000) = cb + q + floor((rr + j ks) / 1000) with kv K = q 1000 + rr,
// ks = kv B <= 2^16; a saturating prefix sum (cap 2^30 > room) counts those
// that fit in `room`.  Returns (iterations, time used, q, rr) after them.
__device__ __noinline__ uint4 leap_wide(uint32_t lane, uint32_t cb, uint32_t q, uint32_t rr, uint32_t ks,
                                        uint32_t room, uint32_t left) {
  constexpr uint32_t kCap = 1u << 30;
  uint32_t n = 0, used = 0;
  while (n < left) {
    const uint32_t x = rr + lane * ks;
    uint32_t incl = cb + q + x / 1000u;
    incl = incl < kCap ? incl : kCap;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= (uint32_t)o) incl = min(incl + y, kCap);
    }
    const uint32_t c = __popc(__ballot_sync(FULL, incl <= room - used && lane < left - n));
    if (c == 0) break;
    used += __shfl_sync(FULL, incl, c - 1u);
    const uint32_t xc = rr + c * ks;
    q += xc / 1000u;
    rr = xc % 1000u;
    n += c;
    if (c < 32u) break;
  }
  return make_uint4(n, used, q, rr);
}

// prefill duration of a request with `in` input words (R6): >= 1 µs
// NEXT-4 token-level costs (R44): w words are clamp(round(w tpw), 1, 2^24)
// tokens (half-up, Q16; the realized-length bound of R11 holds in tokens too);
// tpw = 0 keeps words
__device__ __forceinline__ uint32_t to_tokens(uint32_t w, uint32_t tpw) {
  if (tpw == 0u) return w;
  const uint64_t t = ((uint64_t)w * tpw + (1u << 15)) >> 16;
  return t < 1u ? 1u : (t > (1u << 24) ? (1u << 24) : (uint32_t)t);
}

__device__ __forceinline__ uint32_t prefill_us(uint32_t pf_ns, uint32_t in) {
  const uint32_t pf = (uint32_t)(((uint64_t)pf_ns * in) / 1000u);
  return pf < 1u ? 1u : pf;
}

// Write-only counters (a8) are lane-distributed: counter i lives in lane i's
// register `ctr` and is bumped with a predicated add of a warp-uniform value
// (no branch, no memory), then read once by shuffle in the epilogue.
enum : uint32_t { CT_ADMITTED = 0, CT_SERVED = 1, CT_REWRITTEN = 2, CT_SLO_VIOL = 3, CT_WIN_SERVED = 4, CT_WORDS_IN = 5, CT_IDLE = 6, CT_WIN_WORDS_IN = 7, CT_WIN_IDLE = 8, CT_SUM_QUEUE = 9, CT_SUM_TTFT = 10, CT_SUM_E2E = 11, CT_PREEMPT = 12, CT_RECOMP = 13, CT_N };

// One Cold block per warp of the CTA, in static shared memory so that every
// access is a 32-bit LDS/STS off a known base (no generic pointer).
__shared__ Cold g_cold[kWarpsPerBlock];
__shared__ WarpHist g_hist[kWarpsPerBlock];

// ---------------------------------------------------------------------------
// a2 + a3: refill the warp's shared arrival buffer with the next accepted
// candidates (P:183 Poisson arrivals, S:83 thinning; R17, R32, R33).  Lane l
// draws candidate j + l: Philox block, -ln U, then a warp prefix sum of the
// exponential gaps gives the candidate times; thinning by ballot; accepted
// candidates are compacted (__fns) into entries 0..n-1 together with their
// per-request draws (tag-1 block).  Out of line: it runs once per ~32 arrivals.
// Returns n (0 only when the generator is exhausted).
//
// COUNT = true (the epilogue's queue count, a8): the same candidate stream,
// but accepted arrivals are only counted while they precede `end` — no
// per-request draws, no buffer writes — until the first at or after `end`
// or the end of the trace; the count and last_j (index of the last counted
// arrival + 1, from `last_j` on) are returned as (count lo, count hi, last_j).
// Otherwise returns (n, 0, 0).
template <bool DBG, bool COUNT = false>
__device__ __noinline__ uint4 refill_buffer(const Params &p, uint32_t wid, uint32_t lane, bellman_second_row *dbg,
                                            uint32_t dbg_cap, uint64_t end = 0, uint32_t last_j = 0) {
  Cold &c = g_cold[kWarpsPerBlock == 1 ? 0u : wid];
  const uint64_t H = DBG ? c.H : 0u;  // debug rows count arrivals before the horizon
  __syncwarp();  // every lane's reads of the previous buffer precede the new writes
  uint32_t gen_done = c.gen_done, gen_seg = c.gen_seg, gen_fresh = c.gen_fresh, gen_j = c.gen_j;
  uint32_t gen_acc = c.gen_acc;
  uint64_t gen_tau = c.gen_tau;
  const uint32_t n_seg = c.n_seg, gen_cap = c.gen_cap, k0 = c.k0, wid_lo = c.wid_lo, wid_hi = c.wid_hi;
  const DevSeg *segs = c.segs;
  uint32_t n = 0;
  bool reached = false;  // COUNT: an accepted arrival at or after `end` was met
  uint64_t cn = 0;
  uint32_t lj = last_j;
  if (__builtin_expect(c.replay != 0, 0)) {  // NEXT-4 replay: entries gen_j .. gen_j+31 of the list, draws keyed by index
    do {
      uint32_t left = gen_done ? 0u : n_seg - gen_j;
      if (gen_cap && gen_cap - gen_acc < left) left = gen_cap - gen_acc;
      n = left < 32u ? left : 32u;
      uint64_t tau = 0;
      if (lane < n) {
        const uint32_t jj = gen_j + lane;
        const bellman_arrival A = p.arrivals[c.rep_off + jj];
        tau = (uint64_t)A.a_us;
        if (!COUNT) {
          const uint4 v = philox(k0, kSeedHi, jj, 1u, wid_lo, wid_hi);
          const uint64_t U = ((uint64_t)A.L_words * (uint32_t)__ldg(&p.tabF[v.x >> 20]) + 32768u) >> 16;
          const int32_t P0 = (int32_t)A.L_words + __ldg(&p.tabN[v.y >> 20]);
          const uint32_t in_t = to_tokens(A.input_words, c.tpw);  // the engine's input (R44)
          store_qent(c.q[lane], tau, in_t | (A.cls << 16), U < 1 ? 1u : (uint32_t)U,
                     P0 < 1 ? 1u : (uint32_t)P0,
                     (uint32_t)__ldg(&p.tabC[v.z >> 20]) | ((uint32_t)(__ldg(&p.tabQ[v.w >> 20]) + 2048) << 20),
                     prefill_us(c.pf_ns, in_t), jj, c, p.q_inactive);
        }
        if (DBG && dbg && tau < H) {
          const uint64_t sidx = tau / kUs;
          atomicAdd(&dbg[sidx < dbg_cap ? sidx : dbg_cap - 1u].arrivals, 1u);
        }
      }
      if (COUNT) {  // the list is in time order: the entries before `end` are a prefix
        const uint32_t before = __ballot_sync(FULL, lane < n && tau < end);
        cn += (uint32_t)__popc(before);
        if (before) lj = gen_j + 32u - (uint32_t)__clz(before);
        reached = before != (n >= 32u ? FULL : ((1u << n) - 1u));
      }
      gen_j += n;
      gen_acc += n;
      if (n == 0 || gen_j >= n_seg || (gen_cap && gen_acc >= gen_cap)) gen_done = 1;
    } while (COUNT && !gen_done && !reached);
    if (COUNT) n = 0;
  }
  while (!c.replay && !gen_done && n == 0 && !reached) {
    if (gen_seg >= n_seg) {
      gen_done = 1;
      break;
    }
    const DevSeg S = segs[gen_seg];
    if (gen_fresh) {
      gen_tau = S.ta;
      gen_fresh = 0;
    }
    const uint32_t jj = gen_j + lane;
    const uint4 u = philox(k0, kSeedHi, jj, 0u, wid_lo, wid_hi);
    const uint64_t delta = __umul64hi(neglog_q32(u.x, p.log2tab), S.M);
    uint64_t incl = delta;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    const uint64_t tau = gen_tau + incl;
    const uint32_t om = __ballot_sync(FULL, tau >= S.tb);
    const uint32_t first_over = om ? (uint32_t)(__ffs(om) - 1) : 32u;
    bool acc = false;
    if (lane < first_over) {
      // thinning: u1 * lmax * span < (la (tb - tau) + lb (tau - ta)) * 2^32, in 128 bits
      const uint64_t x = (uint64_t)u.y * S.lmax;
      const uint64_t lhs_hi = __umul64hi(x, S.span), lhs_lo = x * S.span;
      const uint64_t y = (uint64_t)S.la * (S.tb - tau) + (uint64_t)S.lb * (tau - S.ta);
      const uint64_t rhs_hi = y >> 32, rhs_lo = y << 32;
      acc = lhs_hi < rhs_hi || (lhs_hi == rhs_hi && lhs_lo < rhs_lo);
    }
    uint32_t am = __ballot_sync(FULL, acc);
    if (gen_cap) {
      const uint32_t room = gen_cap - gen_acc;
      if ((uint32_t)__popc(am) >= room) {
        const uint32_t cut = room ? __fns(am, 0, (int)room) : 0u;  // position of room-th set bit
        am = room ? (am & (0xffffffffu >> (31u - cut))) : 0u;
        gen_done = 1;
      }
    }
    const bool mine = (am >> lane) & 1u;
    if (COUNT) {  // candidate times increase with the lane: those before `end` are a prefix
      const uint32_t before = __ballot_sync(FULL, mine && tau < end);
      cn += (uint32_t)__popc(before);
      if (before) lj = gen_j + 32u - (uint32_t)__clz(before);
      reached = before != am;
      if (DBG && dbg && mine && tau < H) {
        const uint64_t sidx = tau / kUs;
        atomicAdd(&dbg[sidx < dbg_cap ? sidx : dbg_cap - 1u].arrivals, 1u);
      }
    } else {
      n = (uint32_t)__popc(am);
    }
    // compaction: the accepted candidate of rank l lands in entry l
    if (!COUNT && mine) {
      const uint32_t e = __popc(am & ((1u << lane) - 1u));
      const uint32_t L = (uint32_t)__ldg(&p.tabL[u.z >> 20]);
      const uint32_t x = u.z & 0xFFFFFu;  // class draw from the bits below L's index (NEXT-3)
      const uint32_t cls = x < p.class_cum0 ? 0u : (x < p.class_cum1 ? 1u : (x < p.class_cum2 ? 2u : 3u));
      const uint32_t in = to_tokens((uint32_t)__ldg(&p.tabI[u.w >> 20]), c.tpw);  // engine units (R44)
      const uint4 v = philox(k0, kSeedHi, jj, 1u, wid_lo, wid_hi);  // a3: the request's own draws
      const uint64_t U = ((uint64_t)L * (uint32_t)__ldg(&p.tabF[v.x >> 20]) + 32768u) >> 16;  // S:139, R14
      const int32_t P0 = (int32_t)L + __ldg(&p.tabN[v.y >> 20]);
      store_qent(c.q[e], tau, in | (cls << 16), U < 1 ? 1u : (uint32_t)U, P0 < 1 ? 1u : (uint32_t)P0,
                 (uint32_t)__ldg(&p.tabC[v.z >> 20]) | ((uint32_t)(__ldg(&p.tabQ[v.w >> 20]) + 2048) << 20),
                 prefill_us(c.pf_ns, in), jj, c, p.q_inactive);
      if (DBG && dbg && tau < H) {
        const uint64_t sidx = tau / kUs;
        atomicAdd(&dbg[sidx < dbg_cap ? sidx : dbg_cap - 1u].arrivals, 1u);
      }
    }
    gen_acc += (uint32_t)__popc(am);
    if (first_over < 32u) {
      gen_j += first_over + 1u;  // the crossing candidate is consumed (R17)
      gen_seg++;
      gen_fresh = 1;
    } else {
      gen_j += 32u;
      gen_tau = __shfl_sync(FULL, tau, 31);
    }
  }
  __syncwarp();
  if (!COUNT && lane == 0) {
    c.gen_done = gen_done;
    c.gen_seg = gen_seg;
    c.gen_fresh = gen_fresh;
    c.gen_j = gen_j;
    c.gen_acc = gen_acc;
    c.gen_tau = gen_tau;
  }
  __syncwarp();
  return COUNT ? make_uint4((uint32_t)cn, (uint32_t)(cn >> 32), lj, 0u) : make_uint4(n, 0u, 0u, 0u);
}

// floor(a / b), b > 0: a 32-bit division when both fit (the per-second means
// and the law's quotient almost always do), else the 64-bit routine.
__device__ __forceinline__ uint64_t div_u64(uint64_t a, uint64_t b) {
  if (((a | b) >> 32) == 0) return (uint32_t)a / (uint32_t)b;
  return a / b;
}

// ---------------------------------------------------------------------------
// a6, NEXT-3 laws after P:213 (readings R41-R43, include/bellman_sim.h): MPC,
// BBR-style and PCC-style, one ingest of sample x of the closed second ending
// at sec_bound, w = the decode words emitted in that second (acc_cnt of the
// TBT signal; BBR is TBT-only).  Out of line (one copy, called at most once
// per simulated second), so the MAP / STEP event loops keep their footprint.
// The window ring and its sum are shared with MAP / STEP.  MPC evaluates its
// <= 32 candidate rates one per lane (128-bit exact costs) and takes the
// warp's lexicographic (cost, index) minimum with five xor-shuffle steps; BBR
// and PCC are warp-uniform scalar updates.  Lane 0 writes the state.
__device__ __forceinline__ unsigned __int128 shfl_xor_u128(unsigned __int128 v, int m) {
  const uint64_t lo = __shfl_xor_sync(FULL, (unsigned long long)(uint64_t)v, m);
  const uint64_t hi = __shfl_xor_sync(FULL, (unsigned long long)(uint64_t)(v >> 64), m);
  return ((unsigned __int128)hi << 64) | lo;
}

template <bool DBG>
__device__ __noinline__ uint32_t ingest_ext(uint32_t wid, uint32_t lane, uint64_t sec_bound, uint32_t x, uint32_t w,
                                            uint32_t r_cur, bool dbg) {
  Cold &c = g_cold[kWarpsPerBlock == 1 ? 0u : wid];
  const uint32_t law = c.law, window = c.window, pos = c.ring_pos, t1 = c.t1, rmin = c.rmin, rmax = c.rmax;
  const uint32_t was_active = c.active, nrungs = c.nrungs;
  uint32_t k = c.ring_n, rung = c.rung;
  uint64_t A = c.ringA;
  if (k < window) {
    k++;
    A += x;
  } else {
    A = A + x - c.ring[pos];
  }
  const uint32_t npos = pos + 1u == window ? 0u : pos + 1u;
  // the window's oldest sample once x is in: ring[0] while filling, else the slot after x
  const uint32_t y1 = k == 1u ? x : (k < window ? c.ring[0] : c.ring[npos]);
  uint32_t nr = 0, act = 0;
  uint32_t rt_min = c.rt_min, phase = c.phase, rbase = c.rbase;
  uint64_t cost_a = c.cost_a;
  if (law == BELLMAN_LAW_MPC) {
    // forecast F = A/k + h (x - y1)/(k - 1) as F_num / D; costs scaled by 10^4 D
    int64_t Fn;
    uint64_t D;
    if (k >= 2u) {
      D = (uint64_t)k * (k - 1u);
      Fn = (int64_t)A * (int64_t)(k - 1u) + (int64_t)c.hz * (int64_t)k * ((int64_t)x - (int64_t)y1);
    } else {
      D = 1;
      Fn = (int64_t)A;
    }
    const uint64_t F = Fn < 0 ? 0ull : (uint64_t)Fn;
    const uint32_t nc = nrungs ? nrungs + 1u : 32u;
    uint32_t cand = 0;
    if (lane >= 1u && lane < nc)
      cand = nrungs ? c.rungs[lane - 1u] : rmin + (uint32_t)((uint64_t)(lane - 1u) * (rmax - rmin) / 30u);
    unsigned __int128 J = ~(unsigned __int128)0;
    if (lane < nc) {
      const unsigned __int128 lat = (unsigned __int128)F * (10000u - cand);
      const unsigned __int128 thr = (unsigned __int128)t1 * 10000u * D;
      const unsigned __int128 ex = lat > thr ? lat - thr : 0;
      const uint32_t dr = cand > r_cur ? cand - r_cur : r_cur - cand;
      J = (unsigned __int128)c.wlat * ex +
          (unsigned __int128)(10000ull * D) * ((uint64_t)c.wq * cand + (uint64_t)c.wosc * dr);
    }
    uint32_t idx = lane;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const unsigned __int128 Jo = shfl_xor_u128(J, m);
      const uint32_t io = __shfl_xor_sync(FULL, idx, m);
      if (Jo < J || (Jo == J && io < idx)) {
        J = Jo;
        idx = io;
      }
    }
    nr = __shfl_sync(FULL, cand, (int)idx);
    act = nr > 0u;
  } else if (law == BELLMAN_LAW_BBR) {
    if (x < rt_min) rt_min = x;
    uint32_t bw = w;  // the window's other seconds: wring holds them (0 where unfilled)
    for (uint32_t i = 0; i < window; ++i)
      if (i != pos && c.wring[i] > bw) bw = c.wring[i];
    const bool congested = A >= (uint64_t)k * ((uint64_t)rt_min + t1);
    const bool plateau = 8ull * w >= 7ull * bw;
    nr = r_cur;
    if (congested && plateau) {
      if (nrungs) {
        rung = r_cur == 0u ? 0u : (rung + 1u < nrungs ? rung + 1u : rung);
        nr = c.rungs[rung];
      } else {
        nr = r_cur == 0u ? rmin : (r_cur + c.step > rmax ? rmax : r_cur + c.step);
      }
    } else if (!congested) {
      if (nrungs) {
        if (r_cur == 0u || rung == 0u) {
          nr = 0;
        } else {
          rung--;
          nr = c.rungs[rung];
        }
      } else {
        nr = r_cur <= rmin ? 0u : (r_cur < rmin + c.step ? rmin : r_cur - c.step);
      }
    }
    act = nr > 0u;
  } else {  // BELLMAN_LAW_PCC
    act = A >= (uint64_t)k * t1;
    const uint32_t d = c.step;
    if (!act) {
      phase = 0;
      rbase = 0;
      nr = 0;
    } else {
      const uint64_t cost = (uint64_t)c.wlat * (x > t1 ? x - t1 : 0u) + (uint64_t)c.wq * r_cur;
      if (phase == 0u) {
        rbase = rmin;
      } else if (phase == 1u) {
        cost_a = cost;
      } else {
        if (cost_a < cost) rbase = rbase + d > rmax ? rmax : rbase + d;
        else if (cost < cost_a) rbase = rbase < rmin + d ? rmin : rbase - d;
      }
      if (phase == 1u) {
        nr = rbase < rmin + d ? rmin : rbase - d;
        phase = 2;
      } else {
        nr = rbase + d > rmax ? rmax : rbase + d;
        phase = 1;
      }
    }
  }
  const uint32_t nctrl = DBG ? c.dbg_nctrl : 0u;
  __syncwarp();
  if (lane == 0) {
    c.ring[pos] = x;
    c.wring[pos] = w;
    c.ringA = A;
    c.ring_n = k;
    c.ring_pos = npos;
    c.rung = rung;
    c.rt_min = rt_min;
    c.phase = phase;
    c.rbase = rbase;
    c.cost_a = cost_a;
    c.active = act;
    c.activations += (act && !was_active) ? 1u : 0u;
    c.active_ingests += act;
    if (act != (was_active != 0)) {  // the log is kept by second index (R21)
      const uint32_t second = (uint32_t)(sec_bound / kUs - 1u);
      if (act) {
        if (c.first_act == BELLMAN_NONE) c.first_act = second;
      } else {
        c.last_deact = second;
      }
    }
    if (DBG && dbg) {
      if (nctrl < c.dbg_cap) {
        bellman_ctrl_row cr;
        cr.second = (uint32_t)(sec_bound / kUs - 1u);
        cr.sample = x;
        cr.k = k;
        cr.r_bp = nr;
        cr.active = act;
        cr._pad = 0;
        cr.A = A;
        c.dbg_ctrl[nctrl] = cr;
      }
      c.dbg_nctrl = nctrl + 1u;
    }
  }
  __syncwarp();
  return nr;
}

// ---------------------------------------------------------------------------
// a6: one controller ingest of the closed second ending at sec_bound, whose
// sample is the integer mean x = floor(acc_sum / acc_cnt) (P:134, P:193,
// S:283-301; R3-R5, R12, R38).  Out of line, the 64-bit division included: it
// runs once per simulated second, so it stays out of the event loop's
// instruction-cache footprint.  All lanes compute; only lane 0 writes the
// shared-memory state.
template <bool DBG, bool EXT = true>
__device__ __forceinline__ uint32_t ingest_body(uint32_t wid, uint32_t lane, uint64_t sec_bound, uint64_t acc_sum,
                                               uint32_t acc_cnt, uint32_t r_cur, bool dbg, uint32_t util_maxb) {
  Cold &c = g_cold[kWarpsPerBlock == 1 ? 0u : wid];
  // the whole controller state in five independent 16-byte loads
  const uint4 *g = reinterpret_cast<const uint4 *>(&c.ringA);
  const uint4 g0 = g[0], g1 = g[1], g2 = g[2], g3 = g[3], g4 = g[4];
  // the sample: floor(acc_sum / acc_cnt) truncated to 32 bits (as the oracle); UTIL
  // keeps sum B / count and scales once here: floor(10000 sum B / (max_batch count))
  const uint32_t x = util_maxb ? (uint32_t)(10000u * acc_sum / ((uint64_t)util_maxb * acc_cnt))
                               : (uint32_t)div_u64(acc_sum, acc_cnt);
  uint32_t *const series = reinterpret_cast<uint32_t *>((uint64_t)g4.x | ((uint64_t)g4.y << 32));
  if (series) {
    const uint32_t n = g4.z;
    __syncwarp();  // every lane's read of the state precedes lane 0's write
    if (lane == 0) {
      if (n < g4.w) series[n] = x;
      else c.flags |= BELLMAN_FLAG_SERIES_OVERFLOW;
      c.series_n = n + 1u;
    }
    __syncwarp();
  }
  const uint32_t law = g2.z, window = g2.w;
  if (law != BELLMAN_LAW_MAP && law != BELLMAN_LAW_STEP)
    return (EXT && law >= BELLMAN_LAW_MPC) ? ingest_ext<DBG>(wid, lane, sec_bound, x, acc_cnt, r_cur, dbg) : r_cur;
  const uint32_t pos = g0.w, t1 = g3.x, was_active = g1.y;
  uint32_t k = g0.z, rung = g1.x;
  uint64_t A = (uint64_t)g0.x | ((uint64_t)g0.y << 32);
  const uint32_t ev = c.ring[pos];
  if (k < window) {
    k++;
    A += x;
  } else {
    A = A + x - ev;
  }
  const bool act = A >= (uint64_t)k * t1;  // non-strict (R38)
  uint32_t nr = 0;
  if (act) {
    if (law == BELLMAN_LAW_MAP) {
      const uint32_t rmin = g3.z, rmax = g3.w;
      uint64_t rr = rmin + div_u64((uint64_t)(rmax - rmin) * (A - (uint64_t)k * t1), (uint64_t)k * (g3.y - t1));
      if (rr > rmax) rr = rmax;
      nr = (uint32_t)rr;
      const uint32_t nrungs = c.nrungs;
      if (nrungs) {  // largest rung <= r (R5)
        uint32_t best = c.rungs[0];
        for (uint32_t i = 1; i < nrungs; ++i)
          if (c.rungs[i] <= nr) best = c.rungs[i];
        nr = best;
      }
    } else {  // STEP: rung 0 on activation, one rung up per ingest while active
      rung = was_active ? (rung + 1u < c.nrungs ? rung + 1u : rung) : 0u;
      nr = c.rungs[rung];
    }
  }
  const uint32_t nctrl = DBG ? c.dbg_nctrl : 0u;
  __syncwarp();
  if (lane == 0) {
    c.ring[pos] = x;
    uint4 *gw = reinterpret_cast<uint4 *>(&c.ringA);
    gw[0] = make_uint4((uint32_t)A, (uint32_t)(A >> 32), k, (pos + 1u == window) ? 0u : pos + 1u);
    gw[1] = make_uint4(rung, act, g1.z + (act && !was_active), g1.w + act);
    if (act != (was_active != 0)) {  // the log is kept by second index (R21)
      const uint32_t second = (uint32_t)(sec_bound / kUs - 1u);
      if (act) {
        if (g2.x == BELLMAN_NONE) c.first_act = second;
      } else {
        c.last_deact = second;
      }
    }
    if (DBG && dbg) {
      if (nctrl < c.dbg_cap) {
        bellman_ctrl_row cr;
        cr.second = (uint32_t)(sec_bound / kUs - 1u);
        cr.sample = x;
        cr.k = k;
        cr.r_bp = nr;
        cr.active = act;
        cr._pad = 0;
        cr.A = A;
        c.dbg_ctrl[nctrl] = cr;
      }
      c.dbg_nctrl = nctrl + 1u;
    }
  }
  __syncwarp();
  return nr;
}


template <bool DBG>
__device__ __noinline__ uint32_t ingest_sample(uint32_t wid, uint32_t lane, uint64_t sec_bound, uint64_t acc_sum,
                                               uint32_t acc_cnt, uint32_t r_cur, bool dbg, uint32_t util_maxb) {
  return ingest_body<DBG>(wid, lane, sec_bound, acc_sum, acc_cnt, r_cur, dbg, util_maxb);
}

// ---------------------------------------------------------------------------
// The per-scenario simulation.  Every scalar is warp-uniform.  Derived
// quantities are maintained incrementally so that an event trip does no
// division: the cost base c = t0 + slope max(0, B - knee), the KV term as
// kv K = kq 1000 + kr, the window flag and its next boundary, the arrival time
// of the queue head.
// runs of at most 2^BELLMAN_LEAP_SHIFT iterations are leaped one at a time
// (else 32 per step, lane-parallel)
#ifndef BELLMAN_LEAP_SHIFT
#define BELLMAN_LEAP_SHIFT 3
#endif

// XT (with TBTO): the TBT-specialised loop extended with the runtime features
// the product loop leaves out — token units, NEXT-3 laws, KV-reserve capacity —
// for the generic kernel's TBT scenarios (the product kernel never has XT).
template <bool DBG, bool TBTO, bool KV0 = false, bool XT = false>
struct Sim {
  __device__ explicit Sim(uint32_t w) : wid(w) {}
  // the selected signal is x: a compile-time answer in the TBT-only
  // instantiation (every benchmark configuration), a runtime one otherwise
  __device__ __forceinline__ bool sig(uint32_t x) const { return TBTO ? x == BELLMAN_SIG_TBT : signal == x; }
  // contending prefill (NEXT-4): never in the TBT-specialised instantiation
  __device__ __forceinline__ bool cont() const { return TBTO ? false : pmode != 0u; }
  __device__ __forceinline__ uint32_t n_pending() const { return cont() ? n_pend : 0u; }
  // the KV term's coefficient: a compile-time 0 in the KV-free instantiation
  __device__ __forceinline__ uint32_t kvc() const { return KV0 ? 0u : kv; }
  // NEXT-4 KV preemption (kv_policy 1): never in the TBT-specialised instantiation
  __device__ __forceinline__ bool pre() const { return TBTO ? false : kvpol != 0u; }
  __device__ __forceinline__ bool stk_any() const { return pre() && pstk != 0u; }
  __device__ __forceinline__ Cold &cold() const { return g_cold[kWarpsPerBlock == 1 ? 0u : wid]; }
#ifndef BELLMAN_AB_REGCTR
  uint64_t ctr;  // lane-distributed write-only counters (CT_*)
  __device__ __forceinline__ void cadd(uint32_t i, uint64_t v) { ctr += (lane == i) ? v : 0ull; }
  __device__ __forceinline__ uint64_t cget(uint32_t i) const { return __shfl_sync(FULL, ctr, i); }
#else
  uint64_t ctrs[CT_N];
  __device__ __forceinline__ void cadd(uint32_t i, uint64_t v) { ctrs[i] += v; }
  __device__ __forceinline__ uint64_t cget(uint32_t i) const { return ctrs[i]; }
#endif
  uint32_t lane;
  uint32_t wid;  // warp index in the CTA: selects this warp's Cold block
#ifdef BELLMAN_PROFILE_COUNTERS
  uint32_t *prof;
#endif
  // ---- clock (a4): absolute time = E + 32-bit offset (INF32 / FAR32 above)
  uint64_t E;
  uint32_t Hr;  // horizon offset (FAR32 when beyond the window)
  // profile
  uint32_t kv, maxb;
  // controller
  uint32_t signal;
  uint32_t r;
  // per-second accumulator of the selected signal (a6)
  uint32_t sec_bound;  // offset of (open second + 1) * 1e6, INF32 when nothing consumes the signal
  uint64_t acc_sum;
  uint32_t acc_cnt;
  // recording (a10 source)
  // debug record mode (NEXT-1): per-second rows and controller log, NULL when off
  bellman_second_row *dbg;
  // profile constants used at events
  uint32_t t0, knee, slope, slo_us;
  // ---- counters (a8), updated at events
  uint32_t last_j;
  // ---- serving state (a4, a5, a7)
  uint32_t T;
  uint32_t busy;
  uint32_t iter_end;
  uint32_t iter_d;
  uint64_t iter_align;
  uint32_t ticks;      // iterations started; the running one has index ticks-1
  uint32_t next_done;  // min completion iteration over decoding slots
  uint32_t next_pf;    // min prefill end over prefilling slots
  uint32_t n_ready, B, in_sys;
  uint32_t cbase;             // t0 + slope * max(0, B - knee)
  uint32_t kq, kr;            // kv * K = kq * 1000 + kr, K = context words of the batch
  uint32_t kstep_q, kstep_r;  // kv * B = kstep_q * 1000 + kstep_r (growth per iteration)
  uint32_t win_now;           // T in [w0, w1)
  uint32_t win_next;          // next window boundary after T (INF32 if none)
  uint32_t stop_static;       // min(Hr, win_next)
  // slots (lane-parallel): arrival (absolute), prefill end (offset)
  uint64_t sa[2];
  uint32_t sp[2];
  uint32_t sR[2], sin[2], sdn[2], sph[2];
  // NEXT-4 multi-replica path (R45; generic instantiation only): the replica
  // of each slot; lane q < nrep holds replica q's iteration end (INF32 idle);
  // sdn counts a slot's words emitted there and sp its last word's instant
  uint32_t srep[2];
  uint32_t re;
  uint32_t nrep, route, rrp;
  // ---- generator / queue head (a2)
  uint32_t buf_h, buf_n;  // consumed / filled entries of the shared arrival buffer
  uint32_t pmode;         // NEXT-4 prefill_mode (generic instantiation only)
  uint32_t n_pend, pend_us;  // contending: admitted, prefill not started; sum of their prefill times
  uint32_t kv_res;        // NEXT-4: contexts in the system: reserve policy sum of (input + R),
                          // preempt policy sum of (input + words emitted)
  uint32_t kvpol;         // NEXT-4: kv_policy 1 with a capacity (generic instantiation only)
  uint32_t pstk, pseq;    // preempted requests waiting at the queue front; next admission order
  PreScratch *ps;         // this CTA's preemption scratch
  uint32_t adm_blocked;   // NEXT-4: the arrived queue head does not fit the KV capacity
  uint32_t head_t;     // arrival offset of the queue head (0 if before E), INF32 when none remains
  // ---- counters (a8)
  uint64_t words_out, win_words_out;

  __device__ __forceinline__ uint64_t ab(uint32_t t) const { return E + t; }
  // offset of an absolute instant x: 0 if x <= E (the past), FAR32 if beyond the window
  __device__ __forceinline__ uint32_t rel(uint64_t x) const {
    return x <= E ? 0u : (x - E >= FAR32 ? FAR32 : (uint32_t)(x - E));
  }

  // ------------------------------------------------------------------ a2
  __device__ __forceinline__ void refill(const Params &p) {
    buf_h = 0;
    buf_n = refill_buffer<DBG>(p, wid, lane, DBG ? dbg : nullptr, DBG ? cold().dbg_cap : 0u).x;
    head_t = buf_n ? rel(cold().q[0].a) : INF32;
  }

  // ------------------------------------------------------------------ a6
  __device__ __forceinline__ void ingest() {
    // the TBT loops take the controller inline (C5's paper-trace scenarios
    // ingest every second of long quiet stretches); the others call it
    if (TBTO && !DBG)  // the TBT loops run MAP / STEP / CONST / OFF only (no ingest_ext call site)
      r = ingest_body<DBG, XT>(wid, lane, ab(sec_bound), acc_sum, acc_cnt, r, false, 0u);
    else
      r = ingest_sample<DBG>(wid, lane, ab(sec_bound), acc_sum, acc_cnt, r, DBG && dbg != nullptr,
                           sig(BELLMAN_SIG_UTIL) ? maxb : 0u);
  }

  // close the open second (if it holds samples) and open the one containing t
  __device__ __forceinline__ void roll_second(uint32_t t) {
    if (t < sec_bound) return;
    if (acc_cnt) {
      ingest();
      adm_blocked = 0;  // r may have changed: the queue head may fit now
    }
    acc_sum = 0;
    acc_cnt = 0;
    // the second containing t: usually the next one (no division)
    const uint32_t nb = sec_bound + (uint32_t)kUs;
    sec_bound = ((t < nb) & (nb < FAR32)) ? nb : rel((ab(t) / kUs + 1u) * kUs);
  }

  // debug row of the second containing absolute instant ta
  __device__ __forceinline__ bellman_second_row *row(uint64_t ta) const {
    const uint64_t sidx = ta / kUs;
    return dbg + (sidx < cold().dbg_cap ? sidx : cold().dbg_cap - 1u);
  }

  // idle interval [a, b) (absolute) split over the seconds it overlaps (debug rows only)
  __device__ __forceinline__ void dbg_idle(uint64_t a, uint64_t b) {
    if (!dbg || lane != 0) return;
    for (uint64_t sidx = a / kUs; sidx * kUs < b; ++sidx) {
      const uint64_t lo = a > sidx * kUs ? a : sidx * kUs, hi = b < (sidx + 1) * kUs ? b : (sidx + 1) * kUs;
      atomicAdd(&row(sidx * kUs)->idle_us, (uint32_t)(hi - lo));
    }
  }

  __device__ __forceinline__ void update_window() {
    const uint64_t Ta = ab(T), w0 = cold().w0, w1 = cold().w1;
    win_now = Ta >= w0 && Ta < w1;
    win_next = Ta < w0 ? rel(w0) : (Ta < w1 ? rel(w1) : INF32);
    stop_static = Hr < win_next ? Hr : win_next;
  }

  // move the epoch to T: offsets of pending instants shrink by T (slot prefill
  // ends modulo 2^32: a ready slot's end lies in the past and is only used in
  // differences); instants kept absolute elsewhere are re-derived
  __device__ __forceinline__ void rebase() {
    const uint32_t D = T;
    E += D;
    T = 0;
    iter_end -= D;  // meaningful only while busy
    if (next_pf != INF32) next_pf -= D;
    if (sec_bound != INF32) sec_bound -= D;
    sp[0] -= D;
    sp[1] -= D;
    if (!TBTO && nrep > 1u && re != INF32) re -= D;
    head_t = buf_h < buf_n ? rel(cold().q[buf_h].a) : INF32;
    Hr = rel(cold().H);
    update_window();
  }

  // move the clock to an event instant t >= T
  __device__ __forceinline__ void advance(uint32_t t) {
    T = t;
    // one compare against the earliest of the three boundaries (one branch in
    // the common case, where none is crossed)
    if (__builtin_expect(t < umin(umin(sec_bound, win_next), kRebaseAt), 1)) return;
    roll_second(t);
    if (t >= win_next) update_window();
    if (__builtin_expect(t >= kRebaseAt, 0)) rebase();
  }

  // B changed: cost base and per-iteration KV growth
  __device__ __forceinline__ void batch_changed() {
    cbase = t0 + slope * (B > knee ? B - knee : 0u);
    if (KV0) return;
    const uint32_t ks = kv * B;
    kstep_q = ks / 1000u;
    kstep_r = ks - kstep_q * 1000u;
  }
  __device__ __forceinline__ void kv_add(uint64_t x) {  // kv K += x
    if (KV0) return;
    const uint64_t q = x / 1000u;  // constant divisor: a multiply-high sequence, no branch
    kr += (uint32_t)(x - q * 1000u);
    kq += (uint32_t)q;
    if (kr >= 1000u) {
      kr -= 1000u;
      kq++;
    }
  }
  __device__ __forceinline__ void kv_sub(uint64_t x) {  // kv K -= x
    if (KV0) return;
    const uint64_t q = x / 1000u;  // constant divisor: a multiply-high sequence, no branch
    const uint32_t rem = (uint32_t)(x - q * 1000u);
    kq -= (uint32_t)q;
    if (kr < rem) {
      kr += 1000u;
      kq--;
    }
    kr -= rem;
  }

  // ------------------------------------------------------------------ a5
  __device__ __forceinline__ void complete_sig(uint64_t sum_e2e_w, uint32_t n, uint32_t nslo) {
    if (sig(BELLMAN_SIG_TBT) || sig(BELLMAN_SIG_TTFT)) return;
    if (sig(BELLMAN_SIG_E2E)) {
      acc_sum += sum_e2e_w;
      acc_cnt += n;
    } else if (sig(BELLMAN_SIG_SLO)) {
      acc_sum += 1000ull * nslo;
      acc_cnt += n;
    }
  }

  // the words of an iteration end: B words, TBT gaps, K += B (a5)
  __device__ __forceinline__ void iteration_words() {
    words_out += B;
    if (pre()) kv_res += B;  // every decoding context grows by its word
    if (win_now) win_words_out += B;
    // TBT: the B gaps of this end; UTIL (NEXT-3): the batch size B, one sample
    const bool tbt = sig(BELLMAN_SIG_TBT), util = sig(BELLMAN_SIG_UTIL);
    acc_sum += tbt ? (uint64_t)B * iter_d + iter_align : (util ? (uint64_t)B : 0u);
    acc_cnt += tbt ? B : (util ? 1u : 0u);
    if (DBG && dbg && lane == 0) {
      bellman_second_row *w = row(ab(T));
      atomicAdd(&w->tbt_count, B);
      atomicAdd(&w->words_out, B);
      atomicAdd((unsigned long long *)&w->sum_tbt_us, (unsigned long long)B * iter_d + iter_align);
    }
    if (DBG) __syncwarp();
    if (!KV0) {
      kr += kstep_r;
      kq += kstep_q;
      if (kr >= 1000u) {
        kr -= 1000u;
        kq++;
      }
    }
  }

  // Right after an iteration start: if that iteration's end is quiet — no
  // completion, prefill end, admission, second / window / horizon boundary or
  // epoch move at or before it — apply the end now (the next trip would do
  // exactly this and nothing else) and return true.
  __device__ __forceinline__ bool quiet_end() {
    const uint32_t te = iter_end;
    // every condition evaluated, one branch
    const uint32_t lim = umin(umin(stop_static, sec_bound), umin(kRebaseAt, next_pf));
    if ((te >= lim) | (ticks - 1u == next_done) |
        ((in_sys < maxb) & !adm_blocked & ((head_t <= te) | stk_any())))
      return false;
    if (pre() && in_sys > 1u && (uint64_t)kv_res + B > cold().kv_cap) return false;  // the end preempts
    T = te;
    iteration_words();
    busy = 0;
    return true;
  }

  __device__ __forceinline__ void iteration_end(WarpHist &h) {
    const uint32_t Tn = T;
    iteration_words();
    const uint32_t it = ticks - 1u;
    if (it == next_done) {
      uint64_t e2e_l = 0;
      uint32_t kdrop = 0, nslo = 0, ndone = 0, dmin = 0xffffffffu;
      const uint64_t Ta = ab(Tn);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const bool cpl = sph[s] == PH_DEC && sdn[s] == it;
        ndone += __popc(__ballot_sync(FULL, cpl));
        if (cpl) {
          const uint64_t e = Ta - sa[s];
          e2e_l += e;
          nslo += e > slo_us;
          kdrop += sin[s] + sR[s];
          atomicAdd(&h.e2e[lat_bin_us(e)], 1u);
          sph[s] = PH_EMPTY;
        }
        if (sph[s] == PH_DEC) dmin = min(dmin, sdn[s]);
      }
      next_done = __reduce_min_sync(FULL, dmin);
      const uint64_t se = warp_sum_split(e2e_l);
      const uint32_t ns = __reduce_add_sync(FULL, nslo);
      const uint32_t kd = __reduce_add_sync(FULL, kdrop);
      kv_sub((uint64_t)kvc() * kd);
      kv_res -= kd;  // NEXT-4: completed contexts (input + R) free the KV capacity
      adm_blocked = 0;
      cadd(CT_SERVED, ndone);
      cadd(CT_SUM_E2E, se);
      cadd(CT_SLO_VIOL, ns);
      if (win_now) cadd(CT_WIN_SERVED, ndone);
      if (DBG && dbg && lane == 0) {
        atomicAdd(&row(Ta)->completions, ndone);
        atomicAdd((unsigned long long *)&row(Ta)->sum_e2e_us, (unsigned long long)se);
      }
      if (DBG) __syncwarp();
      in_sys -= ndone;
      B -= ndone;
      batch_changed();
      complete_sig(se, ndone, ns);
    }
    busy = 0;
    if (pre() && in_sys > 1u && kv_res > cold().kv_cap) preempt();
  }

  // NEXT-4 kv_policy 1 at an iteration end whose contexts exceed the capacity:
  // while more than one request is in the system, the latest admitted one
  // (decoding, decode-ready or prefilling) leaves it for the top of the
  // preempted stack (the queue front), keeping its words and realized length.
  __device__ __forceinline__ void preempt() {
    const uint32_t it = ticks - 1u, cap = cold().kv_cap;
    const uint64_t Ta = ab(T);
    bool dec = false, pfl = false;
    while (in_sys > 1u && kv_res > cap) {
      const bool in0 = sph[0] == PH_PREFILL || sph[0] == PH_READY || sph[0] == PH_DEC;
      const bool in1 = sph[1] == PH_PREFILL || sph[1] == PH_READY || sph[1] == PH_DEC;
      const uint32_t q0 = in0 ? ps->seq[lane] + 1u : 0u, q1 = in1 ? ps->seq[lane + 32u] + 1u : 0u;
      const uint32_t best = __reduce_max_sync(FULL, q0 > q1 ? q0 : q1);
      const uint32_t own = (uint32_t)__ffs(__ballot_sync(FULL, q0 == best || q1 == best)) - 1u;
      uint32_t ph = 0, ctx = 0;
      if (lane == own) {
        const uint32_t s = q1 == best ? 1u : 0u, slot = lane + 32u * s;
        ph = s ? sph[1] : sph[0];
        const uint32_t R = s ? sR[1] : sR[0], in = s ? sin[1] : sin[0];
        // words emitted so far: a decoding request's follow from its completion iteration
        const uint32_t em = ph == PH_DEC ? R - ((s ? sdn[1] : sdn[0]) - it) : ps->em[slot];
        const uint64_t lt = ph == PH_DEC ? Ta : (ph == PH_READY ? ab(s ? sp[1] : sp[0]) : ps->lt[slot]);
        PreEnt &e = ps->stk[pstk];
        e.a = s ? sa[1] : sa[0];
        e.lt = lt;
        e.enq = Ta;
        e.in = in;
        e.R = R;
        e.em = em;
        ctx = in + em;
        if (s) sph[1] = PH_EMPTY; else sph[0] = PH_EMPTY;
      }
      ph = __shfl_sync(FULL, ph, own);
      ctx = __shfl_sync(FULL, ctx, own);
      if (ph == PH_DEC) {
        B--;
        kv_sub((uint64_t)kvc() * ctx);  // its context leaves the KV term
        dec = true;
      } else if (ph == PH_READY) {
        n_ready--;
      } else {
        pfl = true;
      }
      pstk++;
      kv_res -= ctx;
      in_sys--;
      cadd(CT_PREEMPT, 1u);
    }
    if (dec) {
      uint32_t dmin = 0xffffffffu;
      if (sph[0] == PH_DEC) dmin = min(dmin, sdn[0]);
      if (sph[1] == PH_DEC) dmin = min(dmin, sdn[1]);
      next_done = __reduce_min_sync(FULL, dmin);
      batch_changed();
    }
    if (pfl) {
      uint32_t mpf = 0xffffffffu;
      if (sph[0] == PH_PREFILL) mpf = min(mpf, sp[0] - T);
      if (sph[1] == PH_PREFILL) mpf = min(mpf, sp[1] - T);
      const uint32_t m = __reduce_min_sync(FULL, mpf);
      next_pf = (m == INF32) ? INF32 : T + m;
    }
    adm_blocked = 0;
    __syncwarp();
  }

  // Prefill ends at instants in [T, lim) (first words, R=1 completions, R9).
  // Called with lim = T + 1 at an event instant, or, inside a running
  // iteration, with lim = min(iteration end, second boundary, window boundary,
  // horizon): those ends fall in one second and one window, and their only
  // effects before the iteration end — statistics of that second, slots made
  // ready or free — do not depend on their order (admission and joins happen
  // at iteration boundaries), so one pass handles them all.
  __device__ __forceinline__ void prefill_end(WarpHist &h, uint32_t lim) {
    const uint32_t Tn = T;
    uint64_t ttft_l = 0, e2e_l = 0;
    uint32_t nfirst = 0, n1 = 0, nslo = 0, nrdy = 0, kfree = 0;
    uint32_t mpf = 0xffffffffu;
    uint64_t rgap_l = 0;  // NEXT-4 preemption: TBT gaps of recompute words
    uint32_t nrec = 0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      bool f = sph[s] == PH_PREFILL && sp[s] < lim;
      if (pre() && f) {
        // a re-admitted request's recompute prefill ends: its next word, a decode
        // word whose TBT gap runs from its last word before the preemption
        const uint32_t slot = lane + 32u * s, em = ps->em[slot];
        if (em > 0u) {
          f = false;
          const uint64_t g = ab(sp[s]) - ps->lt[slot];
          rgap_l += g;
          nrec++;
          if (em + 1u == sR[s]) {
            const uint64_t e = ab(sp[s]) - sa[s];
            kfree += sin[s] + sR[s];
            e2e_l += e;
            nslo += e > slo_us;
            n1++;
            atomicAdd(&h.e2e[lat_bin_us(e)], 1u);
            sph[s] = PH_EMPTY;
          } else {
            ps->em[slot] = em + 1u;
            sph[s] = PH_READY;
            nrdy++;
          }
        } else {
          ps->em[slot] = 1u;
        }
      }
      nfirst += __popc(__ballot_sync(FULL, f));
      if (f) {
        const uint64_t tt = ab(sp[s]) - sa[s];
        const uint32_t lb = lat_bin_us(tt);
        ttft_l += tt;
        atomicAdd(&h.ttft[lb], 1u);
        if (sR[s] == 1u) {  // R9: completes at the prefill end
          kfree += sin[s] + 1u;
          e2e_l += tt;
          nslo += tt > slo_us;
          n1++;
          atomicAdd(&h.e2e[lb], 1u);
          sph[s] = PH_EMPTY;
        } else {
          sph[s] = PH_READY;
          nrdy++;
        }
      }
      if (sph[s] == PH_PREFILL) mpf = min(mpf, sp[s] - Tn);
    }
    const uint32_t m = __reduce_min_sync(FULL, mpf);
    next_pf = (m == INF32) ? INF32 : Tn + m;
    const uint64_t st = warp_sum_split(ttft_l);
    cadd(CT_SUM_TTFT, st);
    words_out += nfirst;
    if (pre()) {  // every word grows its context; recompute words are decode words (TBT)
      const uint32_t nr = __reduce_add_sync(FULL, nrec);
      kv_res += nfirst + nr;
      if (nr) {
        const uint64_t rg = warp_sum_split(rgap_l);
        words_out += nr;
        if (win_now) win_words_out += nr;
        if (sig(BELLMAN_SIG_TBT)) {
          acc_sum += rg;
          acc_cnt += nr;
        }
        if (DBG && dbg && lane == 0) {
          atomicAdd(&row(ab(Tn))->tbt_count, nr);
          atomicAdd(&row(ab(Tn))->words_out, nr);
          atomicAdd((unsigned long long *)&row(ab(Tn))->sum_tbt_us, (unsigned long long)rg);
        }
        if (DBG) __syncwarp();
      }
    }
    if (sig(BELLMAN_SIG_TTFT)) {  // NEXT-3 signal: mean TTFT of the second's first words
      acc_sum += st;
      acc_cnt += nfirst;
    }
    if (DBG && dbg && lane == 0) {
      atomicAdd(&row(ab(Tn))->first_tokens, nfirst);
      atomicAdd(&row(ab(Tn))->words_out, nfirst);
      atomicAdd((unsigned long long *)&row(ab(Tn))->sum_ttft_us, (unsigned long long)st);
    }
    if (DBG) __syncwarp();
    if (win_now) win_words_out += nfirst;
    n_ready += __reduce_add_sync(FULL, nrdy);
    const uint32_t nc = __reduce_add_sync(FULL, n1);
    if (nc) {
      kv_res -= __reduce_add_sync(FULL, kfree);
      adm_blocked = 0;
      const uint64_t se = warp_sum_split(e2e_l);
      const uint32_t ns = __reduce_add_sync(FULL, nslo);
      cadd(CT_SERVED, nc);
      cadd(CT_SUM_E2E, se);
      cadd(CT_SLO_VIOL, ns);
      if (win_now) cadd(CT_WIN_SERVED, nc);
      if (DBG && dbg && lane == 0) {
        atomicAdd(&row(ab(Tn))->completions, nc);
        atomicAdd((unsigned long long *)&row(ab(Tn))->sum_e2e_us, (unsigned long long)se);
      }
      if (DBG) __syncwarp();
      in_sys -= nc;
      complete_sig(se, nc, ns);
    }
  }

  // NEXT-4 kv_policy 1: re-admit preempted requests from the top of the stack
  // (the queue front) while a slot is free and the context input + emitted
  // fits (an empty system always admits); each prefills that context again.
  // Returns false if one stays waiting (FIFO: nothing behind it is admitted).
  __device__ __forceinline__ bool readmit(uint64_t Ta) {
    const uint32_t Tn = T;
    while (pstk) {
      if (in_sys >= maxb) return false;
      const PreEnt e = ps->stk[pstk - 1u];
      const uint32_t ctx = e.in + e.em;
      if (in_sys != 0u && (uint64_t)kv_res + ctx > cold().kv_cap) {
        adm_blocked = 1;
        return false;
      }
      pstk--;
      const uint32_t f0 = __ballot_sync(FULL, sph[0] == PH_EMPTY), f1 = __ballot_sync(FULL, sph[1] == PH_EMPTY);
      const bool s1 = f0 == 0u;
      const uint32_t sl = (uint32_t)__ffs(s1 ? f1 : f0) - 1u;
      const uint32_t pf = prefill_us(cold().pf_ns, ctx);
      if (lane == sl) {
        const uint32_t slot = sl + (s1 ? 32u : 0u);
        ps->seq[slot] = pseq;
        ps->em[slot] = e.em;
        ps->lt[slot] = e.lt;
        if (!s1) {
          sa[0] = e.a;
          sp[0] = Tn + pf;
          sR[0] = e.R;
          sin[0] = e.in;
          sph[0] = PH_PREFILL;
        } else {
          sa[1] = e.a;
          sp[1] = Tn + pf;
          sR[1] = e.R;
          sin[1] = e.in;
          sph[1] = PH_PREFILL;
        }
      }
      pseq++;
      kv_res += ctx;
      in_sys++;
      if (Tn + pf < next_pf) next_pf = Tn + pf;
      cadd(CT_WORDS_IN, ctx);
      if (win_now) cadd(CT_WIN_WORDS_IN, ctx);
      cadd(CT_SUM_QUEUE, Ta - e.enq);
      cadd(CT_RECOMP, ctx);
      if (sig(BELLMAN_SIG_INPUT)) {
        acc_sum += ctx;
        acc_cnt = 1u;
      }
      if (DBG && dbg && lane == 0) {
        atomicAdd(&row(Ta)->words_in, ctx);
        atomicAdd((unsigned long long *)&row(Ta)->sum_queue_us, (unsigned long long)(Ta - e.enq));
      }
      __syncwarp();
    }
    return true;
  }

  // ------------------------------------------------------------------ a7 (+a3)
  // FIFO admission at an admission point (R7): the queue head is admitted while
  // a slot is free and it has arrived (and, NEXT-4, its context fits the KV
  // capacity).  One request at a time, warp-uniformly: every lane reads the
  // head entry (shared-memory broadcast) and computes the same rewrite and
  // statistics, so no reduction is needed; the lane owning the first free slot
  // stores it.  Admission points almost always admit one request.
  // Precondition: in_sys < maxb and head_t <= T.
  __device__ __forceinline__ void admit(const Params &p, WarpHist &h) {
    const uint32_t Tn = T;
    const uint64_t Ta = ab(Tn);
    adm_blocked = 0;
    if (stk_any() && !readmit(Ta)) return;  // preempted requests first (the queue front)
    if (pre() && (in_sys >= maxb || head_t > Tn)) return;
    uint32_t f0 = __ballot_sync(FULL, sph[0] == PH_EMPTY), f1 = __ballot_sync(FULL, sph[1] == PH_EMPTY);
    uint32_t n = 0, n_byp = 0;
    PROF_MARK(pa_);
    do {
      const QEnt &e = cold().q[buf_h];
      const uint64_t a = e.a;
      const uint32_t inc = e.in, Uq = e.U, P = e.P, fcq = e.fcq;
      const uint32_t in = inc & 0xFFFFu, U = Uq & 0xFFFFFFu;
      // r applied to this request: the warp-uniform r unless a bypass rule holds
      // (NEXT-3; decided at refill)
      const bool byp = r > 0 && (inc >> 31);
      const uint32_t ra = byp ? 0u : r;
      // a7 rewrite and NEXT-2 similarity
      // in one block; not rewritten: U and the bin decided at refill
      uint32_t R = U, qb = Uq >> 24;
      if (ra > 0) {
        R = realized_len(p, U, P, fcq, ra);
        int32_t base;
        const int64_t num = ((int64_t)U - (int64_t)R) * 10000, den = U;
        if (num <= (int64_t)p.q_safe * den) {
          base = (int32_t)p.q_active;
        } else if (num >= (int64_t)p.q_end * den) {
          base = (int32_t)p.q_floor;
        } else {
          base = sim_decay(p.q_active, p.q_floor, (uint64_t)(num - (int64_t)p.q_safe * den),
                           (uint64_t)(p.q_end - p.q_safe) * (uint64_t)den);
        }
        int32_t sc = base + (int32_t)(fcq >> 20) - 2048;
        sc = sc < 0 ? 0 : (sc > 10000 ? 10000 : sc);
        qb = (uint32_t)sc / 50u;
      }
      if (!TBTO || XT) R = to_tokens(R, cold().tpw);  // NEXT-4: the realized output decoded as tokens (R44)
      // the product TBT loops run capacity-free profiles only
      const uint32_t kvcap = (TBTO && !XT) ? 0u : cold().kv_cap;
      if (__builtin_expect(kvcap != 0, 0)) {
        // NEXT-4: the whole context (input + realized output) must fit beside
        // the contexts in the system; an oversized head enters an empty system.
        // Preempt policy: only the current context, the input
        const uint32_t need = pre() ? in : in + R;
        if ((uint64_t)kv_res + need > kvcap && in_sys != 0u) {
          adm_blocked = 1;
          break;
        }
        kv_res += need;
      }
      n_byp += byp;
      cadd(CT_REWRITTEN, ra > 0 ? 1u : 0u);
      if (lane == 0) {  // r and similarity histograms
        if (ra > 0) atomicAdd(&h.r[ra / 10u < BELLMAN_HIST_R ? ra / 10u : BELLMAN_HIST_R - 1], 1u);
        atomicAdd(ra > 0 ? &h.qa[qb] : &h.qi[qb], 1u);
      }
      const uint32_t pf = e.pf;
      // the first free slot: lowest lane of slot row 0, then of row 1
      const bool s1 = f0 == 0u;
      const uint32_t fm = s1 ? f1 : f0;
      const uint32_t sl = (uint32_t)__ffs(fm) - 1u;
      if (s1) f1 = fm & (fm - 1u); else f0 = fm & (fm - 1u);
      // contending prefill: the prefill runs inside the next iteration (start_iteration)
      const uint32_t ph = cont() ? PH_PENDING : PH_PREFILL;
      if (pre() && lane == sl) {
        ps->seq[sl + (s1 ? 32u : 0u)] = pseq;
        ps->em[sl + (s1 ? 32u : 0u)] = 0u;
      }
      if (pre()) pseq++;
      if (lane == sl) {
        if (!s1) {
          sa[0] = a;
          sp[0] = Tn + pf;
          sR[0] = R;
          sin[0] = in;
          sph[0] = ph;
        } else {
          sa[1] = a;
          sp[1] = Tn + pf;
          sR[1] = R;
          sin[1] = in;
          sph[1] = ph;
        }
      }
      if (cont()) {  // host-validated: max_batch x max prefill < 2^30, no overflow
        pend_us += pf;
        n_pend++;
      } else if (Tn + pf < next_pf) {
        next_pf = Tn + pf;
      }
      cadd(CT_WORDS_IN, in);
      if (win_now) cadd(CT_WIN_WORDS_IN, in);
      cadd(CT_SUM_QUEUE, Ta - a);
      if (sig(BELLMAN_SIG_INPUT)) {  // NEXT-3: input words admitted in the second
        acc_sum += in;
        acc_cnt = 1u;
      }
      if (DBG && dbg && lane == 0) {
        atomicAdd(&row(Ta)->admitted, 1u);
        atomicAdd(&row(Ta)->words_in, in);
        atomicAdd((unsigned long long *)&row(Ta)->sum_queue_us, (unsigned long long)(Ta - a));
      }
      n++;
      in_sys++;
      last_j = e.j + 1u;
      if (++buf_h < buf_n) {
        head_t = rel(cold().q[buf_h].a);
      } else if (!cold().gen_done) {
        refill(p);
      } else {
        head_t = INF32;
      }
    } while (in_sys < maxb && head_t <= Tn);
    PROF_ACC(19, pa_);
    cadd(CT_ADMITTED, n);
    if (n_byp) {
      if (lane == 0) cold().bypassed += n_byp;
      __syncwarp();
    }
    if (DBG) __syncwarp();
  }


  // ------------------------------------------------------------------ NEXT-4 multi-replica (R45)
  // P:130 "the request scheduler ... picks requests from the arrival queue and
  // assigns to GPU servers": nrep engines share the FIFO queue.  A plain
  // event-at-a-time loop (no leaping): per-replica state is lane-distributed,
  // per-slot state as in the single engine; the controller, window, epoch,
  // generator, counters and epilogue are the single engine's.

  // words of the iteration ends of the replicas in endm (a5): every decoding
  // slot of such a replica emits a word; a slot reaching its R completes
  __device__ __forceinline__ void multi_end(uint32_t endm, WarpHist &h) {
    const uint32_t Tn = T;
    const uint64_t Ta = ab(Tn);
    uint64_t gap_l = 0, e2e_l = 0;
    uint32_t nw = 0, ndone = 0, nslo = 0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (sph[s] == PH_DEC && ((endm >> srep[s]) & 1u)) {
        gap_l += Tn - sp[s];  // 32-bit offsets: exact modulo 2^32
        sp[s] = Tn;
        sdn[s]++;
        nw++;
        if (sdn[s] == sR[s]) {
          const uint64_t e = Ta - sa[s];
          e2e_l += e;
          nslo += e > slo_us;
          ndone++;
          atomicAdd(&h.e2e[lat_bin_us(e)], 1u);
          sph[s] = PH_EMPTY;
        } else {
          sph[s] = PH_READY;
        }
      }
    }
    const uint32_t W = __reduce_add_sync(FULL, nw);
    const uint64_t G = warp_sum_split(gap_l);
    words_out += W;
    if (win_now) win_words_out += W;
    if (sig(BELLMAN_SIG_TBT)) {
      acc_sum += G;
      acc_cnt += W;
    } else if (sig(BELLMAN_SIG_UTIL)) {  // one sample per replica iteration end: its batch size
      acc_sum += W;
      acc_cnt += (uint32_t)__popc(endm);
    }
    if (DBG && dbg && lane == 0) {
      bellman_second_row *w = row(Ta);
      atomicAdd(&w->tbt_count, W);
      atomicAdd(&w->words_out, W);
      atomicAdd((unsigned long long *)&w->sum_tbt_us, (unsigned long long)G);
    }
    if (DBG) __syncwarp();
    const uint32_t nd = __reduce_add_sync(FULL, ndone);
    if (nd) {
      const uint64_t se = warp_sum_split(e2e_l);
      const uint32_t ns = __reduce_add_sync(FULL, nslo);
      cadd(CT_SERVED, nd);
      cadd(CT_SUM_E2E, se);
      cadd(CT_SLO_VIOL, ns);
      if (win_now) cadd(CT_WIN_SERVED, nd);
      if (DBG && dbg && lane == 0) {
        atomicAdd(&row(Ta)->completions, nd);
        atomicAdd((unsigned long long *)&row(Ta)->sum_e2e_us, (unsigned long long)se);
      }
      if (DBG) __syncwarp();
      in_sys -= nd;
      complete_sig(se, nd, ns);
    }
    if ((endm >> lane) & 1u) re = INF32;
  }

  // admission point of the replicas without a running iteration (R45): the
  // arrived queue head goes to one of them with a free slot, by the routing
  // policy; rewrite, similarity and accounting as in admit()
  __device__ __forceinline__ void multi_admit(const Params &p, WarpHist &h) {
    const uint32_t Tn = T;
    const uint64_t Ta = ab(Tn);
    const uint32_t slots_per = maxb;
    uint32_t n = 0, n_byp = 0;
    while (head_t <= Tn) {
      // requests in each replica (lane q keeps replica q's count)
      uint32_t load = 0;
      for (uint32_t q = 0; q < nrep; ++q) {
        const bool a0 = sph[0] != PH_EMPTY && sph[0] != PH_OFF && srep[0] == q;
        const bool a1 = sph[1] != PH_EMPTY && sph[1] != PH_OFF && srep[1] == q;
        const uint32_t c = (uint32_t)(__popc(__ballot_sync(FULL, a0)) + __popc(__ballot_sync(FULL, a1)));
        if (lane == q) load = c;
      }
      const bool el = lane < nrep && re == INF32 && load < slots_per;
      const uint32_t em = __ballot_sync(FULL, el);
      if (em == 0u) break;
      uint32_t q;
      if (route == BELLMAN_ROUTE_RR) {
        const uint32_t hi = em & (0xFFFFFFFFu << rrp);
        q = (uint32_t)__ffs(hi ? hi : em) - 1u;
        rrp = q + 1u == nrep ? 0u : q + 1u;
      } else {  // least loaded, ties to the lowest index
        q = __reduce_min_sync(FULL, el ? (load << 3) | lane : 0xFFFFFFFFu) & 7u;
      }
      const QEnt &e = cold().q[buf_h];
      const uint64_t a = e.a;
      const uint32_t inc = e.in, Uq = e.U, P = e.P, fcq = e.fcq;
      const uint32_t in = inc & 0xFFFFu, U = Uq & 0xFFFFFFu;
      const bool byp = r > 0 && (inc >> 31);
      const uint32_t ra = byp ? 0u : r;
      uint32_t R = U, qb = Uq >> 24;
      if (ra > 0) {
        R = realized_len(p, U, P, fcq, ra);
        int32_t base;
        const int64_t num = ((int64_t)U - (int64_t)R) * 10000, den = U;
        if (num <= (int64_t)p.q_safe * den) {
          base = (int32_t)p.q_active;
        } else if (num >= (int64_t)p.q_end * den) {
          base = (int32_t)p.q_floor;
        } else {
          base = sim_decay(p.q_active, p.q_floor, (uint64_t)(num - (int64_t)p.q_safe * den),
                           (uint64_t)(p.q_end - p.q_safe) * (uint64_t)den);
        }
        int32_t sc = base + (int32_t)(fcq >> 20) - 2048;
        sc = sc < 0 ? 0 : (sc > 10000 ? 10000 : sc);
        qb = (uint32_t)sc / 50u;
      }
      R = to_tokens(R, cold().tpw);
      n_byp += byp;
      cadd(CT_REWRITTEN, ra > 0 ? 1u : 0u);
      if (lane == 0) {
        if (ra > 0) atomicAdd(&h.r[ra / 10u < BELLMAN_HIST_R ? ra / 10u : BELLMAN_HIST_R - 1], 1u);
        atomicAdd(ra > 0 ? &h.qa[qb] : &h.qi[qb], 1u);
      }
      const uint32_t pf = e.pf;
      const uint32_t f0 = __ballot_sync(FULL, sph[0] == PH_EMPTY), f1 = __ballot_sync(FULL, sph[1] == PH_EMPTY);
      const bool s1 = f0 == 0u;
      const uint32_t sl = (uint32_t)__ffs(s1 ? f1 : f0) - 1u;
      if (lane == sl) {  // explicit rows: a runtime index would put the slot arrays in local memory
        if (!s1) {
          sa[0] = a;
          sp[0] = Tn + pf;
          sR[0] = R;
          sin[0] = in;
          sdn[0] = 1u;  // the first word (at the prefill end) is certain
          srep[0] = q;
          sph[0] = PH_PREFILL;
        } else {
          sa[1] = a;
          sp[1] = Tn + pf;
          sR[1] = R;
          sin[1] = in;
          sdn[1] = 1u;
          srep[1] = q;
          sph[1] = PH_PREFILL;
        }
      }
      if (Tn + pf < next_pf) next_pf = Tn + pf;
      cadd(CT_WORDS_IN, in);
      if (win_now) cadd(CT_WIN_WORDS_IN, in);
      cadd(CT_SUM_QUEUE, Ta - a);
      if (sig(BELLMAN_SIG_INPUT)) {
        acc_sum += in;
        acc_cnt = 1u;
      }
      if (DBG && dbg && lane == 0) {
        atomicAdd(&row(Ta)->admitted, 1u);
        atomicAdd(&row(Ta)->words_in, in);
        atomicAdd((unsigned long long *)&row(Ta)->sum_queue_us, (unsigned long long)(Ta - a));
      }
      n++;
      in_sys++;
      last_j = e.j + 1u;
      if (++buf_h < buf_n) {
        head_t = rel(cold().q[buf_h].a);
      } else if (!cold().gen_done) {
        refill(p);
      } else {
        head_t = INF32;
      }
    }
    cadd(CT_ADMITTED, n);
    if (n_byp) {
      if (lane == 0) cold().bypassed += n_byp;
      __syncwarp();
    }
    if (DBG) __syncwarp();
  }

  // every replica without a running iteration and with decode-ready slots starts
  // one with all of them: d = t0 + slope max(0, B - knee) + floor(kv K / 1000)
  __device__ __forceinline__ void multi_start() {
    const uint32_t Tn = T;
    const uint32_t idle = __ballot_sync(FULL, lane < nrep && re == INF32);
    for (uint32_t q = 0; q < nrep; ++q) {
      if (!((idle >> q) & 1u)) continue;
      uint32_t b = 0;
      uint64_t kadd = 0;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (sph[s] == PH_READY && srep[s] == q) {
          sph[s] = PH_DEC;
          b++;
          kadd += (uint64_t)sin[s] + sdn[s];
        }
      }
      const uint32_t Bq = __reduce_add_sync(FULL, b);
      if (Bq == 0u) continue;
      const uint64_t K = warp_sum_split(kadd);
      const uint64_t d = (uint64_t)t0 + (uint64_t)slope * (Bq > knee ? Bq - knee : 0u) + (uint64_t)kv * K / 1000u;
      if (lane == q) re = Tn + (uint32_t)d;
      ticks++;
    }
  }

  // Bulk-execute every replica's uneventful iteration ends: with a fixed batch,
  // a replica's k-th next iteration lasts t0 + slope max(0, B_q - knee) +
  // floor(kv (K_q + k B_q) / 1000) (closed form when kv = 0, stepped otherwise).  The next real event bounds the run: a prefill end, a
  // window / horizon / second boundary, the queue head's arrival while some
  // replica has a free slot, and per replica its first completion end (or its
  // next end if it holds decode-ready requests: they join there).  Every
  // replica's ends strictly before that instant are executed in closed form:
  // B_q words each, the TBT gaps (first gap of each slot from its last word,
  // then d_q), ticks (each end starts the next iteration), window and signal
  // accumulators; the instant itself is then an ordinary trip.
  __device__ __forceinline__ void multi_leap() {
    uint32_t stop = next_pf < stop_static ? next_pf : stop_static;
    if (sec_bound < stop) stop = sec_bound;
    if (kJumpCap < stop) stop = kJumpCap;
    uint32_t Bq = 0, mq = 0xFFFFFFFFu, load = 0, Kq = 0;
    for (uint32_t q = 0; q < nrep; ++q) {
      const bool d0 = sph[0] == PH_DEC && srep[0] == q, d1 = sph[1] == PH_DEC && srep[1] == q;
      const bool r0 = sph[0] == PH_READY && srep[0] == q, r1 = sph[1] == PH_READY && srep[1] == q;
      const bool i0 = sph[0] != PH_EMPTY && sph[0] != PH_OFF && srep[0] == q;
      const bool i1 = sph[1] != PH_EMPTY && sph[1] != PH_OFF && srep[1] == q;
      const uint32_t b = (uint32_t)(__popc(__ballot_sync(FULL, d0)) + __popc(__ballot_sync(FULL, d1)));
      const uint32_t nr = (uint32_t)(__popc(__ballot_sync(FULL, r0)) + __popc(__ballot_sync(FULL, r1)));
      const uint32_t ld = (uint32_t)(__popc(__ballot_sync(FULL, i0)) + __popc(__ballot_sync(FULL, i1)));
      uint32_t m = 0xFFFFFFFFu, k = 0;
      if (d0) {
        m = sR[0] - sdn[0];
        k += sin[0] + sdn[0];
      }
      if (d1) {
        m = min(m, sR[1] - sdn[1]);
        k += sin[1] + sdn[1];
      }
      m = __reduce_min_sync(FULL, m);
      if (kv) k = __reduce_add_sync(FULL, k);  // context words of the running iteration (<= 2^31)
      if (lane == q) {
        Bq = b;
        mq = nr ? 1u : m;
        load = ld;
        Kq = k;
      }
    }
    if (__ballot_sync(FULL, lane < nrep && load < maxb) && head_t < stop) stop = head_t;
    const bool run = lane < nrep && re != INF32 && Bq > 0u;
    const uint32_t cb = run ? t0 + slope * (Bq > knee ? Bq - knee : 0u) : 1u;
    // iteration k >= 1 after the running one: context K + k B, length cb + floor(kv (K + k B) / 1000)
    auto dur = [&](uint32_t k) -> uint32_t {
      return cb + (uint32_t)((uint64_t)kv * ((uint64_t)Kq + (uint64_t)k * Bq) / 1000u);
    };
    // this replica's completion end (its mq-th end from now) bounds everyone
    uint32_t creal = INF32;
    if (run) {
      if (kv == 0u) {
        const uint64_t c = (uint64_t)re + (uint64_t)(mq - 1u) * cb;
        creal = c < INF32 ? (uint32_t)c : INF32;
      } else {  // step through the ends before the static bound
        uint32_t e = re, k = 0;
        while (k + 1u < mq && e < stop) {
          k++;
          e += dur(k);
        }
        if (k + 1u == mq) creal = e;
      }
    }
    const uint32_t cm = __reduce_min_sync(FULL, creal);
    if (cm < stop) stop = cm;
    // the replica's ends before stop: n of them, the last at elast; next end enext
    uint32_t n = 0, elast = 0, enext = re;
    if (run && re < stop) {
      if (kv == 0u) {
        n = (stop - 1u - re) / cb + 1u;
        elast = re + (n - 1u) * cb;
        enext = elast + cb;
      } else {  // enext: the end of index n (0-based) from now
        while (n + 1u < mq && enext < stop) {
          elast = enext;
          n++;
          enext += dur(n);
        }
      }
    }
    const uint32_t nt = __reduce_add_sync(FULL, n);
    if (nt == 0u) return;
    uint64_t gap_l = 0;
    uint32_t nw = 0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const uint32_t nq = __shfl_sync(FULL, n, (int)srep[s]);
      const uint32_t el = __shfl_sync(FULL, elast, (int)srep[s]);
      if (sph[s] == PH_DEC && nq) {
        gap_l += (uint64_t)(el - sp[s]);  // the slot's gaps telescope to last end - last word (exact mod 2^32)
        sp[s] = el;
        sdn[s] += nq;
        nw += nq;
      }
    }
    const uint32_t W = __reduce_add_sync(FULL, nw);
    const uint64_t G = warp_sum_split(gap_l);
    if (run && n) re = enext;
    ticks += nt;
    words_out += W;
    if (win_now) win_words_out += W;
    if (sig(BELLMAN_SIG_TBT)) {
      acc_sum += G;
      acc_cnt += W;
    } else if (sig(BELLMAN_SIG_UTIL)) {
      acc_sum += W;
      acc_cnt += nt;
    }
    if (DBG && dbg && lane == 0) {  // every leaped end lies in the open second
      bellman_second_row *w = row(ab(sec_bound) - kUs);
      atomicAdd(&w->tbt_count, W);
      atomicAdd(&w->words_out, W);
      atomicAdd((unsigned long long *)&w->sum_tbt_us, (unsigned long long)G);
    }
    if (DBG) __syncwarp();
  }

  // the multi-replica event loop; returns true when no event remains (drained)
  __device__ __forceinline__ bool multi_loop(const Params &p, WarpHist &h) {
    for (;;) {
      uint32_t tn = __reduce_min_sync(FULL, lane < nrep ? re : INF32);
      if (next_pf < tn) tn = next_pf;
      // an arrival matters only where a replica could take it at once
      uint32_t load = 0;
      for (uint32_t q = 0; q < nrep; ++q) {
        const bool a0 = sph[0] != PH_EMPTY && sph[0] != PH_OFF && srep[0] == q;
        const bool a1 = sph[1] != PH_EMPTY && sph[1] != PH_OFF && srep[1] == q;
        const uint32_t c = (uint32_t)(__popc(__ballot_sync(FULL, a0)) + __popc(__ballot_sync(FULL, a1)));
        if (lane == q) load = c;
      }
      if (__ballot_sync(FULL, lane < nrep && re == INF32 && load < maxb) && head_t < tn) tn = head_t;
      if (tn == INF32) return true;
      if (tn > kJumpCap) tn = kJumpCap;  // a far event: jump to the cap first; advance() rebases
      if (tn >= Hr) return false;
      if (in_sys == 0) {  // idle interval [T, tn) (R18)
        cadd(CT_IDLE, tn - T);
        const uint64_t a = ab(T), b = ab(tn);
        const uint64_t lo = a > cold().w0 ? a : cold().w0, hi = b < cold().w1 ? b : cold().w1;
        if (hi > lo) cadd(CT_WIN_IDLE, hi - lo);
        dbg_idle(a, b);
      }
      advance(tn);  // rolls closed seconds into the controller (R21), window, epoch
      tn = T;
      const uint32_t endm = __ballot_sync(FULL, lane < nrep && re == tn);
      if (endm) multi_end(endm, h);
      if (next_pf == tn) prefill_end(h, tn + 1u);
      if (__ballot_sync(FULL, lane < nrep && re == INF32) != 0u) {  // some replica at an admission point
        if (head_t <= tn) multi_admit(p, h);
        multi_start();
      }
      multi_leap();
    }
  }

  // ------------------------------------------------------------------ a4/a5 leap
  // Execute in bulk the longest run of iterations whose ends are uneventful —
  // no completion (index < next_done), no prefill end, no admission (head
  // arrival still in the future or no free slot), no cold().window / horizon
  // boundary — exactly as the per-iteration path would: each emits B words
  // with TBT gap d_m = c + floor(kv (K + m B) / 1000) and grows K by B.  A
  // second boundary met inside the run is rolled in place (ingest), as the
  // per-iteration path does at that iteration end.  Called at an iteration
  // start with no joiners, so no alignment term is involved.  All arithmetic
  // is 32-bit (bounds validated on the host: d < 2^31); a leap may always be
  // cut short without changing results, so `room` is capped at 2^32 - 1.
  __device__ __forceinline__ void leap() {
    uint32_t stop = next_pf < stop_static ? next_pf : stop_static;
    if (in_sys < maxb && !adm_blocked && head_t < stop) stop = head_t;
    // a KV-blocked head may fit after an ingest changes r: stop at the second boundary
    if (adm_blocked && sec_bound < stop) stop = sec_bound;
    if (stop > kJumpCap) stop = kJumpCap;  // keeps the next iteration end inside the window
    uint32_t nmax = next_done - ticks;  // iterations ticks .. next_done-1 complete nobody
    if (pre() && in_sys > 1u) {  // NEXT-4: no leaped end may push the contexts over the capacity
      const uint32_t cap = cold().kv_cap;
      const uint32_t nk = kv_res < cap ? (cap - kv_res) / B : 0u;
      if (nk < nmax) nmax = nk;
    }
    if (nmax == 0 || stop <= T + 1u) return;
    const uint32_t cb = cbase, qs = kstep_q, rs = kstep_r;
    uint32_t q = KV0 ? 0u : kq, rr = KV0 ? 0u : kr, done = 0;
    for (;;) {
      const uint32_t lim = stop < sec_bound ? stop : sec_bound;
      const uint32_t room = lim - 1u - T;
      const uint32_t left = nmax - done;
      uint32_t n = 0, used = 0;
      if (kvc() == 0) {
        uint32_t nn;
        if (KV0) {  // umulhi(room, floor((2^32-1)/cb)) is floor(room / cb) or one less
          nn = __umulhi(room, cold().cbm_tab[B]);
          if (room - nn * cb >= cb) nn++;
        } else {
          nn = room / cb;
        }
        n = nn < left ? nn : left;
        used = n * cb;
      } else {
        if (left <= (1u << BELLMAN_LEAP_SHIFT) || (room >> BELLMAN_LEAP_SHIFT) < cb + q) {
          // short runs (dense events): one iteration at a time
          while (n < left) {
            const uint32_t d = cb + q;
            if (d > room - used) break;
            used += d;
            rr += rs;
            const uint32_t carry = rr >= 1000u;
            rr -= carry ? 1000u : 0u;
            q += qs + carry;
            n++;
          }
        } else {  // long runs: 32 iterations per step, out of line
          const uint4 v = leap_wide(lane, cb, q, rr, qs * 1000u + rs, room, left);
          n = v.x;
          used = v.y;
          q = v.z;
          rr = v.w;
        }
      }
      {  // n may be 0: every update below is then a no-op (no branch)
        const uint64_t words = (uint64_t)n * B;
        if (pre()) kv_res += (uint32_t)words;
        ticks += n;
        T += used;
        words_out += words;
        if (win_now) win_words_out += words;
        if (sig(BELLMAN_SIG_TBT)) {
          acc_sum += (uint64_t)B * used;
          acc_cnt += (uint32_t)words;
        } else if (sig(BELLMAN_SIG_UTIL)) {
          acc_sum += (uint64_t)n * B;
          acc_cnt += n;
        }
        if (DBG && dbg && lane == 0) {  // all ends of this chunk lie in the open second
          bellman_second_row *w = row(ab(sec_bound) - kUs);
          atomicAdd(&w->tbt_count, (uint32_t)words);
          atomicAdd(&w->words_out, (uint32_t)words);
          atomicAdd((unsigned long long *)&w->sum_tbt_us, (unsigned long long)B * used);
        }
        if (DBG) __syncwarp();
        done += n;
      }
      const uint32_t tnext = T + (cb + q);  // end of the next iteration
      if ((done == nmax) | (tnext >= stop) | (tnext < sec_bound)) break;
      roll_second(tnext);  // the next end opens a new second: ingest the closed one here
    }
    if (!KV0) {
      kq = q;
      kr = rr;
    }
  }

  // ------------------------------------------------------------------ a4
  __device__ __forceinline__ void start_iteration() {
    const uint32_t Tn = T;
    uint64_t align = 0;
    if (n_ready) {
      const uint32_t it0 = ticks;  // index of the new iteration
      uint32_t jn = 0xffffffffu, kadd = 0;
      uint64_t al = 0;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (sph[s] == PH_READY) {
          // words emitted when joining: 1 (the first), more for a re-admitted request
          const uint32_t ej = pre() ? ps->em[lane + 32u * s] : 1u;
          sph[s] = PH_DEC;
          sdn[s] = it0 + sR[s] - ej - 1u;  // words ej+1..R at the ends of iterations it0..it0+R-ej-1
          al += Tn - sp[s];  // 32-bit offsets: the difference is exact modulo 2^32
          kadd += sin[s] + ej;
          jn = min(jn, sdn[s]);
        }
      }
      align = warp_sum_split(al);
      const uint32_t mj = __reduce_min_sync(FULL, jn);
      if (mj < next_done) next_done = mj;
      if (!KV0) kv_add((uint64_t)kv * __reduce_add_sync(FULL, kadd));
      B += n_ready;
      n_ready = 0;
      batch_changed();
    }
    uint32_t d = cbase + (KV0 ? 0u : kq);
    if (cont()) {  // NEXT-4: cost(B) (nothing when B = 0) + the admitted requests' prefills
      d = (B ? d : 0u) + pend_us;
      if (n_pend) {
#pragma unroll
        for (int s = 0; s < 2; ++s)
          if (sph[s] == PH_PENDING) {
            sph[s] = PH_PREFILL;
            sp[s] = Tn + d;  // first word at this iteration's end, after its decode words (R7)
          }
        next_pf = Tn + d;
      }
      n_pend = 0;
      pend_us = 0;
    }
    iter_d = d;
    iter_align = align;
    iter_end = Tn + d;
    busy = 1;
    ticks++;
  }
};

// ---------------------------------------------------------------------------
__device__ void warp_percentiles(const uint32_t *hist, uint32_t nb, uint64_t n, const uint32_t *ps, uint32_t np,
                                 uint32_t *out, bool lat, uint32_t scale = 10u) {
  const uint32_t lane = lane_id();
  // odd chunk length: lane l's run starts at l * chunk, conflict-free across banks
  const uint32_t chunk = (nb + 31u) / 32u;
  uint32_t csum = 0;
#pragma unroll 1
  for (uint32_t b = 0; b < chunk; ++b)
    if (lane * chunk + b < nb) csum += hist[lane * chunk + b];
  uint32_t incl = csum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  for (uint32_t q = 0; q < np; ++q) {
    if (n == 0) {
      out[q] = BELLMAN_NONE;
      continue;
    }
    uint64_t k = ((uint64_t)ps[q] * n + 99u) / 100u;
    if (k < 1) k = 1;
    const uint32_t m = __ballot_sync(FULL, incl >= k);
    const uint32_t L = __ffs(m) - 1;
    uint32_t res = 0;
    if (lane == L) {
      uint64_t cum = incl - csum;
#pragma unroll 1
      for (uint32_t b = 0; b < chunk && lane * chunk + b < nb; ++b) {
        cum += hist[lane * chunk + b];
        if (cum >= k) {
          res = lat ? lat_edge(lane * chunk + b) : (lane * chunk + b) * scale;
          break;
        }
      }
    }
    out[q] = __shfl_sync(FULL, res, L);
  }
}

// One scenario, a1-a9.  TBTO: the scenario's signal is TBT (compile-time
// specialisation of every signal test in the event loop).  MULTI: a
// multi-replica profile (NEXT-4, R45), run by multi_loop in its own kernel.
template <bool DBG, bool TBTO, bool KV0 = false, bool MULTI = false, bool XT = false>
__device__ __forceinline__ void run_one(const Params &p, const uint64_t sid, const bellman_scenario &sc,
                                        const bellman_ctrl &cc, const uint32_t lane, WarpHist &h) {
  // ---- a1: scenario decode.  Shared-memory (Cold) fields are written by
  // lane 0 only and read after the __syncwarp below.
  Sim<DBG, TBTO, KV0, XT> S(warp_in_block());
  S.lane = lane;
  const bellman_profile pr = p.profs[sc.profile];
  const DevTrace tr = p.traces[sc.trace];
  S.E = 0;
  S.t0 = pr.t0_us;
  S.knee = pr.knee;
  S.slope = pr.slope_us;
  S.kv = pr.kv_ns_per_word;
  S.maxb = pr.max_batch;
  S.signal = cc.signal;
  S.slo_us = cc.slo_us;
  // a10: thresholds from the paired unbounded run's calibration
  uint32_t law = cc.law, t1 = cc.t1, t2 = cc.t2, flags = 0;
  if (cc.calibrated) {
    const uint32_t *cb = p.calib + 4u * p.series_slot[sc.calib_src];
    t1 = cb[0];
    t2 = cb[1];
    if (cb[2] != 0) {
      law = BELLMAN_LAW_OFF;
      flags |= BELLMAN_FLAG_DEGENERATE_CALIB;
    }
  }
  const uint32_t rslot = p.series_slot[sid];
  const uint32_t dslot = DBG ? p.dbg_slot[sid] : BELLMAN_NONE;
  S.dbg = (DBG && dslot != BELLMAN_NONE) ? p.dbg_rows + p.dbg_off[dslot] : nullptr;
  if (lane == 0) {
    Cold &z = S.cold();
    z.k0 = sc.seed_index;
    z.wid_lo = (uint32_t)sc.wid;
    z.wid_hi = (uint32_t)(sc.wid >> 32);
    z.w0 = (uint64_t)(sc.w0_us < 0 ? 0 : sc.w0_us);
    z.w1 = (uint64_t)(sc.w1_us < 0 ? 0 : sc.w1_us);
    z.H = (uint64_t)sc.horizon_us;
    z.law = law;
    z.window = cc.window;
    z.rmin = cc.r_min_bp;
    z.rmax = cc.r_max_bp;
    z.t1 = t1;
    z.t2 = t2;
    z.nrungs = cc.n_rungs;
    z.bypass_mask = cc.bypass_mask;
    z.min_words = cc.min_words_bypass;
    z.bypassed = 0;
    z.kv_cap = pr.kv_cap_words;
    z.pf_ns = pr.prefill_ns_per_word;
    z.tpw = pr.tpw_q16;
    z.hz = cc.horizon_s;
    z.wlat = cc.w_lat;
    z.wq = cc.w_q;
    z.wosc = cc.w_osc;
    z.step = cc.step_bp;
    z.rt_min = BELLMAN_NONE;
    z.phase = z.rbase = 0;
    z.cost_a = 0;
    z.flags = flags;
    z.active = z.rung = z.ring_n = z.ring_pos = 0;
    z.ringA = 0;
    z.activations = z.active_ingests = 0;
    z.first_act = z.last_deact = BELLMAN_NONE;
    z.series = rslot != BELLMAN_NONE ? p.series + p.series_off[rslot] : nullptr;
    z.series_cap = rslot != BELLMAN_NONE ? p.series_cap[rslot] : 0u;
    z.series_n = 0;
    z.dbg_ctrl = (DBG && dslot != BELLMAN_NONE) ? p.dbg_ctrl + p.dbg_off[dslot] : nullptr;
    z.dbg_cap = (DBG && dslot != BELLMAN_NONE) ? p.dbg_cap[dslot] : 0u;
    z.dbg_nctrl = 0;
    z.segs = p.segs + (tr.kind ? 0u : tr.seg_off);
    z.n_seg = tr.n_seg;
    z.replay = tr.kind;
    z.rep_off = tr.kind ? tr.seg_off : 0u;
    z.gen_seg = z.gen_j = z.gen_acc = z.gen_done = 0;
    z.gen_fresh = 1;
    z.gen_cap = tr.cap;
    z.gen_tau = 0;
  }
  if (lane < 8) {
    S.cold().rungs[lane] = cc.rungs_bp[lane];
    S.cold().ring[lane] = 0;
    S.cold().wring[lane] = 0;
  }
  if (KV0) {  // cost(B) = t0 + slope max(0, B - knee) >= 1 (host-validated t0 >= 1)
#pragma unroll 1
    for (uint32_t b = lane; b <= pr.max_batch; b += 32u)
      S.cold().cbm_tab[b] = 0xFFFFFFFFu / (pr.t0_us + pr.slope_us * (b > pr.knee ? b - pr.knee : 0u));
  }
  if (DBG && S.dbg) {  // rows are accumulated with atomics: zero this scenario's region first
    const uint32_t cap = p.dbg_cap[dslot];
    for (uint32_t i = lane; i < cap; i += 32u) S.dbg[i] = bellman_second_row{};
  }
  __syncwarp();
  S.r = law == BELLMAN_LAW_CONST ? cc.r_const_bp : 0u;
  S.acc_sum = 0;
  S.acc_cnt = 0;
  // the per-second signal feeds only the controller (MAP / STEP / NEXT-3 laws) and the recorders
  S.sec_bound = (law >= BELLMAN_LAW_MAP || rslot != BELLMAN_NONE || (DBG && S.dbg))
                    ? (uint32_t)kUs : INF32;
  S.Hr = S.rel((uint64_t)sc.horizon_us);
  S.T = 0;
  S.busy = 0;
  S.iter_end = INF32;
  S.iter_d = 0;
  S.iter_align = 0;
  S.ticks = 0;
  S.next_done = 0xffffffffu;
  S.next_pf = INF32;
  S.n_ready = S.B = S.in_sys = 0;
  S.kq = S.kr = 0;
  S.kstep_q = S.kstep_r = 0;
  S.batch_changed();
  S.update_window();
  // NEXT-4 multi-replica routing (R45): replicas x max_batch slots (generic instantiation)
  S.nrep = MULTI ? pr.replicas : 1u;
  S.route = pr.route;
  S.rrp = 0;
  S.re = INF32;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    S.sa[s] = S.sp[s] = 0;
    S.sR[s] = S.sin[s] = S.sdn[s] = 0;
    S.srep[s] = 0;
    // slots beyond max_batch (x replicas) are never free
    S.sph[s] = (lane + 32u * s < S.maxb * S.nrep) ? PH_EMPTY : PH_OFF;
  }
  S.buf_h = S.buf_n = 0;
  S.pmode = pr.prefill_mode;
  S.n_pend = S.pend_us = 0;
  S.kv_res = 0;
  S.adm_blocked = 0;
  S.kvpol = (pr.kv_policy == BELLMAN_KV_PREEMPT && pr.kv_cap_words > 0) ? 1u : 0u;
  S.pstk = S.pseq = 0;
  S.ps = p.pre + (blockIdx.x * kWarpsPerBlock + warp_in_block());
  S.last_j = 0;
#ifndef BELLMAN_AB_REGCTR
  S.ctr = 0;
#else
#pragma unroll
  for (uint32_t i = 0; i < CT_N; ++i) S.ctrs[i] = 0;
#endif
  S.words_out = S.win_words_out = 0;

  // zero the warp's histograms
  {
    uint4 *z = reinterpret_cast<uint4 *>(&h);
    for (uint32_t i = lane; i < sizeof(WarpHist) / 16u; i += 32u) z[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
  }
  S.refill(p);

  // ---- the event/tick loop (a4-a7)
#ifdef BELLMAN_PROFILE_COUNTERS
  uint32_t prof_[24] = {0};
  S.prof = prof_;
  const long long loop0_ = clock64();
#endif
  bool finished = false;
  if constexpr (MULTI) {
    finished = S.multi_loop(p, h);
  } else for (;;) {
    uint32_t tn;
    // a prefill end strictly inside the running iteration only emits first
    // words / R=1 completions (time-stamped at p): its trip does nothing
    // else; same-instant ends go after the iteration end (E1, R7).  One call
    // site per event handler keeps the loop's instruction footprint small.
    bool mid = false;
    PROF(0);
    if (S.busy) {
      // prefill ends due inside the running iteration, in the open second and
      // window: handled here, at the start of the iteration-end trip (their
      // effects are order-free until the iteration end); any left lie past a
      // second / window boundary and get their own trip
      uint32_t lim = S.iter_end < S.stop_static ? S.iter_end : S.stop_static;
      if (S.sec_bound < lim) lim = S.sec_bound;
      if (S.next_pf < lim) {
        PROF(16);
        S.prefill_end(h, lim);
      }
      mid = S.next_pf < S.iter_end;
      tn = mid ? S.next_pf : S.iter_end;
    } else {
      tn = S.next_pf;
      if (S.in_sys < S.maxb && !S.adm_blocked && S.head_t < tn) tn = S.head_t;
      if (tn == INF32) {
        finished = true;
        break;
      }
      // a far next event: jump (idle) to the cap first; advance() rebases there
      if (tn > kJumpCap) tn = kJumpCap;
    }
    if ((tn >= S.Hr) | (S.in_sys == 0)) {  // rare on a busy server: one branch for both
      if (tn >= S.Hr) break;
      if (S.in_sys == 0) {  // idle interval [T, tn) (R18)
        S.cadd(CT_IDLE, tn - S.T);
        const uint64_t a = S.ab(S.T), b = S.ab(tn);
        const uint64_t lo = a > S.cold().w0 ? a : S.cold().w0, hi = b < S.cold().w1 ? b : S.cold().w1;
        if (hi > lo) S.cadd(CT_WIN_IDLE, hi - lo);
        S.dbg_idle(a, b);
      }
    }
    PROFC(9, S.advance(tn));
    tn = S.T;  // advance() may have moved the epoch
    if (S.busy && !mid) {
      PROF(2);
      if (S.ticks - 1u == S.next_done) PROF(3);
      PROFC(10, S.iteration_end(h));
    }
    if (S.next_pf == tn) {  // always so on a mid-iteration trip
      PROF(4);
      uint32_t lim = tn + 1u;
      if (mid) {
        lim = S.iter_end < S.stop_static ? S.iter_end : S.stop_static;
        if (S.sec_bound < lim) lim = S.sec_bound;
      }
      PROFC(11, S.prefill_end(h, lim));
      if (mid) {  // a mid-iteration trip always has next_pf == tn
        PROF(1);
        continue;
      }
    }
    // the decode loop is idle here: admission point (R7), then the next iteration
    if (S.in_sys < S.maxb && !S.adm_blocked && (S.head_t <= tn || S.stk_any())) {
      PROF(5);
      PROFC(12, S.admit(p, h));
    }
    // at most two passes: a join iteration whose end is quiet is ended here
    // and followed, in the same trip, by a leap and the next start (after a
    // join B > 0, so the second pass needs no re-check)
    if (S.n_ready + S.B + S.n_pending() > 0) {
      bool join;
      do {
        join = S.n_ready + S.n_pending() != 0;
        if (!join) {
          PROF(6);
#ifdef BELLMAN_PROFILE_COUNTERS
          const uint32_t t0_ = S.ticks;
#endif
          PROFC(13, S.leap());
#ifdef BELLMAN_PROFILE_COUNTERS
          prof_[7] += S.ticks - t0_;
#endif
        } else {
          PROF(8);
        }
        PROFC(14, S.start_iteration());
      } while (join && S.quiet_end() && (PROF(17), true));
    }
  }

#ifdef BELLMAN_PROFILE_COUNTERS
  prof_[15] = (uint32_t)(clock64() - loop0_);
  if (lane == 0)
    for (int i = 0; i < 24; ++i) atomicAdd(&g_prof[i], (unsigned long long)prof_[i]);
#endif
  // ---- termination (R20)
  const uint64_t Tend = S.ab(S.T);
  const uint64_t end = (sc.mode == BELLMAN_MODE_DRAIN && finished) ? Tend : (uint64_t)sc.horizon_us;
  if (S.in_sys == 0) {
    S.cadd(CT_IDLE, end - Tend);
    const uint64_t lo = Tend > S.cold().w0 ? Tend : S.cold().w0, hi = end < S.cold().w1 ? end : S.cold().w1;
    if (hi > lo) S.cadd(CT_WIN_IDLE, hi - lo);
    S.dbg_idle(Tend, end);
  }
  if (S.sec_bound != INF32 && S.ab(S.sec_bound) <= end && S.acc_cnt) S.ingest();
  // queued at the end: accepted arrivals before `end` not admitted
#ifdef BELLMAN_PROFILE_COUNTERS
  const long long epi0_ = clock64();
#endif
  uint64_t queued = 0;
  {
    const uint32_t m = __ballot_sync(FULL, lane >= S.buf_h && lane < S.buf_n && S.cold().q[lane].a < end);
    const uint32_t nq = __popc(m);
    queued += nq;
    if (nq) S.last_j = S.cold().q[31 - __clz(m)].j + 1u;
    // the rest of the stream (no arrival at or after `end` in the buffer): counted only
    if (S.buf_h + nq == S.buf_n && !S.cold().gen_done) {
      const uint4 v = refill_buffer<DBG, true>(p, S.wid, lane, DBG ? S.dbg : nullptr, DBG ? S.cold().dbg_cap : 0u,
                                               end, S.last_j);
      queued += (uint64_t)v.x | ((uint64_t)v.y << 32);
      S.last_j = v.z;
    }
  }
  if (S.cold().series && lane == 0) p.series_n[rslot] = S.cold().series_n;
  if (DBG && S.dbg && lane == 0) {
    const uint64_t nr = end / kUs + 1u;
    p.dbg_n[2 * dslot] = (uint32_t)(nr < S.cold().dbg_cap ? nr : S.cold().dbg_cap);
    p.dbg_n[2 * dslot + 1] = S.cold().dbg_nctrl;
  }

#ifdef BELLMAN_PROFILE_COUNTERS
  const long long epi1_ = clock64();
#endif
  // ---- a9: percentiles from the histograms
  uint64_t C_[CT_N];
#pragma unroll
  for (uint32_t i = 0; i < CT_N; ++i) C_[i] = S.cget(i);
  __syncwarp();
  uint32_t pe[2], pt[2], pm[1];
  const uint32_t ps[2] = {50u, 99u};
  const uint32_t p50[1] = {50u};
  warp_percentiles(h.e2e, BELLMAN_HIST_LAT, C_[CT_SERVED], ps, 2, pe, true);
  uint64_t n_ttft = 0;
  {
    uint32_t c = 0;
    for (uint32_t b = lane; b < BELLMAN_HIST_LAT; b += 32u) c += h.ttft[b];
    n_ttft = __reduce_add_sync(FULL, c);
  }
  warp_percentiles(h.ttft, BELLMAN_HIST_LAT, n_ttft, ps, 2, pt, true);
  warp_percentiles(h.r, BELLMAN_HIST_R, C_[CT_REWRITTEN], p50, 1, pm, false);
  uint32_t pqa[1], pqi[1];  // NEXT-2 similarity medians
  warp_percentiles(h.qa, BELLMAN_HIST_Q, C_[CT_REWRITTEN], p50, 1, pqa, false, 50u);
  warp_percentiles(h.qi, BELLMAN_HIST_Q, C_[CT_ADMITTED] - C_[CT_REWRITTEN], p50, 1, pqi, false, 50u);
  // segment merge: integer atomics, order-independent
  unsigned long long *sh = p.seg_hist + (uint64_t)sc.segment * kSegWords;
  for (uint32_t b = lane; b < BELLMAN_HIST_LAT; b += 32u) {
    if (h.e2e[b]) atomicAdd(&sh[b], (unsigned long long)h.e2e[b]);
    if (h.ttft[b]) atomicAdd(&sh[BELLMAN_HIST_LAT + b], (unsigned long long)h.ttft[b]);
  }
  for (uint32_t b = lane; b < BELLMAN_HIST_R; b += 32u)
    if (h.r[b]) atomicAdd(&sh[2 * BELLMAN_HIST_LAT + b], (unsigned long long)h.r[b]);
  for (uint32_t b = lane; b < BELLMAN_HIST_Q; b += 32u) {
    if (h.qa[b]) atomicAdd(&sh[2 * BELLMAN_HIST_LAT + BELLMAN_HIST_R + b], (unsigned long long)h.qa[b]);
    if (h.qi[b]) atomicAdd(&sh[2 * BELLMAN_HIST_LAT + BELLMAN_HIST_R + BELLMAN_HIST_Q + b], (unsigned long long)h.qi[b]);
  }

#ifdef BELLMAN_PROFILE_COUNTERS
  if (lane == 0) {
    atomicAdd(&g_prof[22], (unsigned long long)(epi1_ - epi0_));
    atomicAdd(&g_prof[23], (unsigned long long)(clock64() - epi1_));
  }
#endif
  // ---- a8: summary record
  if (lane == 0) {
    bellman_scenario_stats o;
    o.scenario_id = sid;
    o.ticks = S.ticks;
    o.candidates = S.last_j;
    o.arrivals = C_[CT_ADMITTED] + queued;
    o.admitted = C_[CT_ADMITTED];
    o.served = C_[CT_SERVED];
    o.rewritten = C_[CT_REWRITTEN];
    o.words_in = C_[CT_WORDS_IN];
    o.words_out = S.words_out;
    o.idle_us = C_[CT_IDLE];
    o.end_us = end;
    o.queued_end = queued;
    o.inflight_end = S.in_sys + S.pstk;  // admitted, unfinished (preempted ones waiting too)
    o.win_served = C_[CT_WIN_SERVED];
    o.win_words_in = C_[CT_WIN_WORDS_IN];
    o.win_words_out = S.win_words_out;
    o.win_idle_us = C_[CT_WIN_IDLE];
    o.sum_queue_us = C_[CT_SUM_QUEUE];
    o.sum_ttft_us = C_[CT_SUM_TTFT];
    o.sum_e2e_us = C_[CT_SUM_E2E];
    o.slo_violations = C_[CT_SLO_VIOL];
    o.e2e_p50_ms = pe[0];
    o.e2e_p99_ms = pe[1];
    o.ttft_p50_ms = pt[0];
    o.ttft_p99_ms = pt[1];
    o.median_r_bp = pm[0];
    o.t1 = S.cold().t1;
    o.t2 = S.cold().t2;
    o.activations = S.cold().activations;
    o.first_act_s = S.cold().first_act;
    o.last_deact_s = S.cold().last_deact;
    o.active_ingests = S.cold().active_ingests;
    uint32_t fl = S.cold().flags | BELLMAN_FLAG_DONE;
    if (queued + S.in_sys + S.pstk > 0) fl |= BELLMAN_FLAG_TRUNCATED;
    o.flags = fl;
    o.segment = sc.segment;
    o.bypassed = S.cold().bypassed;
    // energy in fp64 with explicit round-to-nearest ops in a fixed order (R19)
    const double a = __dmul_rn(pr.e_in_j_per_word, (double)C_[CT_WORDS_IN]);
    const double b = __dmul_rn(pr.e_out_j_per_word, (double)S.words_out);
    const double c = __dmul_rn(pr.p_idle_w, (double)C_[CT_IDLE]);
    o.energy_j = __dadd_rn(__dadd_rn(a, b), __ddiv_rn(c, 1e6));
    const double wa = __dmul_rn(pr.e_in_j_per_word, (double)C_[CT_WIN_WORDS_IN]);
    const double wb = __dmul_rn(pr.e_out_j_per_word, (double)S.win_words_out);
    const double wc = __dmul_rn(pr.p_idle_w, (double)C_[CT_WIN_IDLE]);
    o.win_energy_j = __dadd_rn(__dadd_rn(wa, wb), __ddiv_rn(wc, 1e6));
    o.sim_active_p50 = pqa[0];
    o.sim_inactive_p50 = pqi[0];
    o.scored_active = C_[CT_REWRITTEN];
    o.scored_inactive = C_[CT_ADMITTED] - C_[CT_REWRITTEN];
    o.preemptions = (uint32_t)C_[CT_PREEMPT];
    o._pad2 = 0;
    o.recompute_words = C_[CT_RECOMP];
    p.stats[sid] = o;
  }
  if (p.n_peer) {
    // fused exchange (§8(e)): the record, just written by lane 0, goes to every
    // rank's record array over peer memory as 17 x 16-byte stores per peer,
    // spread over the lanes (lane l takes chunks l, l + 32, ... of peers x 17)
    static_assert(sizeof(bellman_scenario_stats) % 16 == 0, "record is copied in 16-byte chunks");
    constexpr uint32_t kChunks = sizeof(bellman_scenario_stats) / 16;
    __syncwarp();  // lane 0's record store precedes the other lanes' reads
    const uint4 *src = reinterpret_cast<const uint4 *>(&p.stats[sid]);
    for (uint32_t k = lane; k < p.n_peer * kChunks; k += 32u) {
      const uint32_t g = k / kChunks, c = k - g * kChunks;
      reinterpret_cast<uint4 *>(&p.peer[g][sid])[c] = src[c];
    }
    __threadfence_system();
  }
  __syncwarp();
  __syncwarp();
}

// Which kernel runs a scenario: debug-recorded (DBG) or not, and its code
// path (KIND, scenario_kind_of in bellman_lane.cuh): 0 the TBT-specialised
// single engine (TBT signal, non-blocking prefill, no KV capacity, word units,
// MAP / STEP / CONST / OFF) when it is outside K2L's bounds, 1 the generic
// single engine, 2 multi-replica; 3 / 4 run in K2L (bellman_lane.cu).
// Debug-recorded single-engine scenarios take the generic path.  Each
// scenario runs in exactly one kernel, so the product kernel <0,0> carries
// only the specialised loops.
__host__ __device__ __forceinline__ uint32_t scenario_kind(const Params &p, const bellman_scenario &sc,
                                                           const bellman_ctrl &cc) {
  return scenario_kind_of(sc, cc, p.profs[sc.profile], p.traces[sc.trace].kind, p.lane_on);
}

template <bool DBG, int KIND>
#ifndef BELLMAN_MIN_BLOCKS
#define BELLMAN_MIN_BLOCKS (16 / BELLMAN_WPB)
#endif
__global__ void __launch_bounds__(kWarpsPerBlock * 32, BELLMAN_MIN_BLOCKS) bellman_tick_kernel(const __grid_constant__ Params p) {
  const uint32_t lane = lane_pinned();
  WarpHist &h = g_hist[warp_in_block()];
  for (;;) {
    uint32_t kidx = 0;
    if (lane == 0) kidx = atomicAdd(p.counter, 1u);
    kidx = __shfl_sync(FULL, kidx, 0);
    if ((uint64_t)kidx >= p.count) break;
    const uint64_t sid = p.order ? (uint64_t)p.order[kidx] : p.first + (uint64_t)kidx * p.stride;
    const bellman_scenario sc = p.sc[sid];
    const bellman_ctrl &cc = p.ctrls[sc.ctrl];
    if ((cc.calibrated != 0) != (p.pass == 2)) continue;
    if (((sc.record & BELLMAN_RECORD_SECONDS) != 0) != DBG) continue;
    if (scenario_kind(p, sc, cc) != (uint32_t)KIND) continue;

#ifdef BELLMAN_PROFILE_COUNTERS
    if (lane == 0 && sid < (1u << 16)) g_span[2 * sid] = gtimer();
#endif
    if constexpr (KIND == 2) {
      run_one<DBG, false, false, true>(p, sid, sc, cc, lane, h);
    } else if constexpr (KIND == 1) {
      const bellman_profile &pf = p.profs[sc.profile];
      if (!DBG && cc.signal == BELLMAN_SIG_TBT && pf.prefill_mode == BELLMAN_PREFILL_NONBLOCKING &&
          (pf.kv_policy != BELLMAN_KV_PREEMPT || pf.kv_cap_words == 0)) {
        // TBT scenarios with token units, a NEXT-3 law or a KV-reserve capacity:
        // the TBT-specialised loop with those features at run time (XT)
        if (pf.kv_ns_per_word == 0)
          run_one<false, true, true, false, true>(p, sid, sc, cc, lane, h);
        else
          run_one<false, true, false, false, true>(p, sid, sc, cc, lane, h);
      } else {
        run_one<DBG, false>(p, sid, sc, cc, lane, h);
      }
    } else {
      // TBT-only loop (one replica, no KV capacity, words: no token conversion
      // at admission; MAP / STEP / CONST / OFF: no NEXT-3 law call site),
      // specialised once more on a KV-free cost law (kv = 0)
      if (p.profs[sc.profile].kv_ns_per_word == 0)
        run_one<false, true, true>(p, sid, sc, cc, lane, h);
      else
        run_one<false, true, false>(p, sid, sc, cc, lane, h);
    }
#ifdef BELLMAN_PROFILE_COUNTERS
    if (lane == 0 && sid < (1u << 16)) g_span[2 * sid + 1] = gtimer();
#endif
  }
}

// ---------------------------------------------------------------------------
// K5: per recorded slot, nearest-rank p50 / p75 of its series
// by bisection on the value: the k-th smallest is the least v with
// #{x <= v} >= k.  One warp per slot.
__device__ uint32_t warp_kth(const uint32_t *x, uint32_t n, uint32_t k) {
  uint32_t lo = 0, hi = 0xffffffffu;
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    uint32_t c = 0;
    for (uint32_t i = lane_id(); i < n; i += 32u) c += x[i] <= mid;
    c = __reduce_add_sync(FULL, c);
    if (c >= k) hi = mid; else lo = mid + 1u;
  }
  return lo;
}

__global__ void bellman_calibrate_kernel(const Params p, uint32_t n_slots) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_slots) return;
  const uint32_t n = min(p.series_n[w], p.series_cap[w]);
  const uint32_t *x = p.series + p.series_off[w];
  uint32_t t1 = 0, t2 = 0, st = 1;
  if (n >= 4) {
    t1 = warp_kth(x, n, (50u * n + 99u) / 100u);
    t2 = warp_kth(x, n, (75u * n + 99u) / 100u);
    st = t1 == t2 ? 2u : 0u;
  }
  if (lane_id() == 0) {
    p.calib[4 * w + 0] = t1;
    p.calib[4 * w + 1] = t2;
    p.calib[4 * w + 2] = st;
    p.calib[4 * w + 3] = n;
  }
}

}  // namespace bellman

#ifdef BELLMAN_PROFILE_COUNTERS
extern "C" int bellman_debug_prof(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, g_prof, sizeof(unsigned long long) * 24);
}
extern "C" int bellman_debug_span(unsigned long long *out, unsigned n) {
  return (int)cudaMemcpyFromSymbol(out, g_span, sizeof(unsigned long long) * 2 * (n < (1u << 16) ? n : (1u << 16)));
}
#endif

int bellman_tick_grid(int device) {
  static int cached[64] = {0};  // per device: the answer does not change within a process
  if (device >= 0 && device < 64 && cached[device] > 0) return cached[device];
  int sms = 0, per_sm = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bellman::bellman_tick_kernel<false, 0>,
                                                    bellman::kWarpsPerBlock * 32, 0) != cudaSuccess)
    return -1;
  const int g = sms * (per_sm > 0 ? per_sm : 1);
  if (device >= 0 && device < 64) cached[device] = g;
  return g;
}

cudaError_t bellman_launch_tick(const bellman::Params &p, int grid, bool dbg, int kind, cudaStream_t stream) {
  const int bs = bellman::kWarpsPerBlock * 32;
  if (dbg && kind == 2) bellman::bellman_tick_kernel<true, 2><<<grid, bs, 0, stream>>>(p);
  else if (dbg) bellman::bellman_tick_kernel<true, 1><<<grid, bs, 0, stream>>>(p);
  else if (kind == 2) bellman::bellman_tick_kernel<false, 2><<<grid, bs, 0, stream>>>(p);
  else if (kind == 1) bellman::bellman_tick_kernel<false, 1><<<grid, bs, 0, stream>>>(p);
  else bellman::bellman_tick_kernel<false, 0><<<grid, bs, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t bellman_launch_calibrate(const bellman::Params &p, uint32_t n_slots, cudaStream_t stream) {
  const uint32_t threads = 128, warps = threads / 32;
  const uint32_t blocks = (n_slots + warps - 1) / warps;
  if (blocks == 0) return cudaSuccess;
  bellman::bellman_calibrate_kernel<<<blocks, threads, 0, stream>>>(p, n_slots);
  return cudaGetLastError();
}

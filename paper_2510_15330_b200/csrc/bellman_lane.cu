// bellman_lane.cu — K2L, the lane-per-scenario product kernel (round 2).
//
// SURVEY §8(d) bounds the method twice: R_issue (one warp per scenario, every
// scalar operation of the event loop takes a whole warp issue slot) and R_lane
// (the integer lanes themselves, "design-independent; shows what
// warp-per-scenario leaves on the table").  K2 (bellman_kernels.cu) runs one
// scenario per warp and reaches ~0.6 of R_issue, i.e. ~2 % of R_lane.  K2L runs
// one scenario per LANE: each thread owns a whole scenario — clock, batch,
// controller, generator, counters in registers; its <= 64 request slots in
// shared memory — and the 32 scenarios of a warp advance through the same
// event loop, each lane handling its own next event (divergent handlers are
// serialised by the SIMT stack, so a warp pays the union of the handlers its
// lanes need per trip, not their sum).
//
// Scope (scenario_kind 3 / 4): the TBT-specialised single-engine
// scenarios of the product kernel (TBT signal, non-blocking prefill, no KV
// capacity, word units, MAP / STEP / CONST / OFF; every benchmark
// configuration) on a Poisson trace with horizon < 2^31 µs, in runs of at
// least 65,536 scenarios; kind 3 is the KV-free cost law (kv = 0), kind 4 has
// the KV term.  Everything else stays on K2.  Semantics are K2's (and the
// oracle's) step for step; only the data layout and the schedule differ:
//  * all instants are absolute 32-bit µs (horizon < 2^31, iteration and
//    prefill durations < 2^31: no epoch, no rebase);
//  * request slots: shared memory [field][slot][lane] (u32; the bank is the
//    lane whatever the slot, so divergent slot indices never conflict): prefill
//    end (then the completion iteration), arrival, realized length R (+ input
//    words with a KV term); slot phases as u64 bit masks in registers;
//  * decoding requests: a 4-ary min-heap per lane of one-byte slot indices
//    (a node's four children are one 32-bit word; byte stores, still one bank
//    per lane) keyed by the completion iteration held in the slot's
//    prefill-end word; every position past the heap's size holds a sentinel
//    slot whose key is kInf (no bounds tests), and a pop returns the new least
//    key: 27.5 KB per warp, 8 warps (one CTA) per SM;
//  * the kv-free leap divides by the iteration cost through a per-profile
//    reciprocal table (exact: bellman_internal.cuh);
//  * one prefill-end site per trip, before the clock advance (a second one
//    only for ends at or past a window / horizon boundary);
//  * the FIFO queue ahead of admission: a head / next register window and a
//    32-entry ring per lane in global memory, refilled 32 candidates at a time
//    by the whole warp (coop_refill: K2's lane-parallel generator, for one lane
//    at a time; same Philox counters, thinning and crossing rule);
//  * the persistent loop starts every trip with a warp vote (reconvergence),
//    and closed seconds are ingested at one site per trip;
//  * histograms (a9): per thread in global memory (L2-resident), bumped with
//    fire-and-forget PTX `red` (atomicAdd compiles to ATOMG with a destination
//    register); a bit mask of the 32-bin groups each scenario touched bounds
//    the epilogue's percentile walk, segment merge and re-zeroing.
//
// The per-scenario code is __host__ __device__: a development build
// (-DBELLMAN_LANECHECK, bellman_host.cu) runs it on the CPU to compare with
// the oracle before any GPU time is spent.  The product path is the kernel.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "bellman_internal.cuh"
#include "bellman_lane.cuh"

namespace bellman {
namespace lane {

#define LHD __host__ __device__ __forceinline__

constexpr uint32_t kInf = 0xffffffffu, kFar = 0xfffffffeu, FULL_MASK = 0xffffffffu;
constexpr uint32_t kNone = BELLMAN_NONE;

LHD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}
LHD uint32_t clz32(uint32_t x) {
#ifdef __CUDA_ARCH__
  return (uint32_t)__clz(x);
#else
  return x ? (uint32_t)__builtin_clz(x) : 32u;
#endif
}
LHD uint32_t ffs64(uint64_t x) {  // 1 + index of the lowest set bit, 0 if none
#if defined(__CUDA_ARCH__)  // (two 32-bit __ffs with a select measured 7 % slower on C5, r02x)
  return (uint32_t)__ffsll((long long)x);
#else
  return (uint32_t)__builtin_ffsll((long long)x);
#endif
}
LHD uint32_t ffs32(uint32_t x) {
#ifdef __CUDA_ARCH__
  return (uint32_t)__ffs((int)x);
#else
  return (uint32_t)__builtin_ffs((int)x);
#endif
}
LHD void red_add(uint32_t *a, uint32_t v) {  // fire-and-forget on the GPU (result unused: RED)
#if defined(__CUDA_ARCH__) && defined(BELLMAN_AB_RED_EVICT_FIRST)
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("red.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
#elif defined(__CUDA_ARCH__) && !defined(BELLMAN_AB_ATOMG)
  // explicit RED: ptxas emits ATOMG (with a destination register, whose
  // scoreboard then stalls the next writer of that register) for atomicAdd
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
#elif defined(__CUDA_ARCH__)
  atomicAdd(a, v);
#else
  *a += v;
#endif
}
LHD void seg_add(unsigned long long *a, unsigned long long v) {
#ifdef __CUDA_ARCH__
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
#else
  *a += v;
#endif
}
template <class T>
LHD T ldg(const T *x) {
#ifdef __CUDA_ARCH__
  return __ldg(x);
#else
  return *x;
#endif
}

struct U4 {
  uint32_t x, y, z, w;
};

// Philox4x32-10 (Salmon et al. SC'11), counter (c0..c3), key (k0, k1).  Inline
// (A/B on full C5, with the leap's integer division: 638 ms inline, 650 ms out
// of line; code-layout effects in this kernel are not additive).
#ifdef BELLMAN_AB_PHILOX_CALL
__host__ __device__ __noinline__
#else
LHD
#endif
U4 philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                                           uint32_t c3) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c0 = n0;
    c1 = (uint32_t)p1;
    c2 = n2;
    c3 = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return U4{c0, c1, c2, c3};
}

// -ln(U), U = (2u+1)/2^33, in Q32 (reading R33): log2 by table + interpolation.
// neglog_split gives the normalised mantissa bits x of v = 2u + 1 (table index
// x >> 20) and its exponent e; neglog_q32 interpolates with the entry t.
LHD uint32_t neglog_split(uint32_t u, uint32_t &e) {
  if (u >= 0x80000000u) {
    e = 32;
    return 2u * u + 1u;
  }
  const uint32_t v = 2u * u + 1u;
  e = 31u - clz32(v);
  return (uint32_t)(((uint64_t)(v - (1u << e))) << (32u - e));
}
LHD uint32_t neglog_index(uint32_t u) {
  uint32_t e;
  return neglog_split(u, e) >> 20;
}
LHD uint64_t neglog_q32(uint32_t u, uint2 t) {
  uint32_t e;
  const uint32_t x = neglog_split(u, e);
  const uint64_t f = x & 0xFFFFFu;
  const uint64_t log2v = ((uint64_t)e << 32) + t.x + (((uint64_t)t.y * f) >> 20);
  const uint64_t neg = (33ull << 32) - log2v;
  const uint64_t lo = neg * 2977044472ull, hi = mulhi64(neg, 2977044472ull);  // round(ln 2 * 2^32)
  return (hi << 32) | (lo >> 32);
}

// latency bin of a value in µs (a9): exact ms below 32, then 32 per octave.
// Instants are < 2^32 here, so every latency fits 32 bits.
// Branch-free (both values, then a select; A/B on full C5: 472.8 -> 465.6 ms
// against an early return, r02zc): for ms >= 32, ms | 32 has ms's top bit.
LHD uint32_t lat_bin(uint32_t us) {
  const uint32_t ms = us / 1000u;
  const uint32_t e = 31u - clz32(ms | 32u);
  const uint32_t big = 32u * (e - 4u) + ((ms >> (e - 5u)) & 31u);
  return ms < 32u ? ms : big;
}
LHD uint32_t lat_edge(uint32_t b) {
  if (b < 32) return b;
  const uint32_t e = b / 32u + 4u, s = b % 32u;
  return (32u + s) << (e - 5u);
}
LHD uint64_t div_u64(uint64_t a, uint64_t b) {
  if (((a | b) >> 32) == 0) return (uint32_t)a / (uint32_t)b;
  return a / b;
}
// NEXT-2 similarity decay: q_active - floor((q_active - q_floor) X / D)
// inline: A/B on full C5 with the one-site prefill loop, 494.3 ms vs 502.6 ms
// out of line (BELLMAN_AB_DECAY_CALL)
#ifndef BELLMAN_AB_DECAY_CALL
LHD
#else
__host__ __device__ __noinline__
#endif
int32_t sim_decay(uint32_t q_active, uint32_t q_floor, uint64_t X, uint64_t D) {
  const uint64_t aX = (uint64_t)(q_active - q_floor) * X;
#ifdef __CUDA_ARCH__
  uint32_t q = (uint32_t)__fmul_rz((float)aX, __frcp_rn((float)D));  // estimate, then an exact fix-up
  while (q && (uint64_t)q * D > aX) q--;
  while ((uint64_t)(q + 1u) * D <= aX) q++;
#else
  const uint32_t q = (uint32_t)(aX / D);
#endif
  return (int32_t)q_active - (int32_t)q;
}

// a7 rewrite (R11), the 128-bit path (out of line)
__host__ __device__ __noinline__ uint32_t rewrite_wide(int64_t poly0, int64_t poly1, int64_t poly2, uint32_t N,
                                                       uint32_t fcq) {
  const int32_t fc = (int32_t)(fcq & 0xFFFFFu);
  const __int128 poly = (__int128)poly0 + (__int128)poly1 * N + (__int128)poly2 * N * N;
  __int128 x = (poly * fc + ((__int128)1 << 31)) >> 32;
  if (x < 1) x = 1;
  if (x > (1 << 24)) x = 1 << 24;
  return (uint32_t)x;
}

LHD uint32_t realized_len(const Params &p, uint32_t P, uint32_t fcq, uint32_t ra) {
  uint32_t N = (P * (10000u - ra) + 5000u) / 10000u;  // P < 2^17
  if (N < 1u) N = 1u;
  if (p.poly_fast) {
    const int64_t n = N;
    const int64_t poly = p.poly0 + p.poly1 * n + p.poly2 * n * n;
    int64_t x = (poly * (int32_t)(fcq & 0xFFFFFu) + (1ll << 31)) >> 32;
    x = x < 1 ? 1 : (x > (1 << 24) ? (1 << 24) : x);
    return (uint32_t)x;
  }
  return rewrite_wide(p.poly0, p.poly1, p.poly2, N, fcq);
}

// slot fields: word (f, s) of this lane at sm[(f * 64 + s) * 32]; the heap follows the fields
#ifdef BELLMAN_AB_NOSENT
constexpr uint32_t F_PF = 0, F_ARR = 1, F_R = 2, F_IN = 3;
#endif

template <bool KV0>
struct Lane {
  static constexpr uint32_t kF = kFields<KV0>;
#ifndef BELLMAN_AB_NOSENT
  // the prefill-end / completion-key field last: its slot 64 is the sentinel
  // word (kInf) that precedes the heap
  static constexpr uint32_t F_ARR = 0, F_R = 1, F_IN = 2, F_PF = kF - 1u, kHeapW = kF * 64u + 1u;
  static constexpr uint32_t kSent = 64;  // sentinel slot index: key(kSent) = kInf
#else
  static constexpr uint32_t kHeapW = kF * 64u;
#endif
  // ---- storage
  uint32_t *sm;    // this lane's word 0 of its warp's slot region (stride 32 words)
  uint32_t *hist;  // this thread's histograms (global, kLaneHistWords)
  uint64_t sid;
  // ---- profile / scenario constants
  uint32_t t0, knee, slope, kv, maxb, slo_us, pf_ns;
  uint32_t H;          // horizon (absolute µs, < 2^31)
  uint32_t w0, w1;     // window [w0, w1), clamped to 32 bits
  uint32_t drain;
  // ---- controller (a6)
  uint32_t law, window, t1, t2, rmin, rmax, nrungs;
  uint32_t rk[4];  // the ladder, two 16-bit rungs per word (rungs <= 5000 bp)
  uint32_t r;
  uint64_t ringA;
  uint32_t ring_n, ring_pos, rung, active, activations, active_ingests, first_act, last_deact;
  // the window's samples live in the thread's global scratch (hist + kHistRing);
  // ev_next is the sample the next full-window ingest evicts, loaded one ingest ahead
  uint32_t ev_next;
  uint32_t *series;
  uint32_t series_n, series_cap, rslot;
  // ---- clock and serving state (a4, a5, a7)
  uint32_t T, busy, iter_end, iter_d, ticks, next_done, next_pf;
  uint64_t iter_align;
  uint32_t n_ready, B, in_sys, cbase, kq, kr, kstep_q, kstep_r;
  const uint64_t *cm;  // kv = 0: this profile's leap reciprocals ceil(2^63 / c(B)), B = 0 .. 64
  uint64_t cmag;       // kv = 0: cm[B] (loaded at each batch change, used by the next leap)
  uint32_t win_now, win_next, stop_static, sec_bound;
  uint64_t acc_sum;
  uint32_t acc_cnt;
  uint64_t pa_sum, pb_sum;  // closed seconds waiting for ingest_pending (npend <= 2)
  uint32_t pa_cnt, pb_cnt, pa_sec, pb_sec, npend;
  uint64_t free_m, pf_m, rdy_m;
  uint64_t rdy_sum;   // sum of the decode-ready slots' prefill ends (their join alignment)
  uint32_t rdy_kadd;  // sum of their (input + 1) context words (KV term)
  uint32_t nheap;
  // ---- the FIFO queue ahead of admission (a2, a3): the head and the next
  // accepted arrival in registers, the ones after them in this thread's FIFO
  // in global memory (fifo, a 32-entry ring of 24-byte entries: frd, fcnt),
  // filled 32 candidates at a time by the whole warp (coop_refill) when it is
  // empty.  An entry: arrival (clamped to 32 bits), input | class << 16, U, P,
  // F_comp | similarity noise, index j.
  uint32_t head_t, h_in, h_U, h_P, h_fcq, h_j;  // head_t = INF: no head
  uint32_t n_t, n_in, n_U, n_P, n_fcq, n_j, n_ok;
  uint2 *fifo;  // entry k: fifo[3k .. 3k+2]
  uint32_t frd, fcnt;
  uint32_t gen_seg, gen_j, gen_acc, gen_done, gen_fresh, gen_cap, n_seg, seg_off;
  uint64_t gen_tau;
  uint32_t k0, wid_lo, wid_hi, bypass_mask, min_words;
  // ---- accounting (a8)
  uint64_t c_admitted, c_served, c_rewritten, c_slo, c_win_served, c_words_in, c_idle, c_win_words_in,
      c_win_idle, c_sum_queue, c_sum_ttft, c_sum_e2e, words_out, win_words_out, n_ttft;
  uint32_t last_j, bypassed, flags, finished;
  uint32_t segment;                       // the scenario's segment (a9 merge)
  uint32_t fin_end;                       // end_us of the finished scenario (R20)
  uint64_t fin_queued;                    // queued at the end
  uint32_t r_e50, r_e99, r_f50, r_f99, r_rm, r_qa, r_qi;  // percentile bins (kNone: empty)
  // touched 32-bin groups of each histogram (epilogue scan bound)
  uint32_t hm_e2e, hm_ttft, hm_r, hm_q;  // hm_q: qa groups in bits 0-7, qi in bits 8-15

  LHD uint32_t &SL(uint32_t f, uint32_t s) const { return sm[(f * 64u + s) * 32u]; }
  // decode heap: position i is byte i & 3 of heap word i >> 2 (slot indices,
  // byte loads / stores; the bank is still the lane); the key of slot s is its
  // completion iteration, kept in the slot's (by then unused) prefill-end word
  LHD uint8_t &HB(uint32_t i) const { return reinterpret_cast<uint8_t *>(&sm[(kHeapW + (i >> 2)) * 32u])[i & 3u]; }
  LHD uint32_t key(uint32_t slot) const { return SL(F_PF, slot); }
  static constexpr uint32_t kHeapRoot = 3;  // the 4-ary heap's node 0 is byte 3

  LHD void hist_add(uint32_t off, uint32_t b, uint32_t &mask, uint32_t shift = 0) {
    red_add(&hist[off + b], 1u);
    mask |= 1u << ((b >> 5) + shift);
  }

  // ------------------------------------------------------------------ decode heap
  // 4-ary min-heap of the decoding slots by completion iteration (ties in any
  // order: completions of one iteration are popped together).  Node i is heap
  // byte i + 3, so the children 4i+1 .. 4i+4 of node i are the four bytes of
  // heap word i + 1: one load per level, then four independent key loads
  // (depth <= 3 for 64 slots).
  LHD uint32_t HW(uint32_t w) const { return sm[(kHeapW + w) * 32u]; }
  LHD void heap_push(uint32_t slot, uint32_t k) {
    uint32_t i = nheap++;
    while (i > 0) {
      const uint32_t par = (i - 1u) >> 2;
      const uint32_t ps = HB(par + 3u);
      if (key(ps) <= k) break;
      HB(i + 3u) = (uint8_t)ps;
      i = par;
    }
    HB(i + 3u) = (uint8_t)slot;
  }
#ifndef BELLMAN_AB_NOSENT
  // Every position >= nheap (up to position 84, the last child of a depth-2
  // node) holds the sentinel slot, whose key is kInf: no bounds tests in the
  // sift-down, which stops when the moved key is <= the least child (kInf
  // included) or at depth 3.
  // Returns the popped slot; rk = the new root's key (kInf: empty), which the
  // first level's comparison already decides (the moved key or the least child).
  LHD uint32_t heap_pop(uint32_t &rk) {
    const uint32_t top = HB(3u);
    const uint32_t n = --nheap;
    const uint32_t last = HB(n + 3u);
    HB(n + 3u) = (uint8_t)kSent;
    const uint32_t lk = key(last);
    uint32_t i = 0;
    rk = kInf;
    if (n) {
#pragma unroll
      for (uint32_t lvl = 0; lvl < 3u; ++lvl) {  // depth <= 3: at most three levels down
        const uint32_t c0 = 4u * i + 1u;
        const uint32_t w = HW(i + 1u);  // the slot indices of children c0 .. c0 + 3
        uint32_t bs = w & 0xFFu, bk = key(bs), bc = c0;
#pragma unroll
        for (uint32_t q = 1; q < 4; ++q) {
          const uint32_t sq = (w >> (8u * q)) & 0xFFu, kq2 = key(sq);
          if (kq2 < bk) {
            bk = kq2;
            bs = sq;
            bc = c0 + q;
          }
        }
#ifndef BELLMAN_AB_NOKEYTRACK
        if (lvl == 0) rk = lk <= bk ? lk : bk;
#endif
        if (lk <= bk) break;
        HB(i + 3u) = (uint8_t)bs;
        i = bc;
      }
      HB(i + 3u) = (uint8_t)last;
    }
#ifdef BELLMAN_AB_NOKEYTRACK
    rk = key(HB(kHeapRoot));
#endif
    return top;
  }
  LHD void heap_reset() {  // all positions sentinel, the sentinel key kInf
    sm[(kHeapW - 1u) * 32u] = kInf;
#pragma unroll
    for (uint32_t w = 0; w < 22u; ++w) sm[(kHeapW + w) * 32u] = kSent * 0x01010101u;
  }
#else
  LHD uint32_t heap_pop(uint32_t &rk) {
    const uint32_t top = HB(3u);
    const uint32_t last = HB(--nheap + 3u);
    const uint32_t n = nheap;
    if (n) {
      const uint32_t lk = key(last);
      uint32_t i = 0;
      for (;;) {
        const uint32_t c0 = 4u * i + 1u;
        if (c0 >= n) break;
        const uint32_t w = HW(i + 1u);  // the slot indices of children c0 .. c0 + 3
        uint32_t bs = w & 0xFFu, bk = key(bs), bc = c0;
#pragma unroll
        for (uint32_t q = 1; q < 4; ++q) {
          if (c0 + q < n) {
            const uint32_t sq = (w >> (8u * q)) & 0xFFu, kq2 = key(sq);
            if (kq2 < bk) {
              bk = kq2;
              bs = sq;
              bc = c0 + q;
            }
          }
        }
        if (lk <= bk) break;
        HB(i + 3u) = (uint8_t)bs;
        i = bc;
      }
      HB(i + 3u) = (uint8_t)last;
    }
    rk = nheap ? key(HB(kHeapRoot)) : kInf;
    return top;
  }

  LHD void heap_reset() {}
#endif

  // ------------------------------------------------------------------ helpers
  LHD uint32_t rung_at(uint32_t i) const {
    uint32_t v = 0;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) v = (i == k) ? (rk[k >> 1] >> (16u * (k & 1u))) & 0xFFFFu : v;
    return v;
  }
  LHD void update_window() {
    win_now = (T >= w0) & (T < w1);
    win_next = T < w0 ? w0 : (T < w1 ? w1 : kInf);
    stop_static = H < win_next ? H : win_next;
  }
  LHD void batch_changed() {
    cbase = t0 + slope * (B > knee ? B - knee : 0u);
#ifndef BELLMAN_AB_LEAPDIV
    if (KV0) cmag = ldg(cm + B);
#endif
    if (KV0) return;
    const uint32_t ks = kv * B;
    kstep_q = ks / 1000u;
    kstep_r = ks - kstep_q * 1000u;
  }
  LHD void kv_add(uint64_t x) {
    if (KV0) return;
    const uint64_t q = x / 1000u;
    kr += (uint32_t)(x - q * 1000u);
    kq += (uint32_t)q;
    if (kr >= 1000u) {
      kr -= 1000u;
      kq++;
    }
  }
  LHD void kv_sub(uint64_t x) {
    if (KV0) return;
    const uint64_t q = x / 1000u;
    const uint32_t rem = (uint32_t)(x - q * 1000u);
    kq -= (uint32_t)q;
    if (kr < rem) {
      kr += 1000u;
      kq--;
    }
    kr -= rem;
  }
  // idle interval [a, b) (R18)
  LHD void idle(uint32_t a, uint32_t b) {
    c_idle += b - a;
    const uint32_t lo = a > w0 ? a : w0, hi = b < w1 ? b : w1;
    if (hi > lo) c_win_idle += hi - lo;
  }

  // ------------------------------------------------------------------ a6
  // one controller ingest of the closed second ending at `sec` with
  // accumulator (sum, cnt) (R3-R5, R12, R21, R38)
  LHD void ingest(uint64_t sum, uint32_t cnt, uint32_t sec) {
    // the sample: floor(sum / cnt) truncated to 32 bits
    // (an fp32 estimate with an exact fix-up, as for the MAP quotient below,
    // measured 5 % slower here: 496.4 vs 472.7 ms on C5, r02z)
    const uint32_t x = (uint32_t)div_u64(sum, cnt);
    if (series) {
      if (series_n < series_cap) series[series_n] = x;
      else flags |= BELLMAN_FLAG_SERIES_OVERFLOW;
      series_n++;
    }
    if (law != BELLMAN_LAW_MAP && law != BELLMAN_LAW_STEP) return;
    const uint32_t was = active;
    uint32_t k = ring_n;
    uint64_t A = ringA;
    if (k < window) {
      k++;
      A += x;
    } else {
      A = A + x - ev_next;
    }
    const uint32_t act = A >= (uint64_t)k * t1 ? 1u : 0u;  // non-strict (R38)
    uint32_t nr = 0;
    if (act) {
      if (law == BELLMAN_LAW_MAP) {
        // r_min + floor((r_max - r_min)(A - k t1) / (k (t2 - t1))), capped at r_max
        const uint64_t ex = A - (uint64_t)k * t1, den = (uint64_t)k * (t2 - t1);
        if (ex >= den) {
          nr = rmax;  // the quotient is >= r_max - r_min
        } else {  // quotient < r_max - r_min <= 5000; den < 2^35
#if defined(__CUDA_ARCH__)
          // fp32 estimate (off by at most one: q < 5000), then the exact fix-up
          // (A/B on full C5: 478.4 -> 474.1 ms against the integer division, r02y)
          const uint64_t num = (uint64_t)(rmax - rmin) * ex;
          uint32_t q = (uint32_t)__fmul_rz((float)num, __frcp_rn((float)den));
          while (q && (uint64_t)q * den > num) q--;
          while ((uint64_t)(q + 1u) * den <= num) q++;
          nr = rmin + q;
#else
          nr = rmin + (uint32_t)div_u64((uint64_t)(rmax - rmin) * ex, den);
#endif
          if (nr > rmax) nr = rmax;
        }
        if (nrungs) {  // largest rung <= r (R5)
          uint32_t best = rk[0] & 0xFFFFu;
#pragma unroll
          for (uint32_t i = 1; i < 8; ++i) {
            const uint32_t g = (rk[i >> 1] >> (16u * (i & 1u))) & 0xFFFFu;
            if (i < nrungs && g <= nr) best = g;
          }
          nr = best;
        }
      } else {  // STEP: rung 0 on activation, one rung up per ingest while active
        rung = was ? (rung + 1u < nrungs ? rung + 1u : rung) : 0u;
        nr = rung_at(rung);
      }
    }
    hist[kHistRing + ring_pos] = x;
    ring_pos = ring_pos + 1u == window ? 0u : ring_pos + 1u;
    ev_next = hist[kHistRing + ring_pos];  // read after the store (window 1: the same word)
    ring_n = k;
    ringA = A;
    active = act;
    activations += (act && !was) ? 1u : 0u;
    active_ingests += act;
    if (act != was) {  // the log is kept by second index (R21)
      const uint32_t second = sec / 1000000u - 1u;
      if (act) {
        if (first_act == kNone) first_act = second;
      } else {
        last_deact = second;
      }
    }
    r = nr;
  }

  // Closed seconds wait in a two-entry queue and are ingested, in order, at
  // one site per trip (ingest_pending, right after advance): the controller's
  // output r is read only at admissions, which come after that site, so the
  // deferral changes nothing — but every lane's ingests run at the same place
  // of the loop, not at two (advance and the leap), which halves the warp's
  // divergent passes over the controller code.  A leap queues at most one
  // second (it stops before a second crossing once the queue is not empty).
  LHD void push_second(uint64_t sum, uint32_t cnt, uint32_t sec) {
    if (npend == 0) {
      pa_sum = sum;
      pa_cnt = cnt;
      pa_sec = sec;
    } else {
      pb_sum = sum;
      pb_cnt = cnt;
      pb_sec = sec;
    }
    npend++;
  }
  LHD void ingest_pending() {
#pragma unroll 1
    for (uint32_t i = 0; i < npend; ++i) {  // one inlined copy of the controller
      const bool b = i != 0;
      ingest(b ? pb_sum : pa_sum, b ? pb_cnt : pa_cnt, b ? pb_sec : pa_sec);
    }
    npend = 0;
  }
  // close the open second (queued if it holds samples) and open the one containing t
  LHD void roll_second(uint32_t t) {
    if (t < sec_bound) return;
    if (acc_cnt) push_second(acc_sum, acc_cnt, sec_bound);
    acc_sum = 0;
    acc_cnt = 0;
    const uint32_t nb = sec_bound + 1000000u;
    if (__builtin_expect(t < nb, 1)) sec_bound = nb;  // usually the next second (no division)
    else sec_bound = (t / 1000000u + 1u) * 1000000u;
  }

  LHD void advance(uint32_t t) {
    T = t;
    const uint32_t b = sec_bound < win_next ? sec_bound : win_next;
    if (t < b) return;
    roll_second(t);
    if (t >= win_next) update_window();
  }

  // ------------------------------------------------------------------ a2 + a3
  // One candidate from the tag-0 block u of candidate j (P:183 Poisson, S:83
  // thinning; R17, R32, R33): its time tau = gen_tau + Exp draw, whether it
  // crosses the segment's end, whether thinning accepts it.
  // The request's attributes and own draws (tag-1 block): the FIFO entry.
#ifdef BELLMAN_AB_ENTRY_CALL
  __device__ __host__ __noinline__ static void make_entry(
#else
  __device__ __host__ static void make_entry(
#endif
      const Params &p, uint32_t key0, uint32_t wl, uint32_t wh, uint32_t j,
                                             const U4 &u, uint64_t tau, uint32_t e[6]) {
    const uint32_t L = (uint32_t)ldg(&p.tabL[u.z >> 20]);
    const uint32_t xc = u.z & 0xFFFFFu;  // class draw (NEXT-3): the bits below L's index
    const uint32_t cls = xc < p.class_cum0 ? 0u : (xc < p.class_cum1 ? 1u : (xc < p.class_cum2 ? 2u : 3u));
    const uint32_t in = (uint32_t)ldg(&p.tabI[u.w >> 20]);
    const U4 v = philox(key0, kSeedHi, j, 1u, wl, wh);
    const uint64_t U = ((uint64_t)L * (uint32_t)ldg(&p.tabF[v.x >> 20]) + 32768u) >> 16;  // S:139, R14
    const int32_t P0 = (int32_t)L + ldg(&p.tabN[v.y >> 20]);
    e[0] = tau < kFar ? (uint32_t)tau : kFar;
    e[1] = in | (cls << 16);
    e[2] = U < 1 ? 1u : (uint32_t)U;
    e[3] = P0 < 1 ? 1u : (uint32_t)P0;
    e[4] = (uint32_t)ldg(&p.tabC[v.z >> 20]) | ((uint32_t)(ldg(&p.tabQ[v.w >> 20]) + 2048) << 20);
    e[5] = j;
  }
  LHD static bool thin_accept(const DevSeg &S, uint32_t u1, uint64_t tau) {
    // u1 lmax span < (la (tb - tau) + lb (tau - ta)) 2^32, in 128 bits
    const uint64_t x = (uint64_t)u1 * S.lmax;
    const uint64_t lhs_hi = mulhi64(x, S.span), lhs_lo = x * S.span;
    const uint64_t y = (uint64_t)S.la * (S.tb - tau) + (uint64_t)S.lb * (tau - S.ta);
    const uint64_t rhs_hi = y >> 32, rhs_lo = y << 32;
    return lhs_hi < rhs_hi || (lhs_hi == rhs_hi && lhs_lo < rhs_lo);
  }
  // Scalar generation (the fallback when the FIFO is empty, and the epilogue's
  // count): the next candidate; false when the generator is exhausted.
  LHD bool candidate(const Params &p, uint32_t &j, uint64_t &tau, U4 &u, bool &acc) {
    for (;;) {
      if (gen_seg >= n_seg) {
        gen_done = 1;
        return false;
      }
      const DevSeg &S = p.segs[seg_off + gen_seg];
      if (gen_fresh) {
        gen_tau = S.ta;
        gen_fresh = 0;
      }
      j = gen_j++;
      u = philox(k0, kSeedHi, j, 0u, wid_lo, wid_hi);
      tau = gen_tau + mulhi64(neglog_q32(u.x, ldg(&p.log2tab[neglog_index(u.x)])), S.M);
      if (tau >= S.tb) {  // the crossing candidate is consumed (R17)
        gen_seg++;
        gen_fresh = 1;
        continue;
      }
      gen_tau = tau;
      acc = thin_accept(S, u.y, tau);
      if (acc) {
        gen_acc++;
        if (gen_cap && gen_acc >= gen_cap) gen_done = 1;  // the capped arrival is still delivered
      }
      return true;
    }
  }
  // the next accepted arrival of the stream into e (false: none)
  LHD bool scalar_next(const Params &p, uint32_t e[6]) {
    for (;;) {
      if (gen_done) return false;
      uint32_t j;
      uint64_t tau;
      U4 u;
      bool acc;
      if (!candidate(p, j, tau, u, acc)) return false;
      if (!acc) continue;
      make_entry(p, k0, wid_lo, wid_hi, j, u, tau, e);
      return true;
    }
  }
  LHD void fifo_pop(uint32_t e[6]) {
    const uint2 a = fifo[3u * frd], b = fifo[3u * frd + 1u], c = fifo[3u * frd + 2u];
    e[0] = a.x;
    e[1] = a.y;
    e[2] = b.x;
    e[3] = b.y;
    e[4] = c.x;
    e[5] = c.y;
    frd = (frd + 1u) & 31u;
    fcnt--;
#ifdef __CUDA_ARCH__
    // the entry after it into L2 (no register waits on a prefetch): the pops
    // come many trips after the refill wrote the ring
    if (fcnt) asm volatile("prefetch.global.L2 [%0];" ::"l"(fifo + 3u * frd));
#endif
  }
  // the head moves on: next -> head, the FIFO's front -> next (its loads are
  // consumed at a later admission); scalar generation when both are empty
  LHD void next_head(const Params &p) {
    uint32_t e[6];
    if (n_ok) {
      head_t = n_t;
      h_in = n_in;
      h_U = n_U;
      h_P = n_P;
      h_fcq = n_fcq;
      h_j = n_j;
      n_ok = 0;
    } else if (fcnt) {
      fifo_pop(e);
      head_t = e[0];
      h_in = e[1];
      h_U = e[2];
      h_P = e[3];
      h_fcq = e[4];
      h_j = e[5];
    } else if (scalar_next(p, e)) {
      head_t = e[0];
      h_in = e[1];
      h_U = e[2];
      h_P = e[3];
      h_fcq = e[4];
      h_j = e[5];
    } else {
      head_t = kInf;
    }
    refill_next();
  }
  LHD void refill_next() {
    if (n_ok || !fcnt || head_t == kInf) return;
    uint32_t e[6];
    fifo_pop(e);
    n_t = e[0];
    n_in = e[1];
    n_U = e[2];
    n_P = e[3];
    n_fcq = e[4];
    n_j = e[5];
    n_ok = 1;
  }

#ifdef __CUDA_ARCH__
  // Warp-cooperative generation for lane `who` (every lane of the warp calls
  // it, converged): its generator state is broadcast, lane l draws candidate
  // j + l (tag-0 Philox block, -ln U, a warp prefix sum of the gaps), the
  // crossing rule and thinning by ballot, and each accepted candidate's lane
  // writes its FIFO entry (tag-1 draws) at its rank — K2's refill, per lane.
  // Candidates after a segment crossing are discarded and redrawn in the next
  // segment (the crossing one is consumed, R17), as in the scalar generator.
  __device__ void coop_refill(const Params &p, uint32_t who, uint32_t lane, uint2 *fifo_warp) {
    const uint32_t F = 0xffffffffu;
    uint32_t gseg = __shfl_sync(F, gen_seg, who), gj = __shfl_sync(F, gen_j, who);
    uint32_t gacc = __shfl_sync(F, gen_acc, who), gdone = __shfl_sync(F, gen_done, who);
    uint32_t gfresh = __shfl_sync(F, gen_fresh, who);
    uint64_t gtau = __shfl_sync(F, (unsigned long long)gen_tau, who);
    const uint32_t nseg = __shfl_sync(F, n_seg, who), soff = __shfl_sync(F, seg_off, who);
    const uint32_t gcap = __shfl_sync(F, gen_cap, who), key0 = __shfl_sync(F, k0, who);
    const uint32_t wl = __shfl_sync(F, wid_lo, who), wh = __shfl_sync(F, wid_hi, who);
    const uint32_t tail0 = (__shfl_sync(F, frd, who) + __shfl_sync(F, fcnt, who)) & 31u;
    uint2 *fw = fifo_warp + 96u * who;
    uint32_t added = 0;
    while (!gdone && added == 0) {
      if (gseg >= nseg) {
        gdone = 1;
        break;
      }
      const DevSeg S = p.segs[soff + gseg];
      if (gfresh) {
        gtau = S.ta;
        gfresh = 0;
      }
      const uint32_t jj = gj + lane;
      const U4 u = philox(key0, kSeedHi, jj, 0u, wl, wh);
      uint64_t incl = mulhi64(neglog_q32(u.x, ldg(&p.log2tab[neglog_index(u.x)])), S.M);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(F, (unsigned long long)incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      const uint64_t tau = gtau + incl;
      const uint32_t om = __ballot_sync(F, tau >= S.tb);
      const uint32_t first_over = om ? (uint32_t)__ffs((int)om) - 1u : 32u;
      const bool acc = lane < first_over && thin_accept(S, u.y, tau);
      uint32_t am = __ballot_sync(F, acc);
      if (gcap) {  // the arrival cap: keep the first `room` accepted
        const uint32_t room = gcap - gacc;
        if ((uint32_t)__popc(am) >= room) {
          const uint32_t cut = room ? __fns(am, 0, (int)room) : 0u;
          am = room ? (am & (0xffffffffu >> (31u - cut))) : 0u;
          gdone = 1;
        }
      }
      if ((am >> lane) & 1u) {
        const uint32_t e = (uint32_t)__popc(am & ((1u << lane) - 1u));
        uint32_t ent[6];
        make_entry(p, key0, wl, wh, jj, u, tau, ent);
        uint2 *f = fw + 3u * ((tail0 + added + e) & 31u);
        f[0] = make_uint2(ent[0], ent[1]);
        f[1] = make_uint2(ent[2], ent[3]);
        f[2] = make_uint2(ent[4], ent[5]);
      }
      const uint32_t na = (uint32_t)__popc(am);
      added += na;
      gacc += na;
      if (first_over < 32u) {
        gj += first_over + 1u;
        gseg++;
        gfresh = 1;
      } else {
        gj += 32u;
        gtau = __shfl_sync(F, (unsigned long long)tau, 31);
      }
    }
    __syncwarp();  // the entries' stores precede lane `who`'s loads
    if (lane == who) {
      gen_seg = gseg;
      gen_j = gj;
      gen_acc = gacc;
      gen_done = gdone;
      gen_fresh = gfresh;
      gen_tau = gtau;
      fcnt += added;
    }
  }
#endif
  // the same FIFO contents one at a time (the CPU development build)
  LHD void fill_host(const Params &p) {
    uint32_t e[6];
    while (fcnt < 32u && scalar_next(p, e)) {
      uint2 *f = fifo + 3u * ((frd + fcnt) & 31u);
      f[0] = make_uint2(e[0], e[1]);
      f[1] = make_uint2(e[2], e[3]);
      f[2] = make_uint2(e[4], e[5]);
      fcnt++;
    }
  }
  // after a refill: the head (a fresh scenario) or the next, from the FIFO
  LHD void after_refill(const Params &p) {
    if (head_t == kInf) {
      if (fcnt || !gen_done) next_head(p);
    } else {
      refill_next();
    }
  }

  // ------------------------------------------------------------------ a1 scenario decode
  LHD void init(const Params &p, uint64_t id, uint32_t *smem_lane, uint32_t *hist_lane, uint2 *fifo_lane) {
    sm = smem_lane;
    hist = hist_lane;
    fifo = fifo_lane;
    sid = id;
    const bellman_scenario sc = p.sc[id];
    const bellman_ctrl &cc = p.ctrls[sc.ctrl];
    const bellman_profile &pr = p.profs[sc.profile];
    const DevTrace tr = p.traces[sc.trace];
    t0 = pr.t0_us;
    cm = p.cost_magic + (uint64_t)kCostMagicB * sc.profile;
    knee = pr.knee;
    slope = pr.slope_us;
    kv = KV0 ? 0u : pr.kv_ns_per_word;
    maxb = pr.max_batch;
    pf_ns = pr.prefill_ns_per_word;
    slo_us = cc.slo_us;
    H = (uint32_t)sc.horizon_us;
    w0 = sc.w0_us <= 0 ? 0u : (sc.w0_us >= (int64_t)kFar ? kFar : (uint32_t)sc.w0_us);
    w1 = sc.w1_us <= 0 ? 0u : (sc.w1_us >= (int64_t)kFar ? kFar : (uint32_t)sc.w1_us);
    drain = sc.mode == BELLMAN_MODE_DRAIN;
    // a10: thresholds from the paired unbounded run's calibration
    law = cc.law;
    t1 = cc.t1;
    t2 = cc.t2;
    flags = 0;
    if (cc.calibrated) {
      const uint32_t *cb = p.calib + 4u * p.series_slot[sc.calib_src];
      t1 = cb[0];
      t2 = cb[1];
      if (cb[2] != 0) {
        law = BELLMAN_LAW_OFF;
        flags |= BELLMAN_FLAG_DEGENERATE_CALIB;
      }
    }
    window = cc.window;
    rmin = cc.r_min_bp;
    rmax = cc.r_max_bp;
    nrungs = cc.n_rungs;
#pragma unroll
    for (int k = 0; k < 4; ++k) rk[k] = cc.rungs_bp[2 * k] | (cc.rungs_bp[2 * k + 1] << 16);
    r = law == BELLMAN_LAW_CONST ? cc.r_const_bp : 0u;
    ringA = 0;
    ring_n = ring_pos = rung = active = activations = active_ingests = 0;
    first_act = last_deact = kNone;
    ev_next = 0;
    rslot = p.series_slot[id];
    series = rslot != kNone ? p.series + p.series_off[rslot] : nullptr;
    series_cap = rslot != kNone ? p.series_cap[rslot] : 0u;
    series_n = 0;
    // the per-second signal feeds only the controller (MAP / STEP) and the recorder
    sec_bound = (law >= BELLMAN_LAW_MAP || rslot != kNone) ? 1000000u : kInf;
    acc_sum = 0;
    acc_cnt = 0;
    npend = 0;
    pa_sum = pb_sum = 0;
    pa_cnt = pb_cnt = pa_sec = pb_sec = 0;
    T = 0;
    busy = 0;
    iter_end = kInf;
    iter_d = 0;
    iter_align = 0;
    ticks = 0;
    next_done = kInf;
    next_pf = kInf;
    n_ready = B = in_sys = 0;
    kq = kr = kstep_q = kstep_r = 0;
    batch_changed();
    update_window();
    free_m = maxb >= 64u ? ~0ull : ((1ull << maxb) - 1ull);
    pf_m = rdy_m = 0;
    rdy_sum = 0;
    rdy_kadd = 0;
    nheap = 0;
    heap_reset();
    // generator
    k0 = sc.seed_index;
    wid_lo = (uint32_t)sc.wid;
    wid_hi = (uint32_t)(sc.wid >> 32);
    bypass_mask = cc.bypass_mask;
    min_words = cc.min_words_bypass;
    n_seg = tr.n_seg;
    seg_off = tr.seg_off;
    gen_cap = tr.cap;
    gen_seg = gen_j = gen_acc = gen_done = 0;
    gen_fresh = 1;
    gen_tau = 0;
    frd = fcnt = 0;
    n_ok = 0;
    head_t = kInf;  // the first refill (coop_refill, or fill_host) sets the head
    c_admitted = c_served = c_rewritten = c_slo = c_win_served = c_words_in = c_idle = c_win_words_in = 0;
    c_win_idle = c_sum_queue = c_sum_ttft = c_sum_e2e = words_out = win_words_out = n_ttft = 0;
    last_j = bypassed = finished = 0;
    segment = sc.segment;
    hm_e2e = hm_ttft = hm_r = hm_q = 0;
  }

  // ------------------------------------------------------------------ a5
  LHD void iteration_words() {
    words_out += B;
    if (win_now) win_words_out += B;
    acc_sum += (uint64_t)B * iter_d + iter_align;  // TBT: the B gaps of this end
    acc_cnt += B;
    if (!KV0) {
      kr += kstep_r;
      kq += kstep_q;
      if (kr >= 1000u) {
        kr -= 1000u;
        kq++;
      }
    }
  }

  LHD void iteration_end() {
    iteration_words();
    const uint32_t it = ticks - 1u;
    if (it == next_done) {
      uint64_t se = 0;
      uint32_t ndone = 0, nslo = 0, kd = 0;
      uint32_t rk;
      do {
        const uint32_t s = heap_pop(rk);
        const uint32_t e = T - SL(F_ARR, s);
        se += e;
        nslo += e > slo_us ? 1u : 0u;
        ndone++;
        if (!KV0) kd += SL(F_IN, s) + SL(F_R, s);
        hist_add(kHistE2E, lat_bin(e), hm_e2e);
        free_m |= 1ull << s;
      } while (rk == it);  // rk: the new root's key (kInf when empty)
      next_done = rk;
      if (!KV0) kv_sub((uint64_t)kv * kd);
      c_served += ndone;
      c_sum_e2e += se;
      c_slo += nslo;
      if (win_now) c_win_served += ndone;
      in_sys -= ndone;
      B -= ndone;
      batch_changed();
    }
    busy = 0;
  }

  // prefill ends at instants in [T, lim): first words, R = 1 completions (R9)
  LHD void prefill_end(uint32_t lim) {
    uint64_t m = pf_m, st = 0, se = 0, done = 0, one = 0;
    uint32_t mpf = kInf, nfirst = 0, n1 = 0, nslo = 0;
    while (m) {
      const uint64_t bit = m & (0ull - m);
      const uint32_t s = ffs64(m) - 1u;
      m ^= bit;
      const uint32_t key = SL(F_PF, s);
      if (key < lim) {
        const uint32_t tt = key - SL(F_ARR, s);
        const uint32_t lb = lat_bin(tt);
        st += tt;
        nfirst++;
        hist_add(kHistTTFT, lb, hm_ttft);
        done |= bit;
        if (SL(F_R, s) == 1u) {  // R = 1: completes with its first word (R9)
          se += tt;
          nslo += tt > slo_us ? 1u : 0u;
          n1++;
          hist_add(kHistE2E, lb, hm_e2e);
          one |= bit;
        } else {
          rdy_sum += key;
          if (!KV0) rdy_kadd += SL(F_IN, s) + 1u;
        }
      } else if (key < mpf) {
        mpf = key;
      }
    }
    // the slot phase masks once per call (A/B on full C5: 488.4 -> 479.7 ms
    // against per-slot mask updates, r02w)
    pf_m &= ~done;
    free_m |= one;
    rdy_m |= done & ~one;
    n_ready += nfirst - n1;
    next_pf = mpf;
    n_ttft += nfirst;
    c_sum_ttft += st;
    words_out += nfirst;
    if (win_now) win_words_out += nfirst;
    if (n1) {
      c_served += n1;
      c_sum_e2e += se;
      c_slo += nslo;
      if (win_now) c_win_served += n1;
      in_sys -= n1;
    }
  }

  // ------------------------------------------------------------------ a7 (+a3)
  // FIFO admission at an admission point (R7).  Precondition: in_sys < maxb, head_t <= T.
  LHD void admit(const Params &p) {
    const uint32_t Tn = T;
    uint32_t n = 0, n_byp = 0;
    do {
      // the head (a3): U, P, F_comp | similarity noise drawn at generation; prefill
      // max(1, floor(pf_ns in / 1000)); the bypass rule (NEXT-3)
      const uint32_t a = head_t, in = h_in & 0xFFFFu, cls = h_in >> 16, U = h_U, P = h_P, fcq = h_fcq;
      const uint32_t pf0 = (uint32_t)(((uint64_t)pf_ns * in) / 1000u);
      const uint32_t pf = pf0 < 1u ? 1u : pf0;
      const bool byp = (r > 0) & ((((bypass_mask >> cls) & 1u) != 0u) | (P < min_words));  // branch-free
      const uint32_t ra = byp ? 0u : r;
      uint32_t R = U, qb;
      if (ra > 0) {
        R = realized_len(p, P, fcq, ra);
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
        c_rewritten++;
        hist_add(kHistR, ra / 10u < BELLMAN_HIST_R ? ra / 10u : BELLMAN_HIST_R - 1u, hm_r);
        hist_add(kHistQA, qb, hm_q);
      } else {  // not rewritten: the inactive base plus the noise
        int32_t sc = (int32_t)p.q_inactive + (int32_t)(fcq >> 20) - 2048;
        sc = sc < 0 ? 0 : (sc > 10000 ? 10000 : sc);
        qb = (uint32_t)sc / 50u;
        hist_add(kHistQI, qb, hm_q, 8u);
      }
      n_byp += byp ? 1u : 0u;
      const uint64_t bit = free_m & (0ull - free_m);  // the lowest free slot (no 64-bit shift)
      const uint32_t s = ffs64(free_m) - 1u;
      free_m ^= bit;
      pf_m |= bit;
      const uint32_t pe = Tn + pf;
      SL(F_PF, s) = pe;
      SL(F_ARR, s) = a;
      SL(F_R, s) = R;
      if (!KV0) SL(F_IN, s) = in;
      if (pe < next_pf) next_pf = pe;
      c_words_in += in;
      if (win_now) c_win_words_in += in;
      c_sum_queue += Tn - a;
      n++;
      in_sys++;
      last_j = h_j + 1u;
      next_head(p);
    } while (in_sys < maxb && head_t <= Tn);
    c_admitted += n;
    bypassed += n_byp;
  }

  // ------------------------------------------------------------------ a4/a5 leap
  // the longest run of uneventful iterations in bulk (K2's leap, scalar)
  LHD void leap() {
    uint32_t stop = next_pf < stop_static ? next_pf : stop_static;
    if (in_sys < maxb && head_t < stop) stop = head_t;
    const uint32_t nmax = next_done - ticks;  // iterations ticks .. next_done-1 complete nobody
    if (nmax == 0 || stop <= T + 1u) return;
    const uint32_t cb = cbase, qs = kstep_q, rs = kstep_r;
    uint32_t q = KV0 ? 0u : kq, rr = KV0 ? 0u : kr, done = 0;
    for (;;) {
      const uint32_t lim = stop < sec_bound ? stop : sec_bound;
      const uint32_t room = lim - 1u - T;
      const uint32_t left = nmax - done;
      uint32_t n = 0, used = 0;
      if (KV0) {
#ifdef BELLMAN_AB_LEAPDIV
        const uint32_t nn = room / cb;
#else
        // floor(room / c(B)) by the profile's reciprocal (exact: bellman_internal.cuh)
        const uint32_t nn = (uint32_t)mulhi64(cmag, (uint64_t)room << 1);
#endif
        n = nn < left ? nn : left;
        used = n * cb;
      } else {
        while (n < left) {
          const uint32_t d = cb + q;
          if (d > room - used) break;
          used += d;
          rr += rs;
          const uint32_t carry = rr >= 1000u ? 1u : 0u;
          rr -= carry ? 1000u : 0u;
          q += qs + carry;
          n++;
        }
      }
      const uint64_t words = (uint64_t)n * B;
      ticks += n;
      T += used;
      words_out += words;
      if (win_now) win_words_out += words;
      acc_sum += (uint64_t)B * used;
      acc_cnt += (uint32_t)words;
      done += n;
      const uint32_t tnext = T + (cb + q);
      if ((done == nmax) | (tnext >= stop) | (tnext < sec_bound) | (npend != 0)) break;
      roll_second(tnext);
    }
    if (!KV0) {
      kq = q;
      kr = rr;
    }
  }

  // ------------------------------------------------------------------ a4
  LHD void start_iteration() {
    const uint32_t Tn = T;
    uint64_t align = 0;
    if (n_ready) {
      const uint32_t it0 = ticks;
      uint64_t m = rdy_m;
      while (m) {
        const uint32_t s = ffs64(m) - 1u;
        m &= m - 1ull;
        // words 2..R at the ends of iterations it0 .. it0 + R - 2
        const uint32_t k = it0 + SL(F_R, s) - 2u;
        SL(F_PF, s) = k;
        heap_push(s, k);
#ifndef BELLMAN_AB_NOKEYTRACK
        next_done = k < next_done ? k : next_done;  // the heap's least key (pushes only add keys)
#endif
      }
      rdy_m = 0;
      align = (uint64_t)n_ready * Tn - rdy_sum;
      rdy_sum = 0;
#ifdef BELLMAN_AB_NOKEYTRACK
      next_done = key(HB(kHeapRoot));
#endif
      if (!KV0) {
        kv_add((uint64_t)kv * rdy_kadd);
        rdy_kadd = 0;
      }
      B += n_ready;
      n_ready = 0;
      batch_changed();
    }
    const uint32_t d = cbase + (KV0 ? 0u : kq);
    iter_d = d;
    iter_align = align;
    iter_end = Tn + d;
    busy = 1;
    ticks++;
  }

  LHD bool quiet_end() {
    const uint32_t te = iter_end;
    uint32_t lim = stop_static < sec_bound ? stop_static : sec_bound;
    lim = lim < next_pf ? lim : next_pf;
    if ((te >= lim) | (ticks - 1u == next_done) | ((in_sys < maxb) & (head_t <= te))) return false;
    T = te;
    iteration_words();
    busy = 0;
    return true;
  }

  // ------------------------------------------------------------------ one event trip
  // Returns true when the scenario's event loop is over (finished: drained).
#ifndef BELLMAN_AB_PF2
  // One prefill-end call site per trip for every lane: before the clock
  // advance, the ends due before min(next event + 1, stop_static) — a busy
  // lane's ends inside its running iteration and at its end, an idle lane's
  // ends at its next event.  Order-free against the iteration end, the clock
  // advance and the ingest of the same trip (disjoint state but commutative
  // sums; the window flag cannot change below stop_static), so each lane's
  // result is the two-site loop's; only ends at or past a window / horizon
  // boundary (stop_static) keep the second, post-advance site (rare).
  LHD bool trip(const Params &p) {
    uint32_t tn, lim;
    bool mid = false;
    if (busy) {
      tn = iter_end;
      lim = iter_end + 1u < stop_static ? iter_end + 1u : stop_static;
    } else {
      tn = next_pf;
      if (in_sys < maxb && head_t < tn) tn = head_t;
      if (tn == kInf) {
        finished = 1;
        return true;
      }
      if ((tn >= H) | (in_sys == 0)) {
        if (tn >= H) return true;
        idle(T, tn);
      }
      lim = tn + 1u < stop_static ? tn + 1u : stop_static;
    }
    if (next_pf < lim) prefill_end(lim);
    if (busy) {
      mid = next_pf < iter_end;
      if (mid) tn = next_pf;
      if (tn >= H) return true;
    }
    advance(tn);
    ingest_pending();
    if (busy && !mid) iteration_end();
    if (next_pf == tn) {  // at or past a window / horizon boundary only
      uint32_t lim2 = tn + 1u;
      if (mid) lim2 = iter_end < stop_static ? iter_end : stop_static;
      prefill_end(lim2);
      if (mid) return false;
    }
    if (in_sys < maxb && head_t <= tn) admit(p);
    if (n_ready + B > 0) {
      bool join;
      do {
        join = n_ready != 0;
        if (!join) leap();
        start_iteration();
      } while (join && quiet_end());
    }
    return false;
  }
#else
  LHD bool trip(const Params &p) {
    uint32_t tn;
    bool mid = false;
    if (busy) {
      // prefill ends due inside the running iteration and window: handled now
      // (order-free until the iteration end; in the TBT-only loop a prefill
      // end touches no per-second state, so a second boundary needs no split)
      uint32_t lim = iter_end < stop_static ? iter_end : stop_static;
#ifdef BELLMAN_AB_PF_SECSPLIT
      if (sec_bound < lim) lim = sec_bound;
#endif
      if (next_pf < lim) prefill_end(lim);
      mid = next_pf < iter_end;
      tn = mid ? next_pf : iter_end;
    } else {
      tn = next_pf;
      if (in_sys < maxb && head_t < tn) tn = head_t;
      if (tn == kInf) {
        finished = 1;
        return true;
      }
    }
    if ((tn >= H) | (in_sys == 0)) {
      if (tn >= H) return true;
      idle(T, tn);
    }
    advance(tn);
    ingest_pending();
    if (busy && !mid) iteration_end();
    if (next_pf == tn) {
      uint32_t lim = tn + 1u;
      if (mid) {
        lim = iter_end < stop_static ? iter_end : stop_static;
#ifdef BELLMAN_AB_PF_SECSPLIT
        if (sec_bound < lim) lim = sec_bound;
#endif
      }
      prefill_end(lim);
      if (mid) return false;
    }
    if (in_sys < maxb && head_t <= tn) admit(p);
    if (n_ready + B > 0) {
      bool join;
      do {
        join = n_ready != 0;
        if (!join) leap();
        start_iteration();
      } while (join && quiet_end());
    }
    return false;
  }
#endif

  // ------------------------------------------------------------------ a9 histogram scan
  // Walk the touched groups of one histogram in bin order: nearest-rank
  // percentiles (k = ceil(p n / 100), the first bin whose
  // cumulative count reaches k), the segment merge (integer atomics) and the
  // re-zeroing of the groups for the thread's next scenario.
  LHD void scan(uint32_t off, uint32_t nb, uint32_t mask, uint64_t n, uint32_t p0, uint32_t p1, uint32_t &b0,
                uint32_t &b1, unsigned long long *seg) {
    const uint64_t k0v = ((uint64_t)p0 * n + 99u) / 100u, k1v = ((uint64_t)p1 * n + 99u) / 100u;
    const uint64_t ka = k0v < 1 ? 1 : k0v, kb = k1v < 1 ? 1 : k1v;
    b0 = b1 = kNone;
    uint64_t cum = 0;
    while (mask) {
      const uint32_t g = ffs32(mask) - 1u;
      mask &= mask - 1u;
      uint4 *v4 = reinterpret_cast<uint4 *>(hist + off + 32u * g);
#pragma unroll 1
      for (uint32_t i = 0; i < 8; ++i) {
        const uint4 v = v4[i];
        if ((v.x | v.y | v.z | v.w) == 0) continue;
        const uint32_t c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
          if (!c[k]) continue;
          const uint32_t b = 32u * g + 4u * i + k;
          cum += c[k];
          seg_add(&seg[b], c[k]);
          if (b0 == kNone && cum >= ka) b0 = b;
          if (p1 && b1 == kNone && cum >= kb) b1 = b;
        }
        v4[i] = make_uint4(0, 0, 0, 0);
      }
    }
    (void)nb;
    if (n == 0) b0 = b1 = kNone;
  }

  // ------------------------------------------------------------------ termination, a8, a9
  // the end of a scenario: termination and the queue count (finish_pre), the
  // histogram walks (scan_all on the host; coop_hists, the whole warp, on the
  // GPU), the record (finish_post)
  LHD void finish_pre(const Params &p) {
    // R20: a drained run ends at its last event, a cutoff run at H
    const uint32_t end = (drain && finished) ? T : H;
    if (in_sys == 0) idle(T, end);
    if (sec_bound != kInf && sec_bound <= end && acc_cnt) push_second(acc_sum, acc_cnt, sec_bound);
    ingest_pending();
    // queued at the end: accepted arrivals before `end` not admitted
    uint64_t queued = 0;
    if (head_t != kInf) {  // the head, the next, the FIFO, then the rest of the stream (counted only)
      bool more = head_t < end;
      if (more) {
        queued = 1;
        last_j = h_j + 1u;
      }
      if (more && n_ok) {
        more = n_t < end;
        if (more) {
          queued++;
          last_j = n_j + 1u;
        }
      }
      while (more && fcnt) {
        uint32_t e[6];
        fifo_pop(e);
        more = e[0] < end;
        if (more) {
          queued++;
          last_j = e[5] + 1u;
        }
      }
      while (more && !gen_done) {  // tag-0 draws and thinning only
        uint32_t j;
        uint64_t tau;
        U4 u;
        bool acc;
        if (!candidate(p, j, tau, u, acc)) break;
        if (!acc) continue;
        if (tau >= end) break;
        queued++;
        last_j = j + 1u;
      }
    }
    if (series) p.series_n[rslot] = series_n;
    fin_end = end;
    fin_queued = queued;
#if defined(__CUDA_ARCH__) && !defined(BELLMAN_AB_NOHISTPF)
    {  // the touched histogram lines into L2 at once (the walks below then hit L2)
      const uint32_t offs[5] = {kHistE2E, kHistTTFT, kHistR, kHistQA, kHistQI};
      const uint32_t masks[5] = {hm_e2e, hm_ttft, hm_r, hm_q & 0xFFu, hm_q >> 8};
#pragma unroll
      for (int h5 = 0; h5 < 5; ++h5)
        for (uint32_t m = masks[h5]; m; m &= m - 1u)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(hist + offs[h5] + 32u * (ffs32(m) - 1u)));
    }
#endif
  }

  // the walks one lane at a time (the CPU development build)
  LHD void scan_all(const Params &p) {
    unsigned long long *seg = p.seg_hist + (uint64_t)segment * kSegWords;
    uint32_t dummy;
    scan(kHistE2E, BELLMAN_HIST_LAT, hm_e2e, c_served, 50u, 99u, r_e50, r_e99, seg);
    scan(kHistTTFT, BELLMAN_HIST_LAT, hm_ttft, n_ttft, 50u, 99u, r_f50, r_f99, seg + BELLMAN_HIST_LAT);
    scan(kHistR, BELLMAN_HIST_R, hm_r, c_rewritten, 50u, 0u, r_rm, dummy, seg + 2 * BELLMAN_HIST_LAT);
    scan(kHistQA, BELLMAN_HIST_Q, hm_q & 0xFFu, c_rewritten, 50u, 0u, r_qa, dummy,
         seg + 2 * BELLMAN_HIST_LAT + BELLMAN_HIST_R);
    scan(kHistQI, BELLMAN_HIST_Q, hm_q >> 8, c_admitted - c_rewritten, 50u, 0u, r_qi, dummy,
         seg + 2 * BELLMAN_HIST_LAT + BELLMAN_HIST_R + BELLMAN_HIST_Q);
  }

#ifdef __CUDA_ARCH__
  // One histogram of lane `who`, by the whole warp (converged): lane l takes
  // the l-th touched 32-bin group (groups in bin order), sums it, merges its
  // non-zero bins into the segment histogram; a warp prefix sum of the group
  // counts finds, for each nearest-rank k = max(1, ceil(p n / 100)),
  // the lane whose group holds the k-th count, which walks its 32 bins; then
  // the groups are re-zeroed.  K2's warp_percentiles over the touched groups.
  __device__ static void coop_one(uint32_t *h, uint32_t mask, uint64_t n, uint32_t p0, uint32_t p1, uint32_t &b0,
                                  uint32_t &b1, unsigned long long *seg, uint32_t lane) {
    const uint32_t F = 0xffffffffu;
    const uint32_t ng = (uint32_t)__popc(mask);
    const bool mine = lane < ng;
    const uint32_t g = mine ? (uint32_t)__fns(mask, 0, (int)lane + 1) : 0u;
    uint4 *v4 = reinterpret_cast<uint4 *>(h + 32u * g);
    uint32_t csum = 0;
    if (mine) {
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) {
        const uint4 v = v4[i];
        const uint32_t c[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k)
          if (c[k]) seg_add(&seg[32u * g + 4u * i + k], c[k]);
        csum += v.x + v.y + v.z + v.w;
      }
    }
    uint32_t incl = csum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(F, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    b0 = b1 = kNone;
    if (n != 0) {
#pragma unroll 1
      for (uint32_t q = 0; q < 2; ++q) {
        const uint32_t pq = q ? p1 : p0;
        if (!pq) break;
        uint64_t k = ((uint64_t)pq * n + 99u) / 100u;
        if (k < 1) k = 1;
        const uint32_t bal = __ballot_sync(F, mine && (uint64_t)incl >= k);
        const uint32_t L = (uint32_t)__ffs((int)bal) - 1u;
        uint32_t res = 0;
        if (lane == L) {
          uint64_t cum = incl - csum;
          const uint32_t *hb = h + 32u * g;
#pragma unroll 1
          for (uint32_t i = 0; i < 32; ++i) {
            cum += hb[i];
            if (cum >= k) {
              res = 32u * g + i;
              break;
            }
          }
        }
        res = __shfl_sync(F, res, (int)L);
        if (q) b1 = res;
        else b0 = res;
      }
    }
    __syncwarp();  // every lane's reads of the groups precede the re-zeroing
    if (mine) {
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) v4[i] = make_uint4(0, 0, 0, 0);
    }
  }
  // every histogram of lane `who` (a finished scenario), by the whole warp
  __device__ void coop_hists(const Params &p, uint32_t who, uint32_t lane, uint32_t *hist_warp) {
    const uint32_t F = 0xffffffffu;
    uint32_t *hb = hist_warp + (uint64_t)who * kLaneHistWords;
    const uint32_t me = __shfl_sync(F, hm_e2e, who), mt = __shfl_sync(F, hm_ttft, who);
    const uint32_t mr = __shfl_sync(F, hm_r, who), mq = __shfl_sync(F, hm_q, who);
    const uint64_t ne = __shfl_sync(F, (unsigned long long)c_served, who);
    const uint64_t nt = __shfl_sync(F, (unsigned long long)n_ttft, who);
    const uint64_t nr = __shfl_sync(F, (unsigned long long)c_rewritten, who);
    const uint64_t na = __shfl_sync(F, (unsigned long long)c_admitted, who);
    unsigned long long *seg = p.seg_hist + (uint64_t)__shfl_sync(F, segment, who) * kSegWords;
    uint32_t o[7], dummy;
    coop_one(hb + kHistE2E, me, ne, 50u, 99u, o[0], o[1], seg, lane);
    coop_one(hb + kHistTTFT, mt, nt, 50u, 99u, o[2], o[3], seg + BELLMAN_HIST_LAT, lane);
    coop_one(hb + kHistR, mr, nr, 50u, 0u, o[4], dummy, seg + 2 * BELLMAN_HIST_LAT, lane);
    coop_one(hb + kHistQA, mq & 0xFFu, nr, 50u, 0u, o[5], dummy, seg + 2 * BELLMAN_HIST_LAT + BELLMAN_HIST_R, lane);
    coop_one(hb + kHistQI, mq >> 8, na - nr, 50u, 0u, o[6], dummy,
             seg + 2 * BELLMAN_HIST_LAT + BELLMAN_HIST_R + BELLMAN_HIST_Q, lane);
    if (lane == who) {
      r_e50 = o[0];
      r_e99 = o[1];
      r_f50 = o[2];
      r_f99 = o[3];
      r_rm = o[4];
      r_qa = o[5];
      r_qi = o[6];
    }
  }
#endif

  // the summary record (a8) from the walks' percentiles
  LHD void finish_post(const Params &p) {
    const bellman_profile &pr = p.profs[p.sc[sid].profile];
    const uint32_t end = fin_end, e50 = r_e50, e99 = r_e99, f50 = r_f50, f99 = r_f99, rm = r_rm, qa = r_qa, qi = r_qi;
    const uint64_t queued = fin_queued;
    bellman_scenario_stats o;
    o.scenario_id = sid;
    o.ticks = ticks;
    o.candidates = last_j;
    o.arrivals = c_admitted + queued;
    o.admitted = c_admitted;
    o.served = c_served;
    o.rewritten = c_rewritten;
    o.words_in = c_words_in;
    o.words_out = words_out;
    o.idle_us = c_idle;
    o.end_us = end;
    o.queued_end = queued;
    o.inflight_end = in_sys;
    o.win_served = c_win_served;
    o.win_words_in = c_win_words_in;
    o.win_words_out = win_words_out;
    o.win_idle_us = c_win_idle;
    o.sum_queue_us = c_sum_queue;
    o.sum_ttft_us = c_sum_ttft;
    o.sum_e2e_us = c_sum_e2e;
    o.slo_violations = c_slo;
    o.e2e_p50_ms = e50 == kNone ? kNone : lat_edge(e50);
    o.e2e_p99_ms = e99 == kNone ? kNone : lat_edge(e99);
    o.ttft_p50_ms = f50 == kNone ? kNone : lat_edge(f50);
    o.ttft_p99_ms = f99 == kNone ? kNone : lat_edge(f99);
    o.median_r_bp = rm == kNone ? kNone : rm * 10u;
    o.t1 = t1;
    o.t2 = t2;
    o.activations = activations;
    o.first_act_s = first_act;
    o.last_deact_s = last_deact;
    o.active_ingests = active_ingests;
    uint32_t fl = flags | BELLMAN_FLAG_DONE;
    if (queued + in_sys > 0) fl |= BELLMAN_FLAG_TRUNCATED;
    o.flags = fl;
    o.segment = segment;
    o.bypassed = bypassed;
    // energy in fp64 with explicit round-to-nearest ops in a fixed order (R19)
#ifdef __CUDA_ARCH__
    const double a = __dmul_rn(pr.e_in_j_per_word, (double)c_words_in);
    const double b = __dmul_rn(pr.e_out_j_per_word, (double)words_out);
    const double c = __dmul_rn(pr.p_idle_w, (double)c_idle);
    o.energy_j = __dadd_rn(__dadd_rn(a, b), __ddiv_rn(c, 1e6));
    const double wa = __dmul_rn(pr.e_in_j_per_word, (double)c_win_words_in);
    const double wb = __dmul_rn(pr.e_out_j_per_word, (double)win_words_out);
    const double wc = __dmul_rn(pr.p_idle_w, (double)c_win_idle);
    o.win_energy_j = __dadd_rn(__dadd_rn(wa, wb), __ddiv_rn(wc, 1e6));
#else
    o.energy_j = (pr.e_in_j_per_word * (double)c_words_in + pr.e_out_j_per_word * (double)words_out) +
                 (pr.p_idle_w * (double)c_idle) / 1e6;
    o.win_energy_j = (pr.e_in_j_per_word * (double)c_win_words_in + pr.e_out_j_per_word * (double)win_words_out) +
                     (pr.p_idle_w * (double)c_win_idle) / 1e6;
#endif
    o.sim_active_p50 = qa == kNone ? kNone : qa * 50u;
    o.sim_inactive_p50 = qi == kNone ? kNone : qi * 50u;
    o.scored_active = c_rewritten;
    o.scored_inactive = c_admitted - c_rewritten;
    o.preemptions = 0;
    o._pad2 = 0;
    o.recompute_words = 0;
    p.stats[sid] = o;
#ifdef __CUDA_ARCH__
    if (p.n_peer) {  // fused exchange (§8(e)): the record to every rank's array over peer memory
      const uint4 *src = reinterpret_cast<const uint4 *>(&o);
      for (uint32_t g = 0; g < p.n_peer; ++g) {
        uint4 *dst = reinterpret_cast<uint4 *>(&p.peer[g][sid]);
#pragma unroll
        for (uint32_t c2 = 0; c2 < sizeof(bellman_scenario_stats) / 16; ++c2) dst[c2] = src[c2];
      }
      __threadfence_system();
    }
#endif
  }
};

// Whether scenario `sid` belongs to lane kernel `kind` (3 or 4) in this pass.
LHD bool mine(const Params &p, uint64_t sid, uint32_t kind) {
  const bellman_scenario &sc = p.sc[sid];
  const bellman_ctrl &cc = p.ctrls[sc.ctrl];
  if ((cc.calibrated != 0) != (p.pass == 2)) return false;
  return scenario_kind_of(sc, cc, p.profs[sc.profile], p.traces[sc.trace].kind, p.lane_on) == kind;
}

}  // namespace lane

// ---------------------------------------------------------------------------
// K2L: persistent, one CTA of kLaneWarps<KV0> warps per SM; every lane fetches
// scenario ids (warp-aggregated atomics on the launch's counter), heavy-first
// through p.order, and runs them one after another.
using lane::FULL_MASK;
template <bool KV0>
__global__ void __launch_bounds__(32 * kLaneWarps<KV0>, 1) bellman_lane_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) uint32_t lane_smem[];
  uint32_t lane_id;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane_id));
  uint32_t *smem = lane_smem + (threadIdx.x >> 5) * kLaneWarpWords<KV0> + lane_id;
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t *hist = p.lane_hist + (uint64_t)gt * kLaneHistWords;
  uint32_t *hist_warp = p.lane_hist + (uint64_t)(gt - lane_id) * kLaneHistWords;  // lane l's at + l x words
  uint2 *fifo_warp = p.lane_fifo + (uint64_t)(gt - lane_id) * 96u;  // lane l's ring at + 96 l
  const uint32_t kind = KV0 ? 3u : 4u;
  lane::Lane<KV0> L;
  bool has = false, alive = true;
  const uint32_t lt = (1u << lane_id) - 1u;
  // Every iteration starts with a warp-wide vote, so the 32 lanes reconverge
  // once per trip (otherwise lanes that finish a trip early run ahead into the
  // next one and the warp splits into groups that issue separately).  Lanes
  // without a scenario fetch one: warp-aggregated atomics on the counter.
  for (;;) {
    const uint32_t need = __ballot_sync(FULL_MASK, !has && alive);
    if (need) {
      uint32_t base = 0;
      if (lane_id == (uint32_t)__ffs((int)need) - 1u) base = atomicAdd(p.counter, (unsigned)__popc(need));
      base = __shfl_sync(FULL_MASK, base, __ffs((int)need) - 1);
      if (!has && alive) {
        const uint32_t kidx = base + (uint32_t)__popc(need & lt);
        if ((uint64_t)kidx >= p.count) {
          alive = false;
        } else {
          const uint64_t sid = p.order ? (uint64_t)p.order[kidx] : p.first + (uint64_t)kidx * p.stride;
          if (lane::mine(p, sid, kind)) {
            L.init(p, sid, smem, hist, fifo_warp + 96u * lane_id);
            has = true;
          }
        }
      }
    }
    if (!__any_sync(FULL_MASK, has || alive)) break;
    // generation: every lane whose FIFO is empty gets 32 candidates drawn by
    // the whole warp (one lane at a time); its head / next window covers the gap
    uint32_t want = __ballot_sync(FULL_MASK, has && !L.gen_done && L.fcnt == 0u);
    if (want) {
      const uint32_t w0 = want;
      while (want) {
        const uint32_t who = (uint32_t)__ffs((int)want) - 1u;
        want &= want - 1u;
        L.coop_refill(p, who, lane_id, fifo_warp);
      }
      if ((w0 >> lane_id) & 1u) L.after_refill(p);
    }
    bool fin = false;
    if (has && L.trip(p)) {
      L.finish_pre(p);
      fin = true;
    }
    // the finished lanes' histogram walks, by the whole warp, one lane at a time
    for (uint32_t fm = __ballot_sync(FULL_MASK, fin); fm; fm &= fm - 1u)
      L.coop_hists(p, (uint32_t)__ffs((int)fm) - 1u, lane_id, hist_warp);
    if (fin) {
      L.finish_post(p);
      has = false;
    }
  }
}

#ifdef BELLMAN_LANECHECK
// Development only: the same per-scenario code on the CPU (one scenario at a time).
void lane_host_run(const Params &p, uint64_t sid, uint32_t *smem_warp, uint32_t *hist, uint2 *fifo) {
  const bellman_profile &pr = p.profs[p.sc[sid].profile];
  if (pr.kv_ns_per_word == 0) {
    lane::Lane<true> L;
    L.init(p, sid, smem_warp, hist, fifo);
    do {
      if (!L.gen_done && L.fcnt == 0u) {
        L.fill_host(p);
        L.after_refill(p);
      }
    } while (!L.trip(p));
    L.finish_pre(p);
    L.scan_all(p);
    L.finish_post(p);
  } else {
    lane::Lane<false> L;
    L.init(p, sid, smem_warp, hist, fifo);
    do {
      if (!L.gen_done && L.fcnt == 0u) {
        L.fill_host(p);
        L.after_refill(p);
      }
    } while (!L.trip(p));
    L.finish_pre(p);
    L.scan_all(p);
    L.finish_post(p);
  }
}
#endif

}  // namespace bellman

int bellman_lane_grid(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return sms < (int)bellman::kLaneMaxCtas ? sms : (int)bellman::kLaneMaxCtas;
}

cudaError_t bellman_launch_lane(const bellman::Params &p, int grid, int kind, cudaStream_t stream) {
  using namespace bellman;
  if (kind == 3) {
    const size_t smem = sizeof(uint32_t) * kLaneWarpWords<true> * kLaneWarps<true>;
    static bool attr = false;
    if (!attr) {
      const cudaError_t e =
          cudaFuncSetAttribute(bellman_lane_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    bellman_lane_kernel<true><<<grid, 32 * kLaneWarps<true>, smem, stream>>>(p);
  } else {
    const size_t smem = sizeof(uint32_t) * kLaneWarpWords<false> * kLaneWarps<false>;
    static bool attr = false;
    if (!attr) {
      const cudaError_t e =
          cudaFuncSetAttribute(bellman_lane_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    bellman_lane_kernel<false><<<grid, 32 * kLaneWarps<false>, smem, stream>>>(p);
  }
  return cudaGetLastError();
}

/*
 * bellman_sim.h — C ABI of the B200-native beLLMan scenario simulator.
 *
 * The library simulates, for thousands to millions of independent scenarios,
 * an LLM serving node under the beLLMan output-length congestion controller
 * (arXiv 2510.15330).  It follows the paper's problem statement as SPEC.md
 * restates it: run_simulation(trace, server, models, controller?, seed) ->
 * RunResult, batched over scenarios.  Persistent sm_100a
 * kernels simulate one scenario per warp, or — for large runs of the
 * benchmark-path scenarios — one scenario per lane (bellman_sim_last_engines);
 * the records do not depend on the engine.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Rn = reading n in
 * DESIGN.md section 3.  Step names a1..a10 are DESIGN.md section 2.
 *
 * Conventions
 *  - All pointers in bellman_sim_desc are HOST pointers owned by the caller and
 *    only read during bellman_sim_create (deep copy into the workspace).
 *  - The workspace is DEVICE memory owned by the caller (e.g. a torch tensor),
 *    at least bellman_sim_workspace_bytes(desc) bytes, 256-byte aligned, and it
 *    must outlive the handle.  The library performs no cudaMalloc.
 *  - Functions taking `stream` are asynchronous and stream-ordered on that
 *    cudaStream_t (NULL = legacy default stream).
 *  - Errors: a non-zero bellman_status is returned and a message is kept in
 *    bellman_sim_last_error(sim) (or the thread-local global message when no
 *    handle exists).  No exception or abort crosses the ABI.  Per-scenario
 *    conditions (truncation, degenerate calibration) are FLAGS in the summary
 *    record, not errors.
 *  - A handle is single-writer: do not call into one handle from two threads.
 *  - Determinism: each summary record is a pure function of (desc, scenario id);
 *    it does not depend on device count, grid shape, stream or run order.
 */
#ifndef BELLMAN_SIM_H
#define BELLMAN_SIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror SPEC.md's exit codes (0 success, 1 validation,
 * 2 IO, 3 degenerate data) plus device/workspace/state errors. */
typedef enum {
  BELLMAN_OK = 0,
  BELLMAN_EINVAL = 1,      /* descriptor failed validation */
  BELLMAN_EIO = 2,         /* reserved (no file IO in the library) */
  BELLMAN_EDEGENERATE = 3, /* reserved: degenerate calibration is a per-scenario flag */
  BELLMAN_ECUDA = 4,       /* a CUDA runtime call or kernel launch failed */
  BELLMAN_EWORKSPACE = 5,  /* workspace NULL, misaligned or too small */
  BELLMAN_ESTATE = 6       /* call not valid in the handle's state / bad range */
} bellman_status;

enum { BELLMAN_LAW_OFF = 0, BELLMAN_LAW_CONST = 1, BELLMAN_LAW_MAP = 2, BELLMAN_LAW_STEP = 3 };
/* NEXT-3 laws after P:213 ("Toward novel LLM congestion control"; readings
 * R41-R43), each at one ingest per closed second:
 *  MPC — forecast the signal horizon_s seconds ahead from the window (mean +
 *        end-to-end slope) and choose, among {0} U rungs (or a 31-point grid of
 *        [r_min, r_max]), the r minimising
 *        w_lat max(0, F (1 - r) - t1) + w_q r + w_osc |r - r_prev|;
 *  BBR — TBT signal only: RTprop = minimum sample so far, BtlBw = maximum
 *        decode words per second over the window; congested iff the moving
 *        average >= RTprop + t1; at the bandwidth plateau (8 w >= 7 BtlBw) a
 *        congested controller raises r one step (step_bp or one rung), an
 *        uncongested one lowers it one step (to 0 below r_min), else it holds;
 *  PCC — while the moving average >= t1: paired one-second experiments
 *        r_base + step_bp then r_base - step_bp (clamped to [r_min, r_max]),
 *        each scored by the cost w_lat max(0, x - t1) + w_q r of the second it
 *        governed; after a pair r_base moves one step toward the cheaper. */
enum { BELLMAN_LAW_MPC = 4, BELLMAN_LAW_BBR = 5, BELLMAN_LAW_PCC = 6 };
/* Per-second congestion signals (a6).  TBT is the paper's; E2E / SLO
 * are SPEC's alternatives; TTFT, INPUT and UTIL are the further
 * signals P:211 names (NEXT-3): TTFT = mean TTFT of the second's first words;
 * INPUT = input words admitted to the engine in the second (its total);
 * UTIL = mean decode-batch occupancy over the second's iteration ends in basis
 * points, floor(10000 sum(B) / (max_batch n)).  A second without a sample of
 * the selected signal is a gap. */
enum {
  BELLMAN_SIG_TBT = 0,
  BELLMAN_SIG_E2E = 1,
  BELLMAN_SIG_SLO = 2,
  BELLMAN_SIG_TTFT = 3,
  BELLMAN_SIG_INPUT = 4,
  BELLMAN_SIG_UTIL = 5
};
enum { BELLMAN_MODE_CUTOFF = 0, BELLMAN_MODE_DRAIN = 1 };

/* summary flags */
#define BELLMAN_FLAG_TRUNCATED 0x1u        /* queued + in flight > 0 at the end */
#define BELLMAN_FLAG_DEGENERATE_CALIB 0x2u /* calibration had < 4 samples or t1 == t2 */
#define BELLMAN_FLAG_SERIES_OVERFLOW 0x4u  /* recorded signal series exceeded its capacity */
#define BELLMAN_FLAG_DONE 0x100u           /* record written by a run */
#define BELLMAN_NONE 0xFFFFFFFFu           /* "no value" in u32 percentile / second fields */

#define BELLMAN_TABLE_N 4096    /* quantile-table entries, indexed by (u32 >> 20) */
#define BELLMAN_HIST_LAT 896    /* latency bins: exact ms < 32, then 32 per octave */
#define BELLMAN_HIST_R 512      /* r bins of 10 bp */
#define BELLMAN_HIST_Q 201      /* similarity-score bins of 0.5 point (NEXT-2) */
#define BELLMAN_SEG_HIST_WORDS (2 * BELLMAN_HIST_LAT + BELLMAN_HIST_R + 2 * BELLMAN_HIST_Q) /* u64 per segment */
#define BELLMAN_MAX_BATCH 64

/* One knot of a piecewise-linear arrival-rate trace ("distinct phases when
 * the request arrivals ramp up, stay put, and ramp down"). */
typedef struct {
  int64_t t_us;      /* knot time, µs, non-decreasing within a trace */
  uint32_t lam_mrps; /* rate at the knot, milli-requests/s, <= 2^20 */
  uint32_t _pad;
} bellman_knot;

typedef struct {
  uint32_t knot_offset; /* kind 0: first knot in desc->knots; kind 1: first entry of desc->arrivals */
  uint32_t n_knots;     /* kind 0: knots, >= 2; kind 1: arrivals in the list */
  uint32_t arrival_cap; /* stop after this many arrivals; 0 = none */
  uint32_t kind;        /* 0: Poisson over the knots (a2); 1: replay of an explicit arrival list (NEXT-4) */
} bellman_trace;

/* One arrival of a replay trace (NEXT-4; SPEC's trace file S:29-34):
 * entries of a trace sorted by arrival; the per-request draws (a3) are keyed
 * by the entry's index in its trace. */
typedef struct {
  int64_t a_us;         /* arrival time, µs, >= 0 */
  uint32_t L_words;     /* natural (unbounded) output words, 1..65535 */
  uint32_t input_words; /* 1..65535 */
  uint32_t cls;         /* request class 0..3 (NEXT-3) */
  uint32_t _pad;
} bellman_arrival; /* 24 bytes */

/* Serving cost profile (decode law S:209-217; prefill S:218-226;
 * energy S:227-235; optional KV term, reading R2). */
typedef struct {
  uint32_t t0_us;               /* base decode iteration time, 1..2^24 */
  uint32_t knee;                /* batch size where slowdown begins, <= max_batch */
  uint32_t slope_us;            /* added µs per decoding request beyond the knee, <= 2^16 */
  uint32_t kv_ns_per_word;      /* ns per resident context word, <= 1024 (0 = SPEC's law) */
  uint32_t max_batch;           /* admission cap, 1..64 */
  uint32_t prefill_ns_per_word; /* prefill time per input word, <= 2^24 */
  /* NEXT-4 KV-capacity admission (S:255 lists KV modelling as
   * a SPEC non-goal): the queue head is admitted only if its whole context
   * (input + realized output words) fits beside the contexts of everything in
   * the system; strict FIFO; an oversized request runs alone.  0 = unlimited. */
  uint32_t kv_cap_words;        /* <= 2^30 */
  /* NEXT-4 prefill/decode contention (S:257 flags it as unmodelled): 0 =
   * SPEC's non-blocking prefill (a request's prefill occupies it for
   * prefill_time, others keep decoding); 1 = contending: the requests admitted
   * at an iteration boundary prefill inside the next iteration, which then
   * lasts cost(B) + sum of their prefill times (just the sum when nothing is
   * decoding, so S:207's idle-server example holds), and emit their first word
   * at its end. */
  uint32_t prefill_mode;
  /* NEXT-4 KV policy when kv_cap_words > 0: 0 = reserve (above: the whole
   * context input + R must fit at admission, so contexts never outgrow the
   * capacity); 1 = preempt (vLLM-style recompute preemption): the head is
   * admitted if its current context (input + words emitted so far) fits; at an
   * iteration end whose contexts exceed the capacity the latest admitted
   * requests go back to the front of the queue (while more than one is in the
   * system) and, re-admitted, prefill input + emitted again, that prefill's
   * end emitting their next word.  1 requires prefill_mode = 0. */
  uint32_t kv_policy;
  /* NEXT-4 token-level costs (S:249 tokens_per_word; reading R44): tokens per
   * word in Q16, 0 = the engine counts words (SPEC's model).  Nonzero (16384 ..
   * 262144, i.e. 0.25 .. 4): a request's input and realized output of w words
   * are clamp(floor((w tpw + 2^15) / 2^16), 1, 2^24) tokens; the engine decodes one
   * token per request per iteration (TBT gaps per token), and every per-unit
   * constant above and below (prefill and KV ns, KV capacity, energy, and the
   * words_in / words_out counters of the summary) is per token.  The rewrite
   * N and the similarity score stay in words.  Inputs must stay < 65536 tokens. */
  uint32_t tpw_q16;
  double e_in_j_per_word, e_out_j_per_word, p_idle_w;
  /* NEXT-4 multi-replica routing ("picks requests from the arrival
   * queue and assigns to GPU servers"; reading R45): `replicas` engines (0 or
   * 1 = one, <= 8) of max_batch slots each (replicas x max_batch <= 64) share
   * the FIFO arrival queue.  At an instant where some replica has no iteration
   * running, the arrived queue head is assigned to such a replica with a free
   * slot chosen by `route`: BELLMAN_ROUTE_LEAST (fewest requests in the
   * replica, ties to the lowest index) or BELLMAN_ROUTE_RR (the first at or
   * after a cyclic pointer, which then moves past it); each replica iterates
   * its own batch under the cost law above; every replica's words feed the
   * controller's signal; idle = the whole node empty.  replicas > 1 requires
   * prefill_mode 0 and kv_cap_words 0. */
  uint32_t replicas;
  uint32_t route;
} bellman_profile; /* 72 bytes */

#define BELLMAN_MAX_REPLICAS 8u
#define BELLMAN_ROUTE_LEAST 0u
#define BELLMAN_ROUTE_RR 1u

#define BELLMAN_PREFILL_NONBLOCKING 0u
#define BELLMAN_PREFILL_CONTENDING 1u
#define BELLMAN_KV_RESERVE 0u
#define BELLMAN_KV_PREEMPT 1u

/* Controller configuration (R3-R5, R22, R38). */
typedef struct {
  uint32_t law;        /* BELLMAN_LAW_* */
  uint32_t signal;     /* BELLMAN_SIG_*: avg TBT (default), avg E2E, SLO per-mille, avg TTFT, admitted
                          input words, batch occupancy bp (per second) */
  uint32_t window;     /* moving-average window in samples, 1..8 (5) */
  uint32_t r_min_bp;   /* MAP: r at t1 (5%) */
  uint32_t r_max_bp;   /* MAP: r at t2 (20%), <= 5000 */
  uint32_t r_const_bp; /* CONST: fixed r */
  uint32_t t1, t2;     /* thresholds in signal units (µs or per-mille), t1 < t2 unless calibrated */
  uint32_t slo_us;     /* SLO signal: E2E threshold */
  uint32_t calibrated; /* 1: t1/t2 = nearest-rank p50/p75 of the paired OFF run's series (a10) */
  uint32_t n_rungs;    /* 0 = continuous; else <= 8 ascending rungs, rung[0] = r_min, last = r_max */
  uint32_t rungs_bp[8];
  uint32_t bypass_mask;      /* NEXT-3 (S:267 class_policy): bit c -> class c never rewritten */
  uint32_t min_words_bypass; /* NEXT-3: predicted length below this never rewritten */
  uint32_t horizon_s;        /* NEXT-3 MPC: forecast horizon in seconds, <= 16 */
  uint32_t w_lat, w_q, w_osc;/* NEXT-3 MPC / PCC cost weights, <= 65535 (MPC and PCC need w_lat >= 1) */
  uint32_t step_bp;          /* NEXT-3 BBR (without rungs) step / PCC experiment delta, >= 1 */
} bellman_ctrl; /* 104 bytes */

/* Workload model inputs (R14, R15, R33): 4096-entry quantile
 * tables drawn with index (u32 >> 20), plus the compliance polynomial. */
typedef struct {
  const int32_t *L_words;  /* natural output words, 1..65535 */
  const int32_t *I_words;  /* input words, 1..65535 */
  const int32_t *fvar_q16; /* unbounded variability factor, Q16, 1..2^18 */
  const int32_t *noise;    /* predictor error in words, |.| <= 65535 */
  const int32_t *fcomp_q16;/* compliance factor, Q16, 0..2^18 */
  int64_t poly_q16[3];     /* realized = poly(N) * fcomp; identity = {0, 65536, 0}; |a_k| <= 2^40 */
  /* Quality model (NEXT-2): every admitted request is
   * scored against its unbounded length U: reduction red = (U - R) / U;
   * inactive (r = 0): base = quality[0]; active: quality[1] for red <=
   * quality[3] bp, quality[2] for red >= quality[4] bp, linear in between
   * (floored); score = clamp(base + qnoise[u >> 20], 0, 10000) centi-points,
   * u = 4th word of the request's tag-1 Philox block. */
  const int32_t *qnoise;   /* centi-points, |.| <= 2047 */
  uint32_t quality[5];     /* inactive, active, floor (centi-points), safe_bp, end_bp */
  /* Request classes (NEXT-3): class = first c with x < class_cum[c], x =
   * the 20 low bits of the candidate's 3rd Philox word (its top 12 bits draw L);
   * non-decreasing, class_cum[3] = 2^20.  One class: all 2^20. */
  uint32_t class_cum[4];
  uint32_t _pad[3];
} bellman_models;

typedef struct {
  uint32_t seed_index; /* Philox key = (seed_index, 0xB311A000) */
  uint32_t trace;      /* index into traces */
  uint64_t wid;        /* workload id: Philox counter words 2,3 (ON/OFF pairs share it) */
  uint32_t profile, ctrl, segment, mode; /* mode: BELLMAN_MODE_* */
  int64_t horizon_us;  /* cutoff H, or the cap of a drain run */
  int64_t w0_us, w1_us;/* window [w0, w1) for the win_* counters (130-500 s) */
  uint32_t calib_src;  /* OFF scenario whose series calibrates this one, or BELLMAN_NONE */
  uint32_t record;     /* bit 0: keep the per-second signal series (a10 source);
                          bit 1: debug record mode — per-second rows + controller log (NEXT-1) */
} bellman_scenario; /* 64 bytes */

#define BELLMAN_RECORD_SIGNAL 0x1u
#define BELLMAN_RECORD_SECONDS 0x2u

/* Per-second aggregate of a debug-recorded scenario.
 * Attribution: arrivals to their arrival second, queueing and input
 * words to the admission second, TTFT and first words to the first-token
 * second, decode words and their TBT gaps to the emission second, E2E to the
 * completion second, idle time split over the seconds it overlaps.  Rows cover
 * seconds 0 .. floor(end_us / 1e6). */
typedef struct {
  uint32_t arrivals, admitted, first_tokens, completions, tbt_count, idle_us, words_in, words_out;
  uint64_t sum_queue_us, sum_ttft_us, sum_e2e_us, sum_tbt_us;
} bellman_second_row; /* 64 bytes */

/* One controller ingest ("second, ma_tbt_ms, r, active"): the moving
 * average is A / k over the last k samples; r and active after the update. */
typedef struct {
  uint32_t second, sample, k, r_bp, active, _pad;
  uint64_t A;
} bellman_ctrl_row; /* 32 bytes */

typedef struct {
  const bellman_knot *knots;
  uint32_t n_knots;
  const bellman_trace *traces;
  uint32_t n_traces;
  const bellman_profile *profiles;
  uint32_t n_profiles;
  const bellman_ctrl *ctrls;
  uint32_t n_ctrls;
  bellman_models models;
  const bellman_scenario *scenarios;
  uint64_t n_scenarios;
  uint32_t n_segments; /* segment ids in [0, n_segments) */
  uint32_t _pad;
  const bellman_arrival *arrivals; /* replay lists of kind-1 traces (may be NULL if none) */
  uint64_t n_arrivals;
} bellman_sim_desc;

/* 272-byte per-scenario summary (a8, a9, a6 logs).  All counts are exact
 * integers; energy_j = (e_in*words_in + e_out*words_out) + p_idle*idle_us/1e6. */
typedef struct {
  uint64_t scenario_id, ticks, candidates, arrivals, admitted, served, rewritten;
  uint64_t words_in, words_out, idle_us, end_us, queued_end, inflight_end;
  uint64_t win_served, win_words_in, win_words_out, win_idle_us;
  uint64_t sum_queue_us, sum_ttft_us, sum_e2e_us, slo_violations;
  uint32_t e2e_p50_ms, e2e_p99_ms, ttft_p50_ms, ttft_p99_ms, median_r_bp;
  uint32_t t1, t2, activations, first_act_s, last_deact_s, active_ingests, flags;
  uint32_t segment;
  uint32_t bypassed; /* NEXT-3: admissions while r > 0 that a bypass rule left unrewritten */
  double energy_j, win_energy_j;
  /* NEXT-2: nearest-rank median similarity (0.5-point bin lower edge, centi-points)
   * of rewritten (active) and not rewritten (inactive) admissions, and their counts */
  uint32_t sim_active_p50, sim_inactive_p50, scored_active, scored_inactive;
  /* NEXT-4 kv_policy 1: requests sent back to the queue, and the context words
   * prefilled again at their re-admissions (part of words_in).  admitted counts
   * first admissions; inflight_end counts admitted, unfinished requests
   * (preempted ones waiting included); sum_queue_us sums every queue stay. */
  uint32_t preemptions, _pad2;
  uint64_t recompute_words;
} bellman_scenario_stats;

typedef struct bellman_sim bellman_sim; /* opaque */

/* Bytes of device workspace the descriptor needs (0 if desc fails validation;
 * see bellman_sim_last_error(NULL)). */
size_t bellman_sim_workspace_bytes(const bellman_sim_desc *desc);

/* Validate desc, lay out and fill the workspace (H2D copies on `stream`),
 * bind to `device`.  *out receives the handle. */
bellman_status bellman_sim_create(const bellman_sim_desc *desc, void *workspace, size_t workspace_bytes,
                                  int device, void *stream, bellman_sim **out);

/* Simulate scenarios first, first+stride, ..., first+(count-1)*stride
 * (interleaved sharding across ranks: first = rank, stride = world size).
 * Calibrated scenarios (a10) need their source in the same set.  Launches the
 * pass-1 kernel, then (if any calibrated scenario is in the set) the
 * calibration kernel and the pass-2 kernel.  Every run hands its scenarios to
 * warps in decreasing order of expected arrivals (heavy first, for load
 * balance; a shard's order is the whole set's order filtered to the shard,
 * uploaded into the workspace on the first run of each distinct
 * (first, stride, count)); results never depend on that order.  Asynchronous. */
bellman_status bellman_sim_run(bellman_sim *sim, uint64_t first, uint64_t count, uint64_t stride,
                               void *stream);

/* Copy `count` summary records of scenario ids [first, first+count) to dst
 * (device or host memory).  Asynchronous for device dst; synchronous on
 * `stream` for host dst. */
bellman_status bellman_sim_stats(bellman_sim *sim, bellman_scenario_stats *dst, uint64_t first,
                                 uint64_t count, int dst_is_device, void *stream);

/* Copy the `count` summary records of scenario ids first, first+stride, ...,
 * first+(count-1)*stride (a rank's interleaved shard) to dst, packed densely
 * (record k of dst = scenario first + k*stride).  One strided copy; same
 * synchronisation as bellman_sim_stats.  BELLMAN_ESTATE if the range leaves
 * [0, n_scenarios) or stride is 0. */
bellman_status bellman_sim_stats_strided(bellman_sim *sim, bellman_scenario_stats *dst, uint64_t first,
                                         uint64_t count, uint64_t stride, int dst_is_device, void *stream);

/* Copy the per-segment histograms, n_segments x BELLMAN_SEG_HIST_WORDS uint64:
 * [E2E 896 | TTFT 896 | r 512 | similarity active 201 | inactive 201] integer
 * counts merged over the segment's runs. */
bellman_status bellman_sim_segment_hist(bellman_sim *sim, uint64_t *dst, int dst_is_device, void *stream);

/* Debug record mode (scenario.record & BELLMAN_RECORD_SECONDS): copy the
 * per-second rows and the controller log of scenario `id` to HOST buffers
 * (synchronous on `stream`).  *n_rows / *n_ctrl receive the counts written by
 * the last run (rows beyond cap are dropped).  BELLMAN_ESTATE if the scenario
 * is not debug-recorded. */
bellman_status bellman_sim_series(bellman_sim *sim, uint64_t id, bellman_second_row *rows, uint64_t cap_rows,
                                  uint64_t *n_rows, bellman_ctrl_row *ctrl, uint64_t cap_ctrl, uint64_t *n_ctrl,
                                  void *stream);

/* Zero all summary records, segment histograms and recorded series. */
bellman_status bellman_sim_reset(bellman_sim *sim, void *stream);

/* ---- Fused summary exchange over peer memory ----------
 * The one exchange step of a sharded run is an all-gather of the summary
 * records (every rank ends with all n_scenarios records).  Instead of a
 * separate collective after the kernel, the tick kernel can store every record
 * it finishes, as it finishes it, into up to BELLMAN_MAX_PEERS full-size record
 * arrays — one per rank, the caller's own included — that the caller has
 * mapped into this process (CUDA IPC over NVLink / NVSwitch, or a local device
 * pointer), at the record's scenario index.  The transfer then overlaps the
 * simulation scenario by scenario; after every rank's run has completed (the
 * caller's stream synchronised and a host barrier), every array holds every
 * record of every rank's shard.  Records are identical to bellman_sim_stats'
 * (the local workspace copy is still written). */
#define BELLMAN_MAX_PEERS 8

/* Export a device allocation for peer mapping: *handle (64 bytes, caller-owned
 * host memory) receives the CUDA IPC handle of the allocation containing
 * dev_ptr and *offset the byte offset of dev_ptr inside it.  Synchronous.
 * BELLMAN_EINVAL on NULL arguments, BELLMAN_ECUDA if CUDA refuses. */
bellman_status bellman_ipc_export(const void *dev_ptr, void *handle, uint64_t *offset);

/* Map a peer allocation exported by bellman_ipc_export in another process
 * (any device of this node with peer access; same device allowed) into this
 * process on `device`: *base receives the mapping (for bellman_ipc_close) and
 * *dev_ptr = base + offset.  Synchronous. */
bellman_status bellman_ipc_open(const void *handle, uint64_t offset, int device, void **base, void **dev_ptr);

/* Unmap a mapping returned by bellman_ipc_open (its `base`). */
bellman_status bellman_ipc_close(void *base);

/* Set the peer record arrays of later runs: peer_stats[0..n_peers) are device
 * pointers valid in this process, each to n_scenarios bellman_scenario_stats;
 * n_peers = 0 turns the fused exchange off.  Pointers are borrowed (caller-
 * owned, must outlive the runs).  BELLMAN_EINVAL if n_peers > BELLMAN_MAX_PEERS
 * or a pointer is NULL or not 16-byte aligned. */
bellman_status bellman_sim_set_peers(bellman_sim *sim, void *const *peer_stats, uint32_t n_peers);

/* Kernel launches issued by the most recent bellman_sim_run. */
uint32_t bellman_sim_last_launches(const bellman_sim *sim);

/* Which engines the most recent bellman_sim_run launched, as a bit mask over
 * BELLMAN_ENGINE_*: the warp-per-scenario kernels (one warp simulates one
 * scenario: the TBT-specialised, generic and multi-replica loops) and the
 * lane-per-scenario kernel K2L (one thread simulates one scenario; DESIGN.md
 * §5).  The results never depend on the engine: every engine computes the
 * same records.  A run takes K2L for the scenarios within its bounds (TBT
 * signal, non-blocking prefill, no KV capacity, word units, one replica,
 * MAP / STEP / CONST / OFF, a Poisson trace, horizon < 2^31 µs) when it has at
 * least 65,536 scenarios; the environment variable BELLMAN_LANE=0 turns K2L
 * off, BELLMAN_LANE=2 takes it for runs of any size (read at every call). */
#define BELLMAN_ENGINE_WARP_TBT 0x1u   /* warp per scenario, TBT-specialised loop */
#define BELLMAN_ENGINE_WARP_GEN 0x2u   /* warp per scenario, generic loop */
#define BELLMAN_ENGINE_WARP_MULTI 0x4u /* warp per scenario, multi-replica loop */
#define BELLMAN_ENGINE_LANE_KV0 0x8u   /* lane per scenario, KV-free cost law */
#define BELLMAN_ENGINE_LANE_KV 0x10u   /* lane per scenario, with the KV term */
uint32_t bellman_sim_last_engines(const bellman_sim *sim);

void bellman_sim_destroy(bellman_sim *sim);
const char *bellman_status_string(bellman_status s);
const char *bellman_sim_last_error(const bellman_sim *sim);

#ifdef __cplusplus
}
#endif
#endif /* BELLMAN_SIM_H */

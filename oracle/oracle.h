/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the beLLMan scenario
 * simulation (arXiv 2510.15330).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_2510_15330_b200/); both take their inputs from workloads/.
 *
 * Structure (deliberately unlike the GPU kernel): all arrivals are generated up
 * front into an array; a binary heap of typed events drives a textbook
 * discrete-event simulation; per-request structs; an explicit FIFO queue; the
 * per-second signal series is kept in full and the moving average recomputed
 * from it at every ingest.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * Rn = reading n in DESIGN.md §3 (== SURVEY.md §8(c).2).
 *
 * Parity pins (tests/test_oracle_*.py): Random123 KATs (Philox), libm -log
 * (neglog), Decimal log2 table, SPEC worked examples, hand fixtures F1-F6
 * (tests/golden/), a brute-force microsecond-stepping simulator on tiny
 * traces, M/D/1 Pollaczek-Khinchine, the uncongested-regime bound, the
 * sample-path Little's law identity, controller law vs exact rationals;
 * round 2: hand-worked controller sequences for STEP / MAP / MPC / BBR / PCC
 * (tests/golden/controller_sequences.json), E2E / SLO signals and the
 * transition log recomputed from the request / controller logs, histogram
 * percentiles bracketing the exact nearest-rank values, token costs (S:207 in
 * tokens, identities), multi-replica routing (one replica == orc_simulate, a
 * hand-worked two-replica timeline, brute force), the A3 saturation brackets.
 * "parity unpinned": the paper's directional outcomes (A4) and the exact
 * saturation capacity of P24/L8B (calibration outputs), see DESIGN.md §6.
 */
#ifndef BELLMAN_ORACLE_H
#define BELLMAN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_LAW_OFF = 0, ORC_LAW_CONST = 1, ORC_LAW_MAP = 2, ORC_LAW_STEP = 3 };
/* NEXT-3 laws after P:213 ("Toward novel LLM congestion control"), readings in
 * DESIGN.md §3 (R41-R43): MPC — forecast the signal over a horizon and pick the
 * r minimising latency + quality/energy + oscillation cost; BBR — operate at
 * Kleinrock's point from the minimum TBT and the maximum delivered words/s;
 * PCC — paired micro-experiments r_base +- delta scored by a utility of
 * latency and quality. */
enum { ORC_LAW_MPC = 4, ORC_LAW_BBR = 5, ORC_LAW_PCC = 6 };
/* INPUT and UTIL (NEXT-3, "input tokens per unit time", "GPU utilization
 * metrics"): input words admitted in the second (the second's total); mean
 * decode-batch occupancy over the second's iteration ends in basis points,
 * floor(10000 sum(B) / (max_batch n)). */
enum { ORC_SIG_TBT = 0, ORC_SIG_E2E = 1, ORC_SIG_SLO = 2, ORC_SIG_TTFT = 3, ORC_SIG_INPUT = 4, ORC_SIG_UTIL = 5 };
enum { ORC_MODE_CUTOFF = 0, ORC_MODE_DRAIN = 1 };
enum { ORC_FLAG_TRUNCATED = 1, ORC_FLAG_DEGENERATE_CALIB = 2 };

#define ORC_NONE 0xFFFFFFFFu
#define ORC_HIST_LAT 896 /* log-linear ms bins, 32 per octave (a9) */
#define ORC_HIST_R 512   /* 10 bp bins of r */
#define ORC_HIST_Q 201   /* similarity-score bins of 0.5 point (NEXT-2) */

/* ---- column inputs, exactly as workloads.Workload.columns() builds them ---- */
typedef struct {
  const int64_t *knot_t;
  const uint32_t *knot_lam;
  const uint32_t *trace_knot_off, *trace_n_knots, *trace_cap;
  const uint32_t *trace_kind; /* 0 Poisson over knots, 1 replay of an explicit arrival list (NEXT-4) */
  const int64_t *arr_a;       /* replay lists: arrival µs, L, input words, class */
  const uint32_t *arr_L, *arr_input, *arr_cls;
  const uint32_t *prof_t0, *prof_knee, *prof_slope, *prof_kv, *prof_maxb, *prof_prefill_ns;
  const uint32_t *prof_kv_cap; /* NEXT-4: KV capacity in context words, 0 = unlimited */
  const uint32_t *prof_prefill_mode; /* NEXT-4: 0 non-blocking prefill, 1 contending */
  const uint32_t *prof_kv_policy;    /* NEXT-4: 0 reserve whole contexts, 1 preempt on overflow */
  const uint32_t *prof_tpw;          /* NEXT-4: tokens per word Q16 (0 = the engine counts words) */
  const uint32_t *prof_replicas, *prof_route; /* NEXT-4 multi-replica routing (R45) */
  const double *prof_e_in, *prof_e_out, *prof_p_idle;
  const uint32_t *ctrl_law, *ctrl_signal, *ctrl_window, *ctrl_rmin, *ctrl_rmax, *ctrl_rconst;
  const uint32_t *ctrl_t1, *ctrl_t2, *ctrl_slo_us, *ctrl_calibrated, *ctrl_nrungs;
  const uint32_t *ctrl_rungs; /* [n_ctrl][8] */
  const uint32_t *ctrl_bypass_mask, *ctrl_min_words; /* NEXT-3 class / short-output bypass */
  const uint32_t *ctrl_horizon, *ctrl_wlat, *ctrl_wq, *ctrl_wosc, *ctrl_step; /* NEXT-3 MPC / BBR / PCC */
  const int32_t *tab_L, *tab_I, *tab_fvar, *tab_noise, *tab_fcomp; /* [4096] each */
  const int64_t *poly_q16;                                          /* [3] */
  const int32_t *tab_qnoise;  /* [4096] similarity noise, centi-points (NEXT-2) */
  const uint32_t *quality;    /* [5] inactive, active, floor (centi-points), safe, end (bp) */
  const uint32_t *class_cum;  /* [4] cumulative class thresholds in 2^-20 units (NEXT-3) */
  const uint32_t *sc_seed;
  const uint64_t *sc_wid;
  const uint32_t *sc_trace, *sc_profile, *sc_ctrl, *sc_segment, *sc_mode;
  const int64_t *sc_horizon, *sc_w0, *sc_w1;
  const uint32_t *sc_calib_src, *sc_record;
  uint64_t n_scenarios;
} orc_inputs;

/* One accepted arrival with its per-request model draws (a2, a3). */
typedef struct {
  uint64_t a_us;       /* arrival time */
  uint32_t j;          /* candidate index (Philox counter word 0) */
  uint32_t L;          /* natural (median) unbounded output words */
  uint32_t input;      /* input words */
  uint32_t U;          /* realized unbounded output words */
  uint32_t P;          /* predicted output words */
  int32_t fcomp_q16;   /* compliance factor */
  int32_t qnoise;      /* similarity-score noise, centi-points (NEXT-2) */
  uint32_t cls;        /* request class 0..3 (NEXT-3) */
} orc_request;

typedef struct {
  uint32_t t0_us, knee, slope_us, kv_ns_per_word, max_batch, prefill_ns_per_word;
  double e_in, e_out, p_idle;
  uint32_t kv_cap_words; /* NEXT-4 KV-capacity admission, 0 = unlimited */
  uint32_t prefill_mode; /* NEXT-4: 0 non-blocking; 1 contending: the requests admitted
                            at an iteration boundary prefill inside the next iteration */
  uint32_t kv_policy;    /* NEXT-4 with kv_cap_words > 0: 0 reserve (admit only whole contexts
                            input + R), 1 preempt (admit on the current context input + emitted;
                            at an iteration end whose contexts exceed the capacity, the latest
                            admitted requests go back to the queue front and later recompute) */
  uint32_t tpw_q16;      /* NEXT-4 token-level costs (R44): tokens per word in Q16; 0 = words.
                            Nonzero: inputs and realized outputs are converted to tokens
                            (max(1, round(w tpw))), the engine decodes one token per request per
                            iteration, and every per-unit constant is per token */
  uint32_t replicas;     /* NEXT-4 (R45): engines sharing the arrival queue, 0/1 = one; max_batch each */
  uint32_t route;        /* NEXT-4 (R45): ORC_ROUTE_LEAST (fewest in the replica) or ORC_ROUTE_RR */
} orc_profile;

#define ORC_MAX_REPLICAS 8
enum { ORC_ROUTE_LEAST = 0, ORC_ROUTE_RR = 1 };

typedef struct {
  uint32_t law, signal, window, r_min_bp, r_max_bp, r_const_bp, t1, t2, slo_us, calibrated, n_rungs;
  uint32_t rungs_bp[8];
  uint32_t bypass_mask;      /* bit c: class c is never rewritten (S:267 class_policy) */
  uint32_t min_words_bypass; /* predicted length below this is never rewritten */
  /* NEXT-3: MPC forecast horizon in seconds and cost weights (latency
   * excess per µs, quality/energy per bp of r, oscillation per bp of |dr|);
   * PCC utility weights w_lat, w_q; BBR / PCC step in bp */
  uint32_t horizon_s, w_lat, w_q, w_osc, step_bp;
} orc_ctrl;

typedef struct {
  uint32_t mode;
  int64_t horizon_us, w0_us, w1_us;
  int64_t poly_q16[3];
  uint32_t quality[5]; /* similarity model (NEXT-2): inactive, active, floor, safe_bp, end_bp */
  uint32_t record; /* bit 0: keep the per-second signal series; bit 1: per-second rows */
} orc_run_cfg;

typedef struct {
  uint64_t ticks, candidates, arrivals, admitted, served, rewritten;
  uint64_t words_in, words_out, idle_us, end_us, queued_end, inflight_end;
  uint64_t win_served, win_words_in, win_words_out, win_idle_us;
  uint64_t sum_queue_us, sum_ttft_us, sum_e2e_us, slo_violations;
  uint32_t e2e_p50_ms, e2e_p99_ms, ttft_p50_ms, ttft_p99_ms, median_r_bp;
  uint32_t t1, t2, activations, first_act_s, last_deact_s, active_ingests, flags;
  double energy_j, win_energy_j;
  uint32_t sim_active_p50, sim_inactive_p50, scored_active, scored_inactive; /* NEXT-2, centi-points */
  uint32_t bypassed; /* NEXT-3: admissions while r > 0 left unrewritten by a bypass rule */
  uint32_t preemptions;     /* NEXT-4 kv_policy 1: requests sent back to the queue */
  uint64_t recompute_words; /* NEXT-4 kv_policy 1: context words prefilled again at re-admission */
  /* ---- self-checks the GPU never computes ---- */
  uint64_t e2e_exact_p50_us, e2e_exact_p99_us, ttft_exact_p50_us, ttft_exact_p99_us;
  uint64_t int_system_us;  /* integral of (queued + in_system) dt, µs*requests */
  uint64_t int_queue_us;   /* integral of queued dt */
  uint64_t sum_sojourn_us; /* sum over completed of (completion - arrival) */
  uint64_t tbt_samples, tbt_sum_us, tbt_max_us;
  uint32_t hist_e2e[ORC_HIST_LAT], hist_ttft[ORC_HIST_LAT], hist_r[ORC_HIST_R];
  uint32_t hist_q_active[ORC_HIST_Q], hist_q_inactive[ORC_HIST_Q];
  uint32_t n_series; /* per-second signal samples written to series[] (record mode) */
} orc_result;

/* Optional per-request / per-gap / controller trace for hand fixtures. */
typedef struct {
  uint64_t admit_us, first_us, done_us; /* UINT64_MAX if the event did not happen */
  uint32_t R, r_bp, n_gaps, _pad;
} orc_req_log;

typedef struct {
  uint32_t second, sample, k, r_bp, active, _pad;
  uint64_t A;
} orc_ctrl_log;

/* Per-second aggregate (NEXT-1; attribution S:382): each
 * event counts toward the second of its own timestamp. */
typedef struct {
  uint32_t arrivals;     /* arrivals in the second (rps_in) */
  uint32_t admitted;     /* admissions (queueing attributed to the admission second) */
  uint32_t first_tokens; /* first words (TTFT attributed to the first-token second) */
  uint32_t completions;  /* completions (E2E attributed to the completion second) */
  uint32_t tbt_count;    /* decode words emitted (TBT samples) */
  uint32_t idle_us;      /* time in the second with nothing in the system */
  uint32_t words_in;     /* input words admitted */
  uint32_t words_out;    /* words emitted (first + decode) */
  uint64_t sum_queue_us, sum_ttft_us, sum_e2e_us, sum_tbt_us;
} orc_second_row;

typedef struct {
  orc_req_log *req;    /* [n_requests] or NULL */
  uint64_t *gaps;      /* pairs (request index, gap µs), capacity cap_gaps pairs, or NULL */
  uint64_t cap_gaps, n_gaps;
  orc_ctrl_log *ctrl;  /* capacity cap_ctrl or NULL */
  uint64_t cap_ctrl, n_ctrl;
  uint32_t *series;    /* per-second samples (record mode), capacity cap_series */
  uint64_t cap_series;
  orc_second_row *rows; /* per-second rows (record & 2), capacity cap_rows */
  uint64_t cap_rows, n_rows;
} orc_log;

/* Philox4x32-10 (Salmon et al., SC'11), key = (k0, k1), counter c[4]. */
void orc_philox(uint32_t k0, uint32_t k1, const uint32_t ctr[4], uint32_t out[4]);
/* -ln(U) in Q32 for U = (2u+1)/2^33 (reading R33). */
uint64_t orc_neglog_q32(uint32_t u);
/* round(2^32 log2(1 + i/4096)), i = 0..4096 (reading R33). */
uint64_t orc_log2_table(uint32_t i);
/* latency bin of a value in ms, and the lower edge of a bin (a9). */
uint32_t orc_lat_bin(uint64_t ms);
uint64_t orc_lat_edge(uint32_t bin);

/* Generate the accepted arrivals of scenario sid (a2 + a3); returns the count
 * (all of them up to the trace end / arrival cap), or -1 on allocation failure.
 * If out is NULL only counts. */
int64_t orc_arrivals(const orc_inputs *in, uint64_t sid, orc_request *out, uint64_t cap_out);

/* The discrete-event simulation (a4-a9) over an explicit request list. */
int orc_simulate(const orc_request *req, uint64_t n_req, const orc_profile *prof,
                 const orc_ctrl *ctrl, const orc_run_cfg *cfg, orc_result *res, orc_log *log);

/* NEXT-4 multi-replica routing (R45): the same DES over prof->replicas engines
 * sharing one arrival queue (orc_simulate dispatches here for replicas > 1;
 * callable directly for any replica count, which pins one replica against
 * orc_simulate).  Returns -1 for more than ORC_MAX_REPLICAS, contending
 * prefill or a KV capacity. */
int orc_simulate_replicas(const orc_request *req, uint64_t n_req, const orc_profile *prof,
                          const orc_ctrl *ctrl, const orc_run_cfg *cfg, orc_result *res, orc_log *log);

/* Full scenario: arrivals + (calibration pass a10) + simulation.  With
 * log->ctrl / log->rows given, the controller log and (record & 2) the
 * per-second rows are written. */
int orc_run_scenario(const orc_inputs *in, uint64_t sid, orc_result *res, orc_log *log);

/* Nearest-rank percentile of a sample list, 0 < p <= 100 (p = 0 -> min). */
uint32_t orc_percentile_u32(const uint32_t *v, uint64_t n, uint32_t p);

/* Threshold calibration (a10): 0 ok, 1 insufficient, 2 degenerate. */
int orc_calibrate(const uint32_t *series, uint64_t n, uint32_t *t1, uint32_t *t2);

/* Similarity score (NEXT-2) in centi-points for a request whose
 * unbounded length is U and realized length R, rewritten (active) or not. */
uint32_t orc_similarity(uint32_t U, uint32_t R, int active, int32_t noise, const uint32_t q[5]);

/* Controller law as a pure function (a6): r in bp for a window sum A over k samples. */
uint32_t orc_map_rate(uint64_t A, uint32_t k, const orc_ctrl *c);

/* The controller alone (a6, every law): ingest n per-second samples x[i] of
 * seconds sec[i] (w[i] = decode words emitted in that second, BBR's delivery
 * rate), starting from the initial state; log[i] receives the state after
 * ingest i, and res the transition log (activations, first_act_s,
 * last_deact_s, active_ingests).  Returns 0, or -1 on allocation failure. */
int orc_ctrl_trace(const orc_ctrl *c, const uint32_t *sec, const uint32_t *x, const uint32_t *w, uint64_t n,
                   orc_result *res, orc_ctrl_log *log);

/* Run many scenarios on nthreads host threads (cpu baseline). Returns 0 on success. */
int orc_run_batch(const orc_inputs *in, const uint64_t *sids, uint64_t n, orc_result *res, int nthreads);

#ifdef __cplusplus
}
#endif
#endif

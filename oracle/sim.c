/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A textbook discrete-event simulation of one LLM serving node under the
 * beLLMan controller (a4-a10).  Times are integer microseconds.
 *
 * Serving model (SPEC serving_sim, readings R6-R9, R18-R21):
 *  - continuous batching: "one global iteration loop; each iteration all active
 *    requests emit one word; new requests admitted between iterations FIFO up
 *    to max_batch; a request's prefill occupies it for prefill_time before its
 *    first decode step but does not block others";
 *  - decode iteration time t0 + slope*max(0, B - knee) + the optional
 *    KV term floor(kv_ns_per_word * K / 1000) (reading R2);
 *  - prefill time prefill_ns_per_word * input / 1000, at least 1 µs;
 *  - first word at prefill end; TBT = inter-token gaps (R6);
 *  - a request admitted while the loop runs joins at the next boundary (R6);
 *  - admission points: every event instant at which the loop is idle (an
 *    iteration end makes it idle); arrivals <= T are eligible (R7);
 *  - simultaneous events: iteration end, prefill ends (by j), arrivals (by j),
 *    then ingest, admission, iteration start (R7).
 * Controller (R3-R5, R12, R21, R38): the per-second
 * signal sample is ingested at each admission point for every closed second;
 * moving average over the last `window` samples; active iff MA >= t1; the
 * linear law maps MA in [t1, t2] to r in [r_min, r_max]; ladders floor it to a
 * rung; STEP climbs a rung per ingest while active.  Rewrite at admission:
 * N = round(P (1 - r)), realized = round(poly(N) * Fcomp).
 * Energy: e_in * words_in + e_out * words_out + p_idle * idle.
 * NEXT-4 KV capacity (S:255 leaves KV out of SPEC): kv_policy 0
 * admits the queue head only if its whole context input + R fits beside the
 * reserved contexts; kv_policy 1 (vLLM-style recompute preemption) admits on
 * the current context input + emitted, and at an iteration end whose contexts
 * exceed the capacity sends the latest admitted requests (one at a time, while
 * more than one is in the system) back to the front of the queue, in front of
 * earlier victims; a re-admitted request prefills its whole context again and
 * that prefill's end emits its next word (a decode word, TBT gap from its last).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define US 1000000ull
#define NEVER UINT64_MAX

enum { EV_ITER_END = 0, EV_PREFILL_END = 1, EV_ARRIVAL = 2 };
enum { RS_FUTURE = 0, RS_QUEUED, RS_PREFILL, RS_READY, RS_DECODING, RS_DONE, RS_PENDING };

typedef struct {
  uint64_t t;
  uint32_t kind, idx;
  uint32_t gen; /* prefill ends: the request's admission generation (stale after a preemption) */
} event;

typedef struct {
  event *v;
  uint64_t n, cap;
} heap;

static int ev_less(const event *a, const event *b) {
  if (a->t != b->t) return a->t < b->t;
  if (a->kind != b->kind) return a->kind < b->kind;
  return a->idx < b->idx;
}

static int heap_push(heap *h, event e) {
  if (h->n == h->cap) {
    uint64_t nc = h->cap ? 2 * h->cap : 64;
    event *nv = (event *)realloc(h->v, nc * sizeof(event));
    if (!nv) return -1;
    h->v = nv;
    h->cap = nc;
  }
  uint64_t i = h->n++;
  h->v[i] = e;
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (!ev_less(&h->v[i], &h->v[p])) break;
    event t = h->v[i]; h->v[i] = h->v[p]; h->v[p] = t;
    i = p;
  }
  return 0;
}

static event heap_pop(heap *h) {
  event top = h->v[0];
  h->v[0] = h->v[--h->n];
  uint64_t i = 0;
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && ev_less(&h->v[l], &h->v[m])) m = l;
    if (r < h->n && ev_less(&h->v[r], &h->v[m])) m = r;
    if (m == i) break;
    event t = h->v[i]; h->v[i] = h->v[m]; h->v[m] = t;
    i = m;
  }
  return top;
}

/* ---------------------------------------------------------------------------
 * latency histogram bins (a9): integer ms, 32 log-linear sub-buckets per
 * octave.  Bin b < 32 holds exactly b ms; above, bin 32(e-4)+s holds
 * [(32+s) 2^(e-5), (33+s) 2^(e-5)).  The bin of a value is found by search
 * over the edges (the definition), not by bit tricks.
 * ------------------------------------------------------------------------- */
uint64_t orc_lat_edge(uint32_t b) {
  if (b < 32) return b;
  uint32_t e = b / 32 + 4, s = b % 32;
  return (uint64_t)(32 + s) << (e - 5);
}

uint32_t orc_lat_bin(uint64_t ms) {
  uint32_t lo = 0, hi = ORC_HIST_LAT - 1; /* largest b with edge(b) <= ms */
  if (ms >= orc_lat_edge(hi)) return hi;
  while (lo < hi) {
    uint32_t mid = (lo + hi + 1) / 2;
    if (orc_lat_edge(mid) <= ms) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/* nearest-rank percentile (R13): rank k = max(1, ceil(p n / 100)) */
static uint64_t nr_rank(uint64_t n, uint32_t p) {
  uint64_t k = (p * n + 99) / 100;
  return k < 1 ? 1 : k;
}

static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return x < y ? -1 : x > y;
}
static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : x > y;
}

uint32_t orc_percentile_u32(const uint32_t *v, uint64_t n, uint32_t p) {
  if (n == 0) return ORC_NONE;
  uint32_t *s = (uint32_t *)malloc(n * sizeof(uint32_t));
  if (!s) return ORC_NONE;
  memcpy(s, v, n * sizeof(uint32_t));
  qsort(s, n, sizeof(uint32_t), cmp_u32);
  uint32_t r = p == 0 ? s[0] : s[nr_rank(n, p) - 1];
  free(s);
  return r;
}

/* a10 — "We pick the median TBT (T1) during the unbounded run ... and the 75th
 * percentile TBT (T2)"; >= 4 samples, t1 != t2. */
int orc_calibrate(const uint32_t *series, uint64_t n, uint32_t *t1, uint32_t *t2) {
  if (n < 4) { *t1 = *t2 = 0; return 1; }
  *t1 = orc_percentile_u32(series, n, 50);
  *t2 = orc_percentile_u32(series, n, 75);
  return *t1 == *t2 ? 2 : 0;
}

/* a6 — the first-cut law: r = 0 below t1; r_min at
 * t1 rising linearly to r_max at t2; clamped.  Exact integer form of
 * r_min + (r_max - r_min)(MA - t1)/(t2 - t1) with MA = A/k, floored to a bp. */
uint32_t orc_map_rate(uint64_t A, uint32_t k, const orc_ctrl *c) {
  if (A < (uint64_t)k * c->t1) return 0;
  uint64_t num = (uint64_t)(c->r_max_bp - c->r_min_bp) * (A - (uint64_t)k * c->t1);
  uint64_t den = (uint64_t)k * (c->t2 - c->t1);
  uint64_t r = c->r_min_bp + num / den;
  if (r > c->r_max_bp) r = c->r_max_bp;
  if (c->n_rungs) { /* ladder (R5): the largest rung <= r */
    uint32_t best = c->rungs_bp[0];
    for (uint32_t i = 0; i < c->n_rungs; ++i)
      if (c->rungs_bp[i] <= r) best = c->rungs_bp[i];
    r = best;
  }
  return (uint32_t)r;
}

/* NEXT-2 similarity model (P:193 87 % active / 88 %
 * inactive; P:102 floor 65 %; P:106 safe window < 20 %).  Reduction vs the
 * request's unbounded length: red = (U - R) / U.  Inactive: base = q[0].
 * Active: base = q[1] for red <= safe, the floor q[2] for red >= end, linear in
 * between (floored to a centi-point); score = clamp(base + noise, 0, 10000). */
uint32_t orc_similarity(uint32_t U, uint32_t R, int active, int32_t noise, const uint32_t q[5]) {
  int64_t base;
  if (!active) {
    base = q[0];
  } else {
    /* red in bp as the exact rational num / den */
    int64_t num = ((int64_t)U - (int64_t)R) * 10000, den = (int64_t)U;
    if (num <= (int64_t)q[3] * den) base = q[1];
    else if (num >= (int64_t)q[4] * den) base = q[2];
    else base = (int64_t)q[1] - ((int64_t)(q[1] - q[2]) * (num - (int64_t)q[3] * den)) /
                                    ((int64_t)(q[4] - q[3]) * den);
  }
  int64_t s = base + noise;
  if (s < 0) s = 0;
  if (s > 10000) s = 10000;
  return (uint32_t)s;
}

/* floor(x / 2^32) for signed 128-bit x */
static __int128 floor_div_2p32(__int128 x) {
  __int128 d = (__int128)1 << 32;
  __int128 q = x / d;
  if ((x % d) != 0 && x < 0) q -= 1;
  return q;
}

/* a7 — bounded target N = round(P (1 - r)) (R11) and realized
 * length round(poly(N) * Fcomp) clamped to [1, 2^24]. */
static uint32_t bounded_realized(uint32_t P, uint32_t r_bp, int32_t fcomp, const int64_t poly[3]) {
  int64_t N = ((int64_t)P * (10000 - (int64_t)r_bp) + 5000) / 10000;
  if (N < 1) N = 1;
  __int128 p = (__int128)poly[0] + (__int128)poly[1] * N + (__int128)poly[2] * N * N;
  __int128 x = floor_div_2p32(p * fcomp + ((__int128)1 << 31));
  if (x < 1) x = 1;
  if (x > (1 << 24)) x = 1 << 24;
  return (uint32_t)x;
}

/* ------------------------------------------------------------------------- */
typedef struct {
  uint64_t admit, first, done, last_tok, prefill_end;
  uint32_t emitted, R, r_bp, state, n_gaps;
  uint64_t enq;      /* start of the current queue stay (arrival, or the preemption instant) */
  uint32_t seq, gen; /* admission order (every admission); admissions so far */
} rstate;

typedef struct {
  const orc_ctrl *c;
  uint32_t law;
  uint32_t *samples;   /* every ingested sample, in order */
  uint64_t n, cap;
  uint32_t *words;     /* BBR: decode words emitted in each ingested second */
  uint64_t nw, capw;
  int active;
  uint32_t r, rung;
  uint32_t rt_min;     /* BBR: minimum sample so far */
  uint32_t phase;      /* PCC: 0 idle, 1 experiment r_base + delta running, 2 r_base - delta running */
  uint32_t r_base;     /* PCC */
  uint64_t cost_a;     /* PCC: cost of experiment 1 */
} cstate;

static int push_u32(uint32_t **v, uint64_t *n, uint64_t *cap, uint32_t x) {
  if (*n == *cap) {
    uint64_t nc = *cap ? 2 * *cap : 64;
    uint32_t *nv = (uint32_t *)realloc(*v, nc * sizeof(uint32_t));
    if (!nv) return -1;
    *v = nv;
    *cap = nc;
  }
  (*v)[(*n)++] = x;
  return 0;
}

/* MPC ("predict the system load and preemptively adjust r ... cost
 * functions that include latency, output quality, and energy efficiency over
 * a moving time horizon and help avoid oscillations in r"; reading R41).
 * Window y_1..y_k (oldest..newest), A = sum.  Forecast h seconds ahead from
 * the window mean and its end-to-end slope:
 *   F = A/k + h (y_k - y_1)/(k - 1)   (k >= 2; F = y_1 for k = 1), floored at 0.
 * Predicted signal under r: x(r) = F (1 - r/10^4) (a shorter output shrinks
 * the decode work in proportion).  Cost of a candidate r:
 *   J(r) = w_lat max(0, x(r) - t1) + w_q r + w_osc |r - r_prev|
 * over the candidates {0} U rungs, or {0} U {r_min + floor(i (r_max - r_min) / 30),
 * i = 0..30}; the smallest r among the minima.  Exact: every term is multiplied
 * by 10^4 D, D = k (k - 1) (1 for k = 1), in 128-bit integers. */
static uint32_t mpc_rate(const orc_ctrl *c, const uint32_t *y, uint32_t k, uint32_t r_prev) {
  __int128 A = 0;
  for (uint32_t i = 0; i < k; ++i) A += y[i];
  __int128 D, F;
  if (k >= 2) {
    D = (__int128)k * (k - 1);
    F = A * (k - 1) + (__int128)c->horizon_s * k * ((__int128)y[k - 1] - (__int128)y[0]);
  } else {
    D = 1;
    F = A;
  }
  if (F < 0) F = 0;
  uint32_t cand[32];
  uint32_t nc = 0;
  cand[nc++] = 0;
  if (c->n_rungs) {
    for (uint32_t i = 0; i < c->n_rungs; ++i) cand[nc++] = c->rungs_bp[i];
  } else {
    for (uint32_t i = 0; i <= 30; ++i) cand[nc++] = c->r_min_bp + (uint32_t)((uint64_t)i * (c->r_max_bp - c->r_min_bp) / 30);
  }
  uint32_t best_r = 0;
  __int128 best = -1;
  for (uint32_t i = 0; i < nc; ++i) {
    __int128 r = cand[i];
    __int128 ex = F * (10000 - r) - (__int128)c->t1 * 10000 * D;
    if (ex < 0) ex = 0;
    __int128 dr = r > (__int128)r_prev ? r - r_prev : (__int128)r_prev - r;
    __int128 J = (__int128)c->w_lat * ex + (__int128)10000 * D * ((__int128)c->w_q * r + (__int128)c->w_osc * dr);
    if (best < 0 || J < best) { best = J; best_r = cand[i]; }
  }
  return best_r;
}

/* one controller ingest of the sample x of closed second `second` (a6);
 * w = decode words emitted in that second (BBR's delivery rate) */
static int ingest(cstate *cs, uint32_t second, uint32_t x, uint32_t w, orc_result *res, orc_log *log) {
  const uint32_t law = cs->law;
  if (law != ORC_LAW_MAP && law != ORC_LAW_STEP && law != ORC_LAW_MPC && law != ORC_LAW_BBR && law != ORC_LAW_PCC)
    return 0;
  if (push_u32(&cs->samples, &cs->n, &cs->cap, x)) return -1;
  if (push_u32(&cs->words, &cs->nw, &cs->capw, w)) return -1;
  const orc_ctrl *c = cs->c;
  /* moving average over the last `window` samples; partial window at start */
  uint32_t k = cs->n < c->window ? (uint32_t)cs->n : c->window;
  uint64_t A = 0;
  for (uint64_t i = cs->n - k; i < cs->n; ++i) A += cs->samples[i];
  const uint32_t r_prev = cs->r;
  int act = 0;
  uint32_t r = 0;
  if (law == ORC_LAW_MAP || law == ORC_LAW_STEP) {
    act = A >= (uint64_t)k * c->t1; /* MA >= T1 triggers (R38); below resets */
    if (act) {
      if (law == ORC_LAW_MAP) {
        r = orc_map_rate(A, k, c);
      } else { /* STEP (R4, R5): rung 0 on activation, one rung up per ingest while active */
        if (!cs->active) cs->rung = 0;
        else if (cs->rung + 1 < c->n_rungs) cs->rung++;
        r = c->rungs_bp[cs->rung];
      }
    }
  } else if (law == ORC_LAW_MPC) {
    r = mpc_rate(c, cs->samples + (cs->n - k), k, r_prev);
    act = r > 0;
  } else if (law == ORC_LAW_BBR) {
    /* BBR-style ("operate at the equivalent of Kleinrock's point, keeping
     * TBT low while maximizing the token generation (tokens/s)"; reading R42):
     * RTprop = the minimum TBT sample so far, BtlBw = the maximum decode words/s
     * over the window.  Congested (queueing delay beyond the allowance t1):
     * MA >= RTprop + t1.  At the bandwidth plateau (8 w >= 7 BtlBw) a congested
     * controller sheds one step of output; a controller below the delay target
     * gives one step back (probing for more tokens/s); else it holds. */
    if (x < cs->rt_min) cs->rt_min = x;
    uint32_t bw = 0;
    for (uint64_t i = cs->nw - k; i < cs->nw; ++i)
      if (cs->words[i] > bw) bw = cs->words[i];
    const int congested = A >= (uint64_t)k * ((uint64_t)cs->rt_min + c->t1);
    const int plateau = 8ull * w >= 7ull * bw;
    r = r_prev;
    if (congested && plateau) {
      if (c->n_rungs) {
        if (r_prev == 0) cs->rung = 0;
        else if (cs->rung + 1 < c->n_rungs) cs->rung++;
        r = c->rungs_bp[cs->rung];
      } else {
        r = r_prev == 0 ? c->r_min_bp : (r_prev + c->step_bp > c->r_max_bp ? c->r_max_bp : r_prev + c->step_bp);
      }
    } else if (!congested) {
      if (c->n_rungs) {
        if (r_prev == 0 || cs->rung == 0) r = 0;
        else r = c->rungs_bp[--cs->rung];
      } else {
        r = r_prev <= c->r_min_bp ? 0 : (r_prev < c->r_min_bp + c->step_bp ? c->r_min_bp : r_prev - c->step_bp);
      }
    }
    act = r > 0;
  } else { /* ORC_LAW_PCC */
    /* PCC-style ("run micro-experiments with different values of r and
     * measure a utility function that combines both latency and response
     * quality"; reading R43).  Active while MA >= t1.  Each monitor interval is
     * one ingested second: experiment 1 runs r_base + delta, experiment 2
     * r_base - delta (clamped to [r_min, r_max]); the ingest after each
     * measures its cost w_lat max(0, x - t1) + w_q r (utility = -cost); after
     * the pair, r_base moves one delta toward the cheaper side (ties stay). */
    act = A >= (uint64_t)k * c->t1;
    const uint32_t d = c->step_bp;
    if (!act) {
      cs->phase = 0;
      cs->r_base = 0;
      r = 0;
    } else {
      const uint64_t cost = (uint64_t)c->w_lat * (x > c->t1 ? x - c->t1 : 0) + (uint64_t)c->w_q * r_prev;
      if (cs->phase == 0) {
        cs->r_base = c->r_min_bp;
      } else if (cs->phase == 1) {
        cs->cost_a = cost;
      } else {
        if (cs->cost_a < cost) cs->r_base = cs->r_base + d > c->r_max_bp ? c->r_max_bp : cs->r_base + d;
        else if (cost < cs->cost_a) cs->r_base = cs->r_base < c->r_min_bp + d ? c->r_min_bp : cs->r_base - d;
      }
      if (cs->phase == 1) { /* start experiment 2 */
        r = cs->r_base < c->r_min_bp + d ? c->r_min_bp : cs->r_base - d;
        cs->phase = 2;
      } else { /* start experiment 1 */
        r = cs->r_base + d > c->r_max_bp ? c->r_max_bp : cs->r_base + d;
        cs->phase = 1;
      }
    }
  }
  if (act && !cs->active) {
    res->activations++;
    if (res->first_act_s == ORC_NONE) res->first_act_s = second;
  }
  if (!act && cs->active) res->last_deact_s = second;
  if (act) res->active_ingests++;
  cs->active = act;
  cs->r = r;
  if (log && log->ctrl) {
    if (log->n_ctrl < log->cap_ctrl) {
      orc_ctrl_log *L = &log->ctrl[log->n_ctrl];
      L->second = second; L->sample = x; L->k = k; L->r_bp = r; L->active = (uint32_t)act; L->A = A;
    }
    log->n_ctrl++;
  }
  return 0;
}

int orc_ctrl_trace(const orc_ctrl *c, const uint32_t *sec, const uint32_t *x, const uint32_t *w, uint64_t n,
                   orc_result *res, orc_ctrl_log *out) {
  memset(res, 0, sizeof(*res));
  res->first_act_s = res->last_deact_s = ORC_NONE;
  cstate cs;
  memset(&cs, 0, sizeof(cs));
  cs.c = c;
  cs.law = c->law;
  cs.rt_min = ORC_NONE;
  orc_log log;
  memset(&log, 0, sizeof(log));
  log.ctrl = out;
  log.cap_ctrl = out ? n : 0;
  int rc = 0;
  for (uint64_t i = 0; i < n && rc == 0; ++i) rc = ingest(&cs, sec[i], x[i], w ? w[i] : 0, res, &log);
  free(cs.samples);
  free(cs.words);
  return rc;
}

static uint64_t overlap(uint64_t a, uint64_t b, int64_t w0, int64_t w1) {
  uint64_t lo = a > (uint64_t)w0 ? a : (uint64_t)w0;
  uint64_t hi = b < (uint64_t)w1 ? b : (uint64_t)w1;
  return hi > lo ? hi - lo : 0;
}

static int in_window(uint64_t t, const orc_run_cfg *cfg) {
  return (int64_t)t >= cfg->w0_us && (int64_t)t < cfg->w1_us;
}

/* Epilogue shared by both event loops: a8 energy, a9 percentiles (+ exact
 * self-check values), the per-second rows and the per-request log. */
static void finish_run(orc_result *res, const orc_profile *prof, uint64_t *e2e_v, uint64_t n_e2e, uint64_t *ttft_v,
                       uint64_t n_ttft, const orc_second_row *rows, uint64_t n_sec, uint64_t end, uint64_t n_series,
                       const rstate *rs, uint64_t n_req, orc_log *log) {
  /* a8 energy, fp64, in this fixed order (R19) */
  {
    double a = prof->e_in * (double)res->words_in;
    double b = prof->e_out * (double)res->words_out;
    double c = prof->p_idle * (double)res->idle_us;
    res->energy_j = (a + b) + c / 1e6;
    double wa = prof->e_in * (double)res->win_words_in;
    double wb = prof->e_out * (double)res->win_words_out;
    double wc = prof->p_idle * (double)res->win_idle_us;
    res->win_energy_j = (wa + wb) + wc / 1e6;
  }
  /* a9 percentiles: nearest rank on the histograms -> bin lower edge */
  {
    uint64_t n = res->served;
    res->e2e_p50_ms = res->e2e_p99_ms = res->ttft_p50_ms = res->ttft_p99_ms = ORC_NONE;
    res->median_r_bp = ORC_NONE;
    const uint32_t ps[2] = {50, 99};
    for (int w = 0; w < 2; ++w) {
      const uint32_t *hh = w == 0 ? res->hist_e2e : res->hist_ttft;
      uint64_t nn = w == 0 ? n : n_ttft;
      for (int q = 0; q < 2; ++q) {
        if (nn == 0) continue;
        uint64_t k = nr_rank(nn, ps[q]), cum = 0;
        uint32_t bsel = 0;
        for (uint32_t b = 0; b < ORC_HIST_LAT; ++b) {
          cum += hh[b];
          if (cum >= k) { bsel = b; break; }
        }
        uint32_t v = (uint32_t)orc_lat_edge(bsel);
        if (w == 0 && q == 0) res->e2e_p50_ms = v;
        if (w == 0 && q == 1) res->e2e_p99_ms = v;
        if (w == 1 && q == 0) res->ttft_p50_ms = v;
        if (w == 1 && q == 1) res->ttft_p99_ms = v;
      }
    }
    if (res->rewritten) {
      uint64_t k = nr_rank(res->rewritten, 50), cum = 0;
      for (uint32_t b = 0; b < ORC_HIST_R; ++b) {
        cum += res->hist_r[b];
        if (cum >= k) { res->median_r_bp = b * 10; break; }
      }
    }
    /* NEXT-2 medians: nearest rank on the 0.5-point score histograms */
    res->sim_active_p50 = res->sim_inactive_p50 = ORC_NONE;
    for (int w = 0; w < 2; ++w) {
      const uint32_t *hq = w == 0 ? res->hist_q_active : res->hist_q_inactive;
      uint64_t nq = w == 0 ? res->scored_active : res->scored_inactive;
      if (!nq) continue;
      uint64_t k = nr_rank(nq, 50), cum = 0;
      for (uint32_t b = 0; b < ORC_HIST_Q; ++b) {
        cum += hq[b];
        if (cum >= k) {
          if (w == 0) res->sim_active_p50 = b * 50; else res->sim_inactive_p50 = b * 50;
          break;
        }
      }
    }
    /* exact nearest-rank values (self-check only) */
    qsort(e2e_v, n_e2e, sizeof(uint64_t), cmp_u64);
    qsort(ttft_v, n_ttft, sizeof(uint64_t), cmp_u64);
    res->e2e_exact_p50_us = n_e2e ? e2e_v[nr_rank(n_e2e, 50) - 1] : NEVER;
    res->e2e_exact_p99_us = n_e2e ? e2e_v[nr_rank(n_e2e, 99) - 1] : NEVER;
    res->ttft_exact_p50_us = n_ttft ? ttft_v[nr_rank(n_ttft, 50) - 1] : NEVER;
    res->ttft_exact_p99_us = n_ttft ? ttft_v[nr_rank(n_ttft, 99) - 1] : NEVER;
  }
  res->n_series = (uint32_t)n_series;
  if (rows && log && log->rows) {
    uint64_t nr = end / US + 1; /* seconds 0 .. floor(end / 1e6) */
    if (nr > n_sec) nr = n_sec;
    for (uint64_t k = 0; k < nr && k < log->cap_rows; ++k) log->rows[k] = rows[k];
    log->n_rows = nr;
  }
  if (log && log->req) {
    for (uint64_t i = 0; i < n_req; ++i) {
      log->req[i].admit_us = rs[i].admit;
      log->req[i].first_us = rs[i].first;
      log->req[i].done_us = rs[i].done;
      log->req[i].R = rs[i].R;
      log->req[i].r_bp = rs[i].r_bp;
      log->req[i].n_gaps = rs[i].n_gaps;
    }
  }
}

/* NEXT-4 token-level costs ("tokens_per_word"; reading R44): with
 * tpw_q16 != 0 the engine works in tokens — a count of w words is
 * clamp(round(w tpw), 1, 2^24) tokens (half-up, Q16) — and every per-unit constant of
 * the profile (prefill and KV ns, KV capacity, energy per unit) is per token. */
static uint32_t to_tokens(uint32_t words, uint32_t tpw_q16) {
  if (tpw_q16 == 0) return words;
  uint64_t t = ((uint64_t)words * tpw_q16 + (1u << 15)) >> 16;
  if (t > (1u << 24)) t = 1u << 24; /* the realized-length bound (R11) holds in tokens too */
  return t < 1 ? 1u : (uint32_t)t;
}

int orc_simulate(const orc_request *req_words, uint64_t n_req, const orc_profile *prof,
                 const orc_ctrl *ctrl, const orc_run_cfg *cfg, orc_result *res, orc_log *log) {
  if (prof->replicas > 1) return orc_simulate_replicas(req_words, n_req, prof, ctrl, cfg, res, log);
  memset(res, 0, sizeof(*res));
  /* the engine's view of each request: its input in tokens (R44) */
  orc_request *req = (orc_request *)malloc((n_req ? n_req : 1) * sizeof(orc_request));
  if (!req) return -1;
  for (uint64_t i = 0; i < n_req; ++i) {
    req[i] = req_words[i];
    req[i].input = to_tokens(req_words[i].input, prof->tpw_q16);
  }
  res->first_act_s = res->last_deact_s = ORC_NONE;
  res->t1 = ctrl->t1;
  res->t2 = ctrl->t2;
  const uint64_t H = (uint64_t)cfg->horizon_us;
  int rc = -1;

  rstate *rs = (rstate *)calloc(n_req ? n_req : 1, sizeof(rstate));
  uint32_t *queue = (uint32_t *)malloc((n_req ? n_req : 1) * sizeof(uint32_t));
  uint32_t *ready = (uint32_t *)malloc((n_req ? n_req : 1) * sizeof(uint32_t));
  uint32_t *batch = (uint32_t *)malloc((n_req ? n_req : 1) * sizeof(uint32_t));
  uint32_t *pending = (uint32_t *)malloc((n_req ? n_req : 1) * sizeof(uint32_t)); /* contending prefill */
  uint32_t *stack = (uint32_t *)malloc((n_req ? n_req : 1) * sizeof(uint32_t));   /* preempted: queue front */
  uint64_t *e2e_v = (uint64_t *)malloc((n_req ? n_req : 1) * sizeof(uint64_t));
  uint64_t *ttft_v = (uint64_t *)malloc((n_req ? n_req : 1) * sizeof(uint64_t));
  uint64_t n_sec = H / US + 2;
  uint64_t *sec_tbt_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_tbt_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_e2e_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_e2e_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_slo_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_ttft_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_ttft_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_in_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));   /* NEXT-3 INPUT */
  uint64_t *sec_in_any = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_util_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t)); /* NEXT-3 UTIL */
  uint64_t *sec_util_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  orc_second_row *rows = (cfg->record & 2) ? (orc_second_row *)calloc(n_sec, sizeof(orc_second_row)) : NULL;
  heap h = {0, 0, 0};
  cstate cs;
  memset(&cs, 0, sizeof(cs));
  cs.c = ctrl;
  cs.law = ctrl->law;
  cs.rt_min = ORC_NONE;
  if (!rs || !queue || !ready || !batch || !pending || !stack || !e2e_v || !ttft_v || !sec_tbt_sum || !sec_tbt_cnt ||
      !sec_e2e_sum || !sec_e2e_cnt || !sec_slo_cnt || !sec_ttft_sum || !sec_ttft_cnt || !sec_in_sum ||
      !sec_in_any || !sec_util_sum || !sec_util_cnt ||
      ((cfg->record & 2) && !rows))
    goto out;
  if (cs.law == ORC_LAW_CONST) cs.r = ctrl->r_const_bp; /* S:320-326 constant policy */

  for (uint64_t i = 0; i < n_req; ++i) {
    rs[i].admit = rs[i].first = rs[i].done = NEVER;
    rs[i].enq = req[i].a_us;
    if (heap_push(&h, (event){req[i].a_us, EV_ARRIVAL, (uint32_t)i, 0})) goto out;
  }

  uint64_t q_head = 0, q_tail = 0, n_ready = 0, n_batch = 0, in_sys = 0;
  uint64_t kv_reserved = 0; /* NEXT-4: sum of (input + R) over requests in the system */
  uint64_t n_pend = 0, pend_us = 0; /* NEXT-4 contending prefill: admitted, prefill not started */
  uint64_t n_stack = 0;             /* NEXT-4 kv_policy 1: preempted requests at the queue front */
  uint32_t next_seq = 0;            /* admission order */
  const int preempt = prof->kv_policy == 1 && prof->kv_cap_words > 0;
  uint64_t n_e2e = 0, n_ttft = 0;
  int busy = 0;
  uint64_t next_sec = 0; /* first second not yet ingested */
  uint64_t T_prev = 0, last_T = 0;
  uint64_t n_series = 0;

#define INGEST_UNTIL(TT)                                                                 \
  do {                                                                                   \
    for (; (next_sec + 1) * US <= (TT); ++next_sec) {                                    \
      uint64_t cnt, sum;                                                                 \
      if (next_sec >= n_sec) continue;                                                   \
      if (ctrl->signal == ORC_SIG_TBT) { cnt = sec_tbt_cnt[next_sec]; sum = sec_tbt_sum[next_sec]; } \
      else if (ctrl->signal == ORC_SIG_TTFT) { cnt = sec_ttft_cnt[next_sec]; sum = sec_ttft_sum[next_sec]; } \
      else if (ctrl->signal == ORC_SIG_E2E) { cnt = sec_e2e_cnt[next_sec]; sum = sec_e2e_sum[next_sec]; } \
      else if (ctrl->signal == ORC_SIG_INPUT) { cnt = sec_in_any[next_sec]; sum = sec_in_sum[next_sec]; } \
      else if (ctrl->signal == ORC_SIG_UTIL) { cnt = (uint64_t)prof->max_batch * sec_util_cnt[next_sec];    \
                                               sum = 10000 * sec_util_sum[next_sec]; }                  \
      else { cnt = sec_e2e_cnt[next_sec]; sum = 1000 * sec_slo_cnt[next_sec]; }          \
      if (cnt == 0) continue; /* a second with no samples is a gap */     \
      uint32_t x = (uint32_t)(sum / cnt);                                                \
      if (cfg->record & 1) {                                                             \
        if (log && log->series && n_series < log->cap_series) log->series[n_series] = x; \
        n_series++;                                                                      \
      }                                                                                  \
      if (ingest(&cs, (uint32_t)next_sec, x, (uint32_t)sec_tbt_cnt[next_sec], res, log)) goto out; \
    }                                                                                    \
  } while (0)

  for (;;) {
    if (h.n == 0) break;
    uint64_t T = h.v[0].t;
    if (T >= H) break;
    /* integrate piecewise-constant state over [T_prev, T) */
    {
      uint64_t dt = T - T_prev, nq = q_tail - q_head + n_stack;
      if (in_sys == 0) {
        res->idle_us += dt;
        res->win_idle_us += overlap(T_prev, T, cfg->w0_us, cfg->w1_us);
        if (rows)
          for (uint64_t s = T_prev / US; s * US < T && s < n_sec; ++s)
            rows[s].idle_us += (uint32_t)overlap(T_prev, T, (int64_t)(s * US), (int64_t)((s + 1) * US));
      }
      res->int_system_us += (nq + in_sys) * dt;
      res->int_queue_us += nq * dt;
    }
    T_prev = T;
    last_T = T;
    uint64_t s_idx = T / US;
    while (h.n && h.v[0].t == T) {
      event e = heap_pop(&h);
      if (e.kind == EV_ITER_END) {
        /* UTIL: the decode batch size at this iteration end */
        sec_util_sum[s_idx] += n_batch;
        sec_util_cnt[s_idx] += 1;
        /* E1: every request in the iteration emits a word at T */
        for (uint64_t b = 0; b < n_batch; ++b) {
          uint32_t m = batch[b];
          uint64_t gap = T - rs[m].last_tok;
          sec_tbt_sum[s_idx] += gap;
          sec_tbt_cnt[s_idx] += 1;
          res->tbt_samples++;
          res->tbt_sum_us += gap;
          if (gap > res->tbt_max_us) res->tbt_max_us = gap;
          if (log && log->gaps && log->n_gaps < log->cap_gaps) {
            log->gaps[2 * log->n_gaps] = m;
            log->gaps[2 * log->n_gaps + 1] = gap;
          }
          if (log) log->n_gaps++;
          rs[m].n_gaps++;
          rs[m].last_tok = T;
          rs[m].emitted++;
          res->words_out++;
          if (rows) {
            rows[s_idx].tbt_count++;
            rows[s_idx].sum_tbt_us += gap;
            rows[s_idx].words_out++;
          }
          if (in_window(T, cfg)) res->win_words_out++;
          if (rs[m].emitted == rs[m].R) { /* completes: E2E = completion - arrival */
            uint64_t e2e = T - req[m].a_us;
            rs[m].done = T;
            rs[m].state = RS_DONE;
            in_sys--;
            kv_reserved -= (uint64_t)req[m].input + rs[m].R;
            res->served++;
            res->sum_e2e_us += e2e;
            res->sum_sojourn_us += e2e;
            e2e_v[n_e2e++] = e2e;
            res->hist_e2e[orc_lat_bin(e2e / 1000)]++;
            if (in_window(T, cfg)) res->win_served++;
            sec_e2e_sum[s_idx] += e2e;
            sec_e2e_cnt[s_idx] += 1;
            if (e2e > ctrl->slo_us) { sec_slo_cnt[s_idx] += 1; res->slo_violations++; }
            if (rows) {
              rows[s_idx].completions++;
              rows[s_idx].sum_e2e_us += e2e;
            }
          } else {
            rs[m].state = RS_READY;
            ready[n_ready++] = m;
          }
        }
        n_batch = 0;
        busy = 0;
        if (preempt) {
          /* contexts of everything in the system: input + words emitted so far */
          uint64_t F = 0;
          for (uint64_t i = 0; i < n_req; ++i)
            if (rs[i].state == RS_PREFILL || rs[i].state == RS_READY || rs[i].state == RS_DECODING)
              F += (uint64_t)req[i].input + rs[i].emitted;
          while (F > prof->kv_cap_words && in_sys > 1) {
            /* the latest admitted request in the system goes back to the queue front */
            uint64_t v = n_req;
            for (uint64_t i = 0; i < n_req; ++i)
              if ((rs[i].state == RS_PREFILL || rs[i].state == RS_READY) && (v == n_req || rs[i].seq > rs[v].seq))
                v = i;
            if (rs[v].state == RS_READY) { /* leaves the decode-ready list */
              uint64_t w = 0;
              for (uint64_t b = 0; b < n_ready; ++b)
                if (ready[b] != v) ready[w++] = ready[b];
              n_ready = w;
            }
            F -= (uint64_t)req[v].input + rs[v].emitted;
            rs[v].state = RS_QUEUED; /* a pending prefill end of it is now stale (gen) */
            rs[v].enq = T;
            stack[n_stack++] = (uint32_t)v;
            in_sys--;
            res->preemptions++;
          }
        }
      } else if (e.kind == EV_PREFILL_END) {
        uint32_t m = e.idx;
        if (rs[m].state != RS_PREFILL || rs[m].gen != e.gen) continue; /* preempted meanwhile */
        if (rs[m].emitted > 0) {
          /* a re-admitted request's recompute prefill ends: its next word, a decode
           * word whose TBT gap runs from its last word (before the preemption) */
          uint64_t gap = T - rs[m].last_tok;
          sec_tbt_sum[s_idx] += gap;
          sec_tbt_cnt[s_idx] += 1;
          res->tbt_samples++;
          res->tbt_sum_us += gap;
          if (gap > res->tbt_max_us) res->tbt_max_us = gap;
          if (log && log->gaps && log->n_gaps < log->cap_gaps) {
            log->gaps[2 * log->n_gaps] = m;
            log->gaps[2 * log->n_gaps + 1] = gap;
          }
          if (log) log->n_gaps++;
          rs[m].n_gaps++;
          rs[m].last_tok = T;
          rs[m].emitted++;
          res->words_out++;
          if (rows) {
            rows[s_idx].tbt_count++;
            rows[s_idx].sum_tbt_us += gap;
            rows[s_idx].words_out++;
          }
          if (in_window(T, cfg)) res->win_words_out++;
          if (rs[m].emitted == rs[m].R) {
            uint64_t e2e = T - req[m].a_us;
            rs[m].done = T;
            rs[m].state = RS_DONE;
            in_sys--;
            res->served++;
            res->sum_e2e_us += e2e;
            res->sum_sojourn_us += e2e;
            e2e_v[n_e2e++] = e2e;
            res->hist_e2e[orc_lat_bin(e2e / 1000)]++;
            if (in_window(T, cfg)) res->win_served++;
            sec_e2e_sum[s_idx] += e2e;
            sec_e2e_cnt[s_idx] += 1;
            if (e2e > ctrl->slo_us) { sec_slo_cnt[s_idx] += 1; res->slo_violations++; }
            if (rows) {
              rows[s_idx].completions++;
              rows[s_idx].sum_e2e_us += e2e;
            }
          } else {
            rs[m].state = RS_READY;
            ready[n_ready++] = m;
          }
          continue;
        }
        /* E2: first word at prefill end; TTFT = first token - arrival */
        uint64_t ttft = T - req[m].a_us;
        rs[m].first = T;
        rs[m].last_tok = T;
        rs[m].emitted = 1;
        res->words_out++;
        if (in_window(T, cfg)) res->win_words_out++;
        res->sum_ttft_us += ttft;
        sec_ttft_sum[s_idx] += ttft;
        sec_ttft_cnt[s_idx] += 1;
        ttft_v[n_ttft++] = ttft;
        res->hist_ttft[orc_lat_bin(ttft / 1000)]++;
        if (rows) {
          rows[s_idx].first_tokens++;
          rows[s_idx].sum_ttft_us += ttft;
          rows[s_idx].words_out++;
        }
        if (rs[m].R == 1) { /* R9: realized length 1 completes at prefill end */
          uint64_t e2e = ttft;
          rs[m].done = T;
          rs[m].state = RS_DONE;
          in_sys--;
          kv_reserved -= (uint64_t)req[m].input + rs[m].R;
          res->served++;
          res->sum_e2e_us += e2e;
          res->sum_sojourn_us += e2e;
          e2e_v[n_e2e++] = e2e;
          res->hist_e2e[orc_lat_bin(e2e / 1000)]++;
          if (in_window(T, cfg)) res->win_served++;
          sec_e2e_sum[s_idx] += e2e;
          sec_e2e_cnt[s_idx] += 1;
          if (e2e > ctrl->slo_us) { sec_slo_cnt[s_idx] += 1; res->slo_violations++; }
          if (rows) {
            rows[s_idx].completions++;
            rows[s_idx].sum_e2e_us += e2e;
          }
        } else {
          rs[m].state = RS_READY;
          ready[n_ready++] = m;
        }
      } else { /* E3: arrival -> FIFO queue */
        uint32_t m = e.idx;
        rs[m].state = RS_QUEUED;
        queue[q_tail++] = m;
        res->arrivals++;
        if (rows) rows[s_idx].arrivals++;
        res->candidates = (uint64_t)req[m].j + 1;
      }
    }
    if (!busy) {
      /* admission point: ingest every closed second, then admit FIFO */
      INGEST_UNTIL(T);
      while (in_sys < prof->max_batch && (n_stack > 0 || q_head < q_tail)) {
        if (n_stack > 0) {
          /* NEXT-4 kv_policy 1: a preempted request (queue front) is admitted again
           * if its context fits; its rewrite R stays; it prefills input + emitted */
          uint32_t m = stack[n_stack - 1];
          uint64_t ctx = (uint64_t)req[m].input + rs[m].emitted, F = 0;
          for (uint64_t i = 0; i < n_req; ++i)
            if (rs[i].state == RS_PREFILL || rs[i].state == RS_READY || rs[i].state == RS_DECODING)
              F += (uint64_t)req[i].input + rs[i].emitted;
          if (in_sys > 0 && F + ctx > prof->kv_cap_words) break;
          n_stack--;
          rs[m].seq = next_seq++;
          rs[m].gen++;
          uint64_t pf = ((uint64_t)prof->prefill_ns_per_word * ctx) / 1000;
          if (pf < 1) pf = 1;
          rs[m].prefill_end = T + pf;
          rs[m].state = RS_PREFILL;
          in_sys++;
          res->sum_queue_us += T - rs[m].enq;
          res->words_in += ctx;
          res->recompute_words += ctx;
          sec_in_sum[T / US] += ctx;
          sec_in_any[T / US] = 1;
          if (in_window(T, cfg)) res->win_words_in += ctx;
          if (rows) {
            rows[T / US].sum_queue_us += T - rs[m].enq;
            rows[T / US].words_in += (uint32_t)ctx;
          }
          if (heap_push(&h, (event){rs[m].prefill_end, EV_PREFILL_END, m, rs[m].gen})) goto out;
          continue;
        }
        uint32_t m = queue[q_head];
        uint32_t r = cs.r;
        /* NEXT-3 bypass: class policy or a short predicted output */
        int bypass = r > 0 && (((ctrl->bypass_mask >> req[m].cls) & 1u) || req[m].P < ctrl->min_words_bypass);
        if (bypass) r = 0;
        /* realized output in words (the rewrite), decoded as tokens (R44) */
        const uint32_t R_words = r > 0 ? bounded_realized(req[m].P, r, req[m].fcomp_q16, cfg->poly_q16) : req[m].U;
        const uint32_t R = to_tokens(R_words, prof->tpw_q16);
        /* NEXT-4 KV-capacity admission: the head's full context (input + realized
         * output) must fit beside everything admitted; strict FIFO; an oversized
         * request is admitted only into an empty system */
        uint64_t need = (uint64_t)req[m].input + R;
        if (preempt) {
          /* kv_policy 1: only the current context (the input) has to fit */
          uint64_t F = 0;
          for (uint64_t i = 0; i < n_req; ++i)
            if (rs[i].state == RS_PREFILL || rs[i].state == RS_READY || rs[i].state == RS_DECODING)
              F += (uint64_t)req[i].input + rs[i].emitted;
          if (in_sys > 0 && F + req[m].input > prof->kv_cap_words) break;
        } else if (prof->kv_cap_words && in_sys > 0 && kv_reserved + need > prof->kv_cap_words) {
          break;
        }
        q_head++;
        rs[m].seq = next_seq++;
        rs[m].gen++;
        kv_reserved += need;
        if (bypass) res->bypassed++;
        rs[m].admit = T;
        rs[m].r_bp = r;
        rs[m].R = R;
        uint64_t pf = ((uint64_t)prof->prefill_ns_per_word * req[m].input) / 1000;
        if (pf < 1) pf = 1;
        if (prof->prefill_mode) { /* contending: prefills run inside the next iteration */
          rs[m].state = RS_PENDING;
          pending[n_pend++] = m;
          pend_us += pf;
        } else {
          rs[m].prefill_end = T + pf;
          rs[m].state = RS_PREFILL;
        }
        in_sys++;
        res->admitted++;
        res->sum_queue_us += T - req[m].a_us;
        res->words_in += req[m].input;
        sec_in_sum[T / US] += req[m].input;
        sec_in_any[T / US] = 1;
        if (in_window(T, cfg)) res->win_words_in += req[m].input;
        if (rows) {
          uint64_t sa = T / US;
          rows[sa].admitted++;
          rows[sa].sum_queue_us += T - req[m].a_us;
          rows[sa].words_in += req[m].input;
        }
        if (r > 0) {
          res->rewritten++;
          res->hist_r[r / 10 < ORC_HIST_R ? r / 10 : ORC_HIST_R - 1]++;
        }
        { /* NEXT-2: score the admitted request against its unbounded counterpart */
          uint32_t sc = orc_similarity(req[m].U, R_words, r > 0, req[m].qnoise, cfg->quality);
          uint32_t qb = sc / 50 < ORC_HIST_Q ? sc / 50 : ORC_HIST_Q - 1;
          if (r > 0) { res->hist_q_active[qb]++; res->scored_active++; }
          else { res->hist_q_inactive[qb]++; res->scored_inactive++; }
        }
        if (!prof->prefill_mode && heap_push(&h, (event){rs[m].prefill_end, EV_PREFILL_END, m, rs[m].gen})) goto out;
      }
      /* iteration start with every decode-ready request (and, contending, the
       * prefills of everything just admitted) */
      if (n_ready > 0 || n_pend > 0) {
        uint64_t K = 0;
        for (uint64_t b = 0; b < n_ready; ++b) {
          uint32_t m = ready[b];
          batch[b] = m;
          rs[m].state = RS_DECODING;
          K += req[m].input + rs[m].emitted;
        }
        n_batch = n_ready;
        n_ready = 0;
        uint64_t B = n_batch;
        uint64_t d = B == 0 ? 0
                            : prof->t0_us + (uint64_t)prof->slope_us * (B > prof->knee ? B - prof->knee : 0) +
                                  ((uint64_t)prof->kv_ns_per_word * K) / 1000;
        d += pend_us; /* contending prefill (NEXT-4): cost(B) + sum of the prefills */
        for (uint64_t i = 0; i < n_pend; ++i) {
          uint32_t m = pending[i];
          rs[m].prefill_end = T + d;
          rs[m].state = RS_PREFILL;
          /* same instant as the iteration end; popped after it (kind order, R7) */
          if (heap_push(&h, (event){T + d, EV_PREFILL_END, m, rs[m].gen})) goto out;
        }
        n_pend = 0;
        pend_us = 0;
        if (heap_push(&h, (event){T + d, EV_ITER_END, 0, 0})) goto out;
        busy = 1;
        res->ticks++;
      }
    }
  }

  /* termination (R20): cutoff -> end at H; drain -> last event, unless capped */
  uint64_t end = (cfg->mode == ORC_MODE_DRAIN && h.n == 0) ? last_T : H;
  {
    uint64_t dt = end - T_prev, nq = q_tail - q_head + n_stack;
    if (in_sys == 0) {
      res->idle_us += dt;
      res->win_idle_us += overlap(T_prev, end, cfg->w0_us, cfg->w1_us);
      if (rows)
        for (uint64_t s = T_prev / US; s * US < end && s < n_sec; ++s)
          rows[s].idle_us += (uint32_t)overlap(T_prev, end, (int64_t)(s * US), (int64_t)((s + 1) * US));
    }
    res->int_system_us += (nq + in_sys) * dt;
    res->int_queue_us += nq * dt;
  }
  res->end_us = end;
  INGEST_UNTIL(end);
  res->queued_end = q_tail - q_head;
  res->inflight_end = in_sys + n_stack; /* admitted and not completed (preempted ones waiting too) */
  if (res->queued_end + res->inflight_end > 0) res->flags |= ORC_FLAG_TRUNCATED;

  finish_run(res, prof, e2e_v, n_e2e, ttft_v, n_ttft, rows, n_sec, end, n_series, rs, n_req, log);
  rc = 0;
out:
  free(req); free(rs); free(queue); free(ready); free(batch); free(pending); free(stack); free(e2e_v); free(ttft_v);
  free(sec_tbt_sum); free(sec_tbt_cnt); free(sec_e2e_sum); free(sec_e2e_cnt); free(sec_slo_cnt);
  free(sec_ttft_sum); free(sec_ttft_cnt); free(sec_in_sum); free(sec_in_any); free(sec_util_sum);
  free(sec_util_cnt);
  free(h.v); free(cs.samples); free(cs.words); free(rows);
  return rc;
}


/* NEXT-4 multi-replica routing ("the request scheduler ... picks requests
 * from the arrival queue and assigns to GPU servers"; P:183 8 GPUs; reading
 * R45).  `replicas` continuous-batching engines share one FIFO arrival queue
 * (the queue beLLMan rewrites in).  Replica q is at an admission point
 * at T when no iteration of q is running at T.  At an instant where some
 * replica is, the closed seconds are ingested and, while the queue holds an
 * arrived request and a replica at an admission point has a free slot, the
 * head is assigned to one of them chosen by the routing policy: least loaded
 * (fewest requests in the replica: prefilling, decode-ready or decoding; ties
 * to the lowest index) or round robin (the first such replica at or after a
 * cyclic pointer, which then moves past it).  Every replica at an admission
 * point with decode-ready requests then starts an iteration of its own batch
 * under the profile's cost law (B and K of that replica).  The controller sees
 * the node: every replica's words feed the per-second signal.  Idle (energy,
 * R18) = the whole node empty.  One replica is exactly orc_simulate (pinned by
 * tests); several require prefill_mode 0 and no KV capacity. */
int orc_simulate_replicas(const orc_request *req_words, uint64_t n_req, const orc_profile *prof,
                          const orc_ctrl *ctrl, const orc_run_cfg *cfg, orc_result *res, orc_log *log) {
  memset(res, 0, sizeof(*res));
  const uint32_t NR = prof->replicas ? prof->replicas : 1;
  if (NR > ORC_MAX_REPLICAS || prof->prefill_mode || prof->kv_cap_words) return -1;
  orc_request *req = (orc_request *)malloc((n_req ? n_req : 1) * sizeof(orc_request));
  if (!req) return -1;
  for (uint64_t i = 0; i < n_req; ++i) {
    req[i] = req_words[i];
    req[i].input = to_tokens(req_words[i].input, prof->tpw_q16);
  }
  res->first_act_s = res->last_deact_s = ORC_NONE;
  res->t1 = ctrl->t1;
  res->t2 = ctrl->t2;
  const uint64_t H = (uint64_t)cfg->horizon_us;
  int rc = -1;
  const uint64_t nq1 = n_req ? n_req : 1;
  rstate *rs = (rstate *)calloc(nq1, sizeof(rstate));
  uint32_t *rep = (uint32_t *)calloc(nq1, sizeof(uint32_t)); /* the replica a request was assigned to */
  uint32_t *queue = (uint32_t *)malloc(nq1 * sizeof(uint32_t));
  uint32_t *ready = (uint32_t *)malloc(NR * nq1 * sizeof(uint32_t)); /* [replica][...] */
  uint32_t *batch = (uint32_t *)malloc(NR * nq1 * sizeof(uint32_t));
  uint64_t *e2e_v = (uint64_t *)malloc(nq1 * sizeof(uint64_t));
  uint64_t *ttft_v = (uint64_t *)malloc(nq1 * sizeof(uint64_t));
  uint64_t n_sec = H / US + 2;
  uint64_t *sec_tbt_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_tbt_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_e2e_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_e2e_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_slo_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_ttft_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_ttft_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_in_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_in_any = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_util_sum = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  uint64_t *sec_util_cnt = (uint64_t *)calloc(n_sec, sizeof(uint64_t));
  orc_second_row *rows = (cfg->record & 2) ? (orc_second_row *)calloc(n_sec, sizeof(orc_second_row)) : NULL;
  heap h = {0, 0, 0};
  cstate cs;
  memset(&cs, 0, sizeof(cs));
  cs.c = ctrl;
  cs.law = ctrl->law;
  cs.rt_min = ORC_NONE;
  int busy[ORC_MAX_REPLICAS] = {0};
  uint64_t n_ready[ORC_MAX_REPLICAS] = {0}, n_batch[ORC_MAX_REPLICAS] = {0}, in_rep[ORC_MAX_REPLICAS] = {0};
  uint32_t rr = 0; /* round-robin pointer */
  if (!rs || !rep || !queue || !ready || !batch || !e2e_v || !ttft_v || !sec_tbt_sum || !sec_tbt_cnt ||
      !sec_e2e_sum || !sec_e2e_cnt || !sec_slo_cnt || !sec_ttft_sum || !sec_ttft_cnt || !sec_in_sum ||
      !sec_in_any || !sec_util_sum || !sec_util_cnt || ((cfg->record & 2) && !rows))
    goto out;
  if (cs.law == ORC_LAW_CONST) cs.r = ctrl->r_const_bp;
  for (uint64_t i = 0; i < n_req; ++i) {
    rs[i].admit = rs[i].first = rs[i].done = NEVER;
    if (heap_push(&h, (event){req[i].a_us, EV_ARRIVAL, (uint32_t)i, 0})) goto out;
  }
  uint64_t q_head = 0, q_tail = 0, in_sys = 0, n_e2e = 0, n_ttft = 0;
  uint64_t next_sec = 0, T_prev = 0, last_T = 0, n_series = 0;

#define COMPLETE(m, T, s_idx)                                                          \
  do {                                                                                 \
    uint64_t e2e_ = (T) - req[m].a_us;                                                 \
    rs[m].done = (T);                                                                  \
    rs[m].state = RS_DONE;                                                             \
    in_sys--;                                                                          \
    in_rep[rep[m]]--;                                                                  \
    res->served++;                                                                     \
    res->sum_e2e_us += e2e_;                                                           \
    res->sum_sojourn_us += e2e_;                                                       \
    e2e_v[n_e2e++] = e2e_;                                                             \
    res->hist_e2e[orc_lat_bin(e2e_ / 1000)]++;                                         \
    if (in_window((T), cfg)) res->win_served++;                                        \
    sec_e2e_sum[s_idx] += e2e_;                                                        \
    sec_e2e_cnt[s_idx] += 1;                                                           \
    if (e2e_ > ctrl->slo_us) { sec_slo_cnt[s_idx] += 1; res->slo_violations++; }       \
    if (rows) { rows[s_idx].completions++; rows[s_idx].sum_e2e_us += e2e_; }            \
  } while (0)

  for (;;) {
    if (h.n == 0) break;
    uint64_t T = h.v[0].t;
    if (T >= H) break;
    {
      uint64_t dt = T - T_prev, nq = q_tail - q_head;
      if (in_sys == 0) {
        res->idle_us += dt;
        res->win_idle_us += overlap(T_prev, T, cfg->w0_us, cfg->w1_us);
        if (rows)
          for (uint64_t s = T_prev / US; s * US < T && s < n_sec; ++s)
            rows[s].idle_us += (uint32_t)overlap(T_prev, T, (int64_t)(s * US), (int64_t)((s + 1) * US));
      }
      res->int_system_us += (nq + in_sys) * dt;
      res->int_queue_us += nq * dt;
    }
    T_prev = T;
    last_T = T;
    uint64_t s_idx = T / US;
    while (h.n && h.v[0].t == T) {
      event e = heap_pop(&h);
      if (e.kind == EV_ITER_END) { /* E1 on replica e.idx */
        const uint32_t q = e.idx;
        uint32_t *bq = batch + (uint64_t)q * nq1;
        sec_util_sum[s_idx] += n_batch[q];
        sec_util_cnt[s_idx] += 1;
        for (uint64_t b = 0; b < n_batch[q]; ++b) {
          uint32_t m = bq[b];
          uint64_t gap = T - rs[m].last_tok;
          sec_tbt_sum[s_idx] += gap;
          sec_tbt_cnt[s_idx] += 1;
          res->tbt_samples++;
          res->tbt_sum_us += gap;
          if (gap > res->tbt_max_us) res->tbt_max_us = gap;
          if (log && log->gaps && log->n_gaps < log->cap_gaps) {
            log->gaps[2 * log->n_gaps] = m;
            log->gaps[2 * log->n_gaps + 1] = gap;
          }
          if (log) log->n_gaps++;
          rs[m].n_gaps++;
          rs[m].last_tok = T;
          rs[m].emitted++;
          res->words_out++;
          if (rows) {
            rows[s_idx].tbt_count++;
            rows[s_idx].sum_tbt_us += gap;
            rows[s_idx].words_out++;
          }
          if (in_window(T, cfg)) res->win_words_out++;
          if (rs[m].emitted == rs[m].R) {
            COMPLETE(m, T, s_idx);
          } else {
            rs[m].state = RS_READY;
            ready[(uint64_t)q * nq1 + n_ready[q]++] = m;
          }
        }
        n_batch[q] = 0;
        busy[q] = 0;
      } else if (e.kind == EV_PREFILL_END) { /* E2: first word */
        uint32_t m = e.idx;
        uint64_t ttft = T - req[m].a_us;
        rs[m].first = T;
        rs[m].last_tok = T;
        rs[m].emitted = 1;
        res->words_out++;
        if (in_window(T, cfg)) res->win_words_out++;
        res->sum_ttft_us += ttft;
        sec_ttft_sum[s_idx] += ttft;
        sec_ttft_cnt[s_idx] += 1;
        ttft_v[n_ttft++] = ttft;
        res->hist_ttft[orc_lat_bin(ttft / 1000)]++;
        if (rows) {
          rows[s_idx].first_tokens++;
          rows[s_idx].sum_ttft_us += ttft;
          rows[s_idx].words_out++;
        }
        if (rs[m].R == 1) {
          COMPLETE(m, T, s_idx);
        } else {
          rs[m].state = RS_READY;
          ready[(uint64_t)rep[m] * nq1 + n_ready[rep[m]]++] = m;
        }
      } else { /* E3: arrival -> the central FIFO queue */
        uint32_t m = e.idx;
        rs[m].state = RS_QUEUED;
        queue[q_tail++] = m;
        res->arrivals++;
        if (rows) rows[s_idx].arrivals++;
        res->candidates = (uint64_t)req[m].j + 1;
      }
    }
    int any_idle = 0;
    for (uint32_t q = 0; q < NR; ++q) any_idle |= !busy[q];
    if (!any_idle) continue;
    INGEST_UNTIL(T);
    while (q_head < q_tail) {
      /* routing: a replica at an admission point with a free slot */
      uint32_t q = NR;
      if (prof->route == ORC_ROUTE_RR) {
        for (uint32_t i = 0; i < NR && q == NR; ++i) {
          uint32_t c = (rr + i) % NR;
          if (!busy[c] && in_rep[c] < prof->max_batch) q = c;
        }
        if (q < NR) rr = (q + 1) % NR;
      } else {
        for (uint32_t c = 0; c < NR; ++c)
          if (!busy[c] && in_rep[c] < prof->max_batch && (q == NR || in_rep[c] < in_rep[q])) q = c;
      }
      if (q == NR) break;
      uint32_t m = queue[q_head++];
      uint32_t r = cs.r;
      int bypass = r > 0 && (((ctrl->bypass_mask >> req[m].cls) & 1u) || req[m].P < ctrl->min_words_bypass);
      if (bypass) r = 0;
      const uint32_t R_words = r > 0 ? bounded_realized(req[m].P, r, req[m].fcomp_q16, cfg->poly_q16) : req[m].U;
      if (bypass) res->bypassed++;
      rep[m] = q;
      rs[m].admit = T;
      rs[m].r_bp = r;
      rs[m].R = to_tokens(R_words, prof->tpw_q16);
      uint64_t pf = ((uint64_t)prof->prefill_ns_per_word * req[m].input) / 1000;
      if (pf < 1) pf = 1;
      rs[m].prefill_end = T + pf;
      rs[m].state = RS_PREFILL;
      in_sys++;
      in_rep[q]++;
      res->admitted++;
      res->sum_queue_us += T - req[m].a_us;
      res->words_in += req[m].input;
      sec_in_sum[T / US] += req[m].input;
      sec_in_any[T / US] = 1;
      if (in_window(T, cfg)) res->win_words_in += req[m].input;
      if (rows) {
        rows[T / US].admitted++;
        rows[T / US].sum_queue_us += T - req[m].a_us;
        rows[T / US].words_in += req[m].input;
      }
      if (r > 0) {
        res->rewritten++;
        res->hist_r[r / 10 < ORC_HIST_R ? r / 10 : ORC_HIST_R - 1]++;
      }
      {
        uint32_t sc = orc_similarity(req[m].U, R_words, r > 0, req[m].qnoise, cfg->quality);
        uint32_t qb = sc / 50 < ORC_HIST_Q ? sc / 50 : ORC_HIST_Q - 1;
        if (r > 0) { res->hist_q_active[qb]++; res->scored_active++; }
        else { res->hist_q_inactive[qb]++; res->scored_inactive++; }
      }
      if (heap_push(&h, (event){rs[m].prefill_end, EV_PREFILL_END, m, 0})) goto out;
    }
    /* every replica at an admission point with decode-ready requests starts an iteration */
    for (uint32_t q = 0; q < NR; ++q) {
      if (busy[q] || n_ready[q] == 0) continue;
      uint64_t K = 0;
      uint32_t *bq = batch + (uint64_t)q * nq1;
      for (uint64_t b = 0; b < n_ready[q]; ++b) {
        uint32_t m = ready[(uint64_t)q * nq1 + b];
        bq[b] = m;
        rs[m].state = RS_DECODING;
        K += req[m].input + rs[m].emitted;
      }
      n_batch[q] = n_ready[q];
      n_ready[q] = 0;
      uint64_t B = n_batch[q];
      uint64_t d = prof->t0_us + (uint64_t)prof->slope_us * (B > prof->knee ? B - prof->knee : 0) +
                   ((uint64_t)prof->kv_ns_per_word * K) / 1000;
      if (heap_push(&h, (event){T + d, EV_ITER_END, q, 0})) goto out;
      busy[q] = 1;
      res->ticks++;
    }
  }
#undef COMPLETE
  uint64_t end = (cfg->mode == ORC_MODE_DRAIN && h.n == 0) ? last_T : H;
  {
    uint64_t dt = end - T_prev, nq = q_tail - q_head;
    if (in_sys == 0) {
      res->idle_us += dt;
      res->win_idle_us += overlap(T_prev, end, cfg->w0_us, cfg->w1_us);
      if (rows)
        for (uint64_t s = T_prev / US; s * US < end && s < n_sec; ++s)
          rows[s].idle_us += (uint32_t)overlap(T_prev, end, (int64_t)(s * US), (int64_t)((s + 1) * US));
    }
    res->int_system_us += (nq + in_sys) * dt;
    res->int_queue_us += nq * dt;
  }
  res->end_us = end;
  INGEST_UNTIL(end);
  res->queued_end = q_tail - q_head;
  res->inflight_end = in_sys;
  if (res->queued_end + res->inflight_end > 0) res->flags |= ORC_FLAG_TRUNCATED;
  finish_run(res, prof, e2e_v, n_e2e, ttft_v, n_ttft, rows, n_sec, end, n_series, rs, n_req, log);
  rc = 0;
out:
  free(req); free(rs); free(rep); free(queue); free(ready); free(batch); free(e2e_v); free(ttft_v);
  free(sec_tbt_sum); free(sec_tbt_cnt); free(sec_e2e_sum); free(sec_e2e_cnt); free(sec_slo_cnt);
  free(sec_ttft_sum); free(sec_ttft_cnt); free(sec_in_sum); free(sec_in_any); free(sec_util_sum);
  free(sec_util_cnt);
  free(h.v); free(cs.samples); free(cs.words); free(rows);
  return rc;
}

/* ------------------------------------------------------------------------- */
static void scenario_cfg(const orc_inputs *in, uint64_t sid, orc_profile *p, orc_ctrl *c, orc_run_cfg *cfg) {
  uint32_t pi = in->sc_profile[sid], ci = in->sc_ctrl[sid];
  p->t0_us = in->prof_t0[pi];
  p->knee = in->prof_knee[pi];
  p->slope_us = in->prof_slope[pi];
  p->kv_ns_per_word = in->prof_kv[pi];
  p->max_batch = in->prof_maxb[pi];
  p->prefill_ns_per_word = in->prof_prefill_ns[pi];
  p->e_in = in->prof_e_in[pi];
  p->e_out = in->prof_e_out[pi];
  p->p_idle = in->prof_p_idle[pi];
  p->kv_cap_words = in->prof_kv_cap[pi];
  p->prefill_mode = in->prof_prefill_mode[pi];
  p->kv_policy = in->prof_kv_policy[pi];
  p->tpw_q16 = in->prof_tpw[pi];
  p->replicas = in->prof_replicas[pi];
  p->route = in->prof_route[pi];
  memset(c, 0, sizeof(*c));
  c->law = in->ctrl_law[ci];
  c->signal = in->ctrl_signal[ci];
  c->window = in->ctrl_window[ci];
  c->r_min_bp = in->ctrl_rmin[ci];
  c->r_max_bp = in->ctrl_rmax[ci];
  c->r_const_bp = in->ctrl_rconst[ci];
  c->t1 = in->ctrl_t1[ci];
  c->t2 = in->ctrl_t2[ci];
  c->slo_us = in->ctrl_slo_us[ci];
  c->calibrated = in->ctrl_calibrated[ci];
  c->n_rungs = in->ctrl_nrungs[ci];
  for (int k = 0; k < 8; ++k) c->rungs_bp[k] = in->ctrl_rungs[8 * ci + k];
  c->bypass_mask = in->ctrl_bypass_mask[ci];
  c->min_words_bypass = in->ctrl_min_words[ci];
  c->horizon_s = in->ctrl_horizon[ci];
  c->w_lat = in->ctrl_wlat[ci];
  c->w_q = in->ctrl_wq[ci];
  c->w_osc = in->ctrl_wosc[ci];
  c->step_bp = in->ctrl_step[ci];
  cfg->mode = in->sc_mode[sid];
  cfg->horizon_us = in->sc_horizon[sid];
  cfg->w0_us = in->sc_w0[sid];
  cfg->w1_us = in->sc_w1[sid];
  for (int k = 0; k < 3; ++k) cfg->poly_q16[k] = in->poly_q16[k];
  for (int k = 0; k < 5; ++k) cfg->quality[k] = in->quality[k];
  cfg->record = in->sc_record[sid];
}

static int run_internal(const orc_inputs *in, uint64_t sid, int force_record, orc_result *res, orc_log *log) {
  orc_profile prof;
  orc_ctrl ctrl;
  orc_run_cfg cfg;
  scenario_cfg(in, sid, &prof, &ctrl, &cfg);
  if (force_record) cfg.record |= 1;
  uint32_t flags = 0;
  if (ctrl.calibrated && (ctrl.law == ORC_LAW_MAP || ctrl.law == ORC_LAW_STEP)) {
    /* a10: two-pass calibration from the paired unbounded run */
    uint64_t src = in->sc_calib_src[sid];
    uint64_t cap = (uint64_t)in->sc_horizon[src] / US + 2;
    uint32_t *series = (uint32_t *)malloc(cap * sizeof(uint32_t));
    orc_result *tmp = (orc_result *)malloc(sizeof(orc_result));
    if (!series || !tmp) { free(series); free(tmp); return -1; }
    orc_log slog;
    memset(&slog, 0, sizeof(slog));
    slog.series = series;
    slog.cap_series = cap;
    if (run_internal(in, src, 1, tmp, &slog)) { free(series); free(tmp); return -1; }
    uint32_t t1, t2;
    int st = orc_calibrate(series, tmp->n_series, &t1, &t2);
    ctrl.t1 = t1;
    ctrl.t2 = t2;
    if (st) { /* degenerate / insufficient -> controller off, flagged */
      flags |= ORC_FLAG_DEGENERATE_CALIB;
      ctrl.law = ORC_LAW_OFF;
    }
    free(series);
    free(tmp);
  }
  int64_t n = orc_arrivals(in, sid, NULL, 0);
  orc_request *req = (orc_request *)malloc((n > 0 ? (uint64_t)n : 1) * sizeof(orc_request));
  if (!req) return -1;
  if (orc_arrivals(in, sid, req, (uint64_t)n) != n) { free(req); return -1; }
  int rc = orc_simulate(req, (uint64_t)n, &prof, &ctrl, &cfg, res, log);
  res->flags |= flags;
  free(req);
  return rc;
}

int orc_run_scenario(const orc_inputs *in, uint64_t sid, orc_result *res, orc_log *log) {
  if (sid >= in->n_scenarios) return -1;
  return run_internal(in, sid, 0, res, log);
}

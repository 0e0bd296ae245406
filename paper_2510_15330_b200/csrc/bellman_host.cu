// bellman_host.cu — C ABI of the beLLMan simulator (include/bellman_sim.h):
// validation, workspace layout, host-side precomputation, launches.
#include <cuda.h>  // CUdeviceptr / CUresult types only (the driver call is resolved at run time)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <new>
#include <unordered_map>
#include <vector>

#include "bellman_internal.cuh"

using namespace bellman;

// K2L (the lane-per-scenario kernel) is a throughput engine: 32 scenarios per
// warp, one CTA of 5-7 warps per SM, so it needs several scenarios per lane
// (B200: 23-33k lanes) to beat the warp engine, which runs each scenario's
// serial chain faster.  A run takes K2L for the scenarios within its bounds
// when it has at least kLaneMinScenarios of them in total (C5 and its 8-way
// shards; C1-C4 stay on K2), unless the environment sets BELLMAN_LANE=0 (A/B
// measurements), or BELLMAN_LANE=2 (every run, any size: parity tests of K2L
// on small sets).  Read at workspace sizing, create and run.
constexpr uint64_t kLaneMinScenarios = 65536;
static uint32_t lane_mode() {
  const char *e = std::getenv("BELLMAN_LANE");
  return e ? (e[0] == '0' ? 0u : (e[0] == '2' ? 2u : 1u)) : 1u;
}

static uint32_t kind_of(const bellman_sim_desc *d, const bellman_scenario &sc, uint32_t lane_on) {
  return scenario_kind_of(sc, d->ctrls[sc.ctrl], d->profiles[sc.profile], d->traces[sc.trace].kind, lane_on);
}

// whether a descriptor's workspace carries K2L's histograms
static bool lane_possible(const bellman_sim_desc *d) {
  if (lane_mode() == 0 || (lane_mode() == 1 && d->n_scenarios < kLaneMinScenarios)) return false;
  for (uint64_t s = 0; s < d->n_scenarios; ++s)
    if (kind_of(d, d->scenarios[s], 1u) >= 3u) return true;
  return false;
}

struct bellman_sim {
  int device = 0;
  uint64_t n_scenarios = 0;
  uint32_t n_segments = 0, n_slots = 0;
  bool has_calibrated = false;
  int grid = 0;
  uint32_t last_launches = 0;
  uint32_t last_engines = 0;  // BELLMAN_ENGINE_* of the last run (bit k = scenario kind k)
  Params params{};
  unsigned int *counters = nullptr;  // [16]: one per launch of a run
  bool has_dbg = false;
  bool has_kind[2][2][5] = {};       // [K2L on][debug-recorded][kind]: some scenario runs in that kernel
  int lane_grid = 0;                 // K2L CTAs (one per SM)
  bool lane_ok = false;              // the workspace holds K2L's per-thread histograms
  std::vector<uint8_t> calibrated;   // per scenario: ctrl is calibrated
  std::vector<uint32_t> calib_src;
  std::vector<uint32_t> dbg_slot;    // per scenario: debug-record slot or NONE
  std::vector<uint64_t> dbg_off;
  std::vector<uint32_t> dbg_cap;
  const uint32_t *order = nullptr;   // device: scenarios by decreasing expected work
  uint32_t *shard_order = nullptr;   // device: the heavy-first order of the last strided shard run
  std::vector<uint32_t> host_order;  // host copy of `order`
  std::vector<uint32_t> host_shard;  // host copy of `shard_order` (its key below)
  uint64_t shard_key[3] = {~0ull, ~0ull, ~0ull};  // (first, stride, count) that host_shard holds
  uint64_t shard_gen = 0;            // this handle's upload stamp (see shard_region_owner)
  char err[512] = {0};
};

static thread_local char g_err[512];

// Several handles may be created on one caller-owned workspace (one at a time
// in use).  The shard-order region is written by bellman_sim_run, so a handle
// may reuse its cached upload only if no other handle wrote that region since:
// every upload stamps the region's address with a fresh generation.
static std::mutex g_shard_mu;
static std::unordered_map<const void *, uint64_t> g_shard_owner;
static uint64_t g_shard_gen = 0;

static bellman_status fail(bellman_sim *sim, bellman_status st, const char *fmt, ...) {
  char *dst = sim ? sim->err : g_err;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(dst, 512, fmt, ap);
  va_end(ap);
  return st;
}

#define CUDA_TRY(sim, call)                                                                   \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(sim, BELLMAN_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                  \
  } while (0)

// ---------------------------------------------------------------------------
// validation (S:185 max_batch >= 1, knee <= max_batch; S:269 0 < r_min <= r_max < 1,
// t1 < t2, window >= 1; S:51 positive durations, non-negative rates)
// One scenario's descriptor checks; `report` writes the message (the caller's
// thread only: the message buffer is thread-local).
#define REPORT(...) (report ? fail(nullptr, BELLMAN_EINVAL, __VA_ARGS__) : BELLMAN_EINVAL)
static bellman_status check_scenario(const bellman_sim_desc *d, uint64_t s, bool report) {
  const bellman_scenario &sc = d->scenarios[s];
  if (sc.trace >= d->n_traces || sc.profile >= d->n_profiles || sc.ctrl >= d->n_ctrls)
    return REPORT("scenario %llu: index out of range", (unsigned long long)s);
  if (sc.segment >= d->n_segments) return REPORT("scenario %llu: segment out of range", (unsigned long long)s);
  if (sc.mode > BELLMAN_MODE_DRAIN) return REPORT("scenario %llu: bad mode", (unsigned long long)s);
  if (sc.horizon_us <= 0 || sc.horizon_us > (1ll << 43))
    return REPORT("scenario %llu: horizon out of range", (unsigned long long)s);
  if (sc.w0_us > sc.w1_us) return REPORT("scenario %llu: w0 > w1", (unsigned long long)s);
  {  // the kernel counts iterations in 32 bits: every iteration starts before H and lasts >= t0
     // (a contending prefill-only iteration >= 1 µs), so ticks <= H / min_iter + 1 must stay < 2^32
    const bellman_profile &pf = d->profiles[sc.profile];
    const uint64_t min_iter = pf.prefill_mode == BELLMAN_PREFILL_CONTENDING ? 1u : pf.t0_us;
    // horizon / min_iter + 1 >= 2^32 - 1, without a 64-bit division per scenario
    if ((uint64_t)sc.horizon_us >= 0xFFFFFFFEull * min_iter)
      return REPORT("scenario %llu: horizon / t0 allows >= 2^32 iterations",
                  (unsigned long long)s);
  }
  const bellman_ctrl &c = d->ctrls[sc.ctrl];
  if (c.calibrated && (c.law == BELLMAN_LAW_MAP || c.law == BELLMAN_LAW_STEP)) {
    if (sc.calib_src >= d->n_scenarios) return REPORT("scenario %llu: calib_src out of range", (unsigned long long)s);
    const bellman_scenario &src = d->scenarios[sc.calib_src];
    const bellman_ctrl &sctl = d->ctrls[src.ctrl];
    if (sctl.calibrated || sctl.law != BELLMAN_LAW_OFF)
      return REPORT("scenario %llu: calibration source must be an OFF run", (unsigned long long)s);
    if (sctl.signal != c.signal)
      return REPORT("scenario %llu: calibration source records another signal", (unsigned long long)s);
  }
  return BELLMAN_OK;
}
#undef REPORT

// Runs f(lo, hi, chunk) over [0, n) on up to 16 host threads (one chunk each);
// sets under 32k elements run inline.
static std::mutex g_par_mu;
template <class F>
static void parallel_chunks(uint64_t n, F f) {
  unsigned nt = std::thread::hardware_concurrency();
  nt = nt < 1 ? 1 : (nt > 16 ? 16 : nt);
  if (n < (1u << 15)) nt = 1;
  const uint64_t step = (n + nt - 1) / nt;
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nt; ++t) {
    const uint64_t lo = t * step, hi = std::min<uint64_t>(n, lo + step);
    if (lo < hi) th.emplace_back(f, lo, hi, t);
  }
  f(0, std::min<uint64_t>(n, step), 0u);
  for (auto &x : th) x.join();
}

static bellman_status validate(const bellman_sim_desc *d) {
  if (!d) return fail(nullptr, BELLMAN_EINVAL, "desc is NULL");
  if (d->n_traces && (!d->traces || !d->knots)) return fail(nullptr, BELLMAN_EINVAL, "traces/knots NULL");
  if (!d->n_profiles || !d->profiles) return fail(nullptr, BELLMAN_EINVAL, "no profiles");
  if (!d->n_ctrls || !d->ctrls) return fail(nullptr, BELLMAN_EINVAL, "no controller configs");
  if (d->n_scenarios && !d->scenarios) return fail(nullptr, BELLMAN_EINVAL, "scenarios NULL");
  if (d->n_scenarios >= 0xFFFFFFFFull) return fail(nullptr, BELLMAN_EINVAL, "too many scenarios");
  if (!d->n_segments) return fail(nullptr, BELLMAN_EINVAL, "n_segments must be >= 1");
  const bellman_models &m = d->models;
  if (!m.L_words || !m.I_words || !m.fvar_q16 || !m.noise || !m.fcomp_q16 || !m.qnoise)
    return fail(nullptr, BELLMAN_EINVAL, "model tables NULL");
  if (!(m.quality[2] <= m.quality[1] && m.quality[1] <= m.quality[0] && m.quality[0] <= 10000))
    return fail(nullptr, BELLMAN_EINVAL, "quality: need floor <= active <= inactive <= 10000");
  if (!(m.quality[3] > 0 && m.quality[3] < m.quality[4] && m.quality[4] <= 10000))
    return fail(nullptr, BELLMAN_EINVAL, "quality: need 0 < safe_bp < end_bp <= 10000");
  if (!(m.class_cum[0] <= m.class_cum[1] && m.class_cum[1] <= m.class_cum[2] && m.class_cum[2] <= m.class_cum[3] &&
        m.class_cum[3] == (1u << 20)))
    return fail(nullptr, BELLMAN_EINVAL, "class_cum must be non-decreasing with class_cum[3] = 2^20");
  for (int i = 0; i < BELLMAN_TABLE_N; ++i) {
    if (m.L_words[i] < 1 || m.L_words[i] > 65535) return fail(nullptr, BELLMAN_EINVAL, "L table[%d] out of range", i);
    if (m.I_words[i] < 1 || m.I_words[i] > 65535) return fail(nullptr, BELLMAN_EINVAL, "I table[%d] out of range", i);
    if (m.fvar_q16[i] < 1 || m.fvar_q16[i] > (1 << 18)) return fail(nullptr, BELLMAN_EINVAL, "fvar[%d] out of range", i);
    if (m.noise[i] < -65535 || m.noise[i] > 65535) return fail(nullptr, BELLMAN_EINVAL, "noise[%d] out of range", i);
    if (m.fcomp_q16[i] < 0 || m.fcomp_q16[i] > (1 << 18)) return fail(nullptr, BELLMAN_EINVAL, "fcomp[%d] out of range", i);
    if (m.qnoise[i] < -2047 || m.qnoise[i] > 2047) return fail(nullptr, BELLMAN_EINVAL, "qnoise[%d] out of range", i);
  }
  for (int k = 0; k < 3; ++k)
    if (m.poly_q16[k] > (1ll << 40) || m.poly_q16[k] < -(1ll << 40))
      return fail(nullptr, BELLMAN_EINVAL, "poly_q16[%d] out of range", k);
  for (uint32_t t = 0; t < d->n_traces; ++t) {
    const bellman_trace &tr = d->traces[t];
    if (tr.kind > 1) return fail(nullptr, BELLMAN_EINVAL, "trace %u: unknown kind", t);
    if (tr.kind == 1) {  // NEXT-4 replay list
      if ((uint64_t)tr.knot_offset + tr.n_knots > d->n_arrivals || (tr.n_knots && !d->arrivals))
        return fail(nullptr, BELLMAN_EINVAL, "trace %u: bad arrival range", t);
      for (uint32_t k = 0; k < tr.n_knots; ++k) {
        const bellman_arrival &a = d->arrivals[tr.knot_offset + k];
        if (a.a_us < 0 || a.a_us > (1ll << 43) || a.L_words < 1 || a.L_words > 65535 || a.input_words < 1 ||
            a.input_words > 65535 || a.cls > 3)
          return fail(nullptr, BELLMAN_EINVAL, "trace %u arrival %u: field out of range", t, k);
        if (k && a.a_us < d->arrivals[tr.knot_offset + k - 1].a_us)
          return fail(nullptr, BELLMAN_EINVAL, "trace %u: arrivals not sorted at %u", t, k);
      }
      continue;
    }
    if (tr.n_knots < 2 || (uint64_t)tr.knot_offset + tr.n_knots > d->n_knots)
      return fail(nullptr, BELLMAN_EINVAL, "trace %u: bad knot range", t);
    for (uint32_t k = 0; k < tr.n_knots; ++k) {
      const bellman_knot &kn = d->knots[tr.knot_offset + k];
      if (kn.t_us < 0 || kn.t_us > (1ll << 43)) return fail(nullptr, BELLMAN_EINVAL, "trace %u knot %u: time out of range", t, k);
      if (kn.lam_mrps > (1u << 20)) return fail(nullptr, BELLMAN_EINVAL, "trace %u knot %u: rate > 2^20 mRPS", t, k);
      if (k && kn.t_us < d->knots[tr.knot_offset + k - 1].t_us)
        return fail(nullptr, BELLMAN_EINVAL, "trace %u: knot times decrease at %u", t, k);
    }
  }
  for (uint32_t i = 0; i < d->n_profiles; ++i) {
    const bellman_profile &p = d->profiles[i];
    if (p.max_batch < 1 || p.max_batch > BELLMAN_MAX_BATCH) return fail(nullptr, BELLMAN_EINVAL, "profile %u: max_batch not in 1..64", i);
    if (p.knee > p.max_batch) return fail(nullptr, BELLMAN_EINVAL, "profile %u: knee > max_batch", i);
    if (p.t0_us < 1 || p.t0_us > (1u << 24)) return fail(nullptr, BELLMAN_EINVAL, "profile %u: t0_us not in 1..2^24", i);
    if (p.slope_us > (1u << 16)) return fail(nullptr, BELLMAN_EINVAL, "profile %u: slope_us > 2^16", i);
    if (p.prefill_ns_per_word > (1u << 24)) return fail(nullptr, BELLMAN_EINVAL, "profile %u: prefill too large", i);
    if (p.kv_ns_per_word > 1024u) return fail(nullptr, BELLMAN_EINVAL, "profile %u: kv_ns_per_word > 1024", i);
    if (p.kv_cap_words > (1u << 30)) return fail(nullptr, BELLMAN_EINVAL, "profile %u: kv_cap_words > 2^30", i);
    if (p.prefill_mode > BELLMAN_PREFILL_CONTENDING) return fail(nullptr, BELLMAN_EINVAL, "profile %u: unknown prefill_mode", i);
    if (p.kv_policy > BELLMAN_KV_PREEMPT) return fail(nullptr, BELLMAN_EINVAL, "profile %u: unknown kv_policy", i);
    if (p.kv_policy == BELLMAN_KV_PREEMPT && p.prefill_mode != BELLMAN_PREFILL_NONBLOCKING)
      return fail(nullptr, BELLMAN_EINVAL, "profile %u: kv_policy 1 (preempt) needs prefill_mode 0", i);
    // a recompute prefill covers a preempted context, at most the capacity plus one iteration's and one
    // instant's words (a request over the capacity alone is never preempted): keep it < 2^30 µs (32-bit clock)
    if (p.kv_policy == BELLMAN_KV_PREEMPT &&
        (uint64_t)p.prefill_ns_per_word * ((uint64_t)p.kv_cap_words + 2u * BELLMAN_MAX_BATCH) / 1000u >= (1ull << 30))
      return fail(nullptr, BELLMAN_EINVAL, "profile %u: kv_policy 1: prefill of the capacity >= 2^30 us", i);
    // contending prefill: one iteration may carry max_batch prefills; keep it < 2^30 µs (32-bit clock)
    if (p.prefill_mode == BELLMAN_PREFILL_CONTENDING &&
        (uint64_t)p.max_batch * ((uint64_t)p.prefill_ns_per_word * 65535u / 1000u + 1u) >= (1ull << 30))
      return fail(nullptr, BELLMAN_EINVAL, "profile %u: contending prefill: max_batch x max prefill >= 2^30 us", i);
    if (p.replicas > BELLMAN_MAX_REPLICAS) return fail(nullptr, BELLMAN_EINVAL, "profile %u: replicas > 8", i);
    if (p.route > BELLMAN_ROUTE_RR) return fail(nullptr, BELLMAN_EINVAL, "profile %u: unknown route", i);
    if (p.replicas > 1u) {
      if (p.replicas * p.max_batch > BELLMAN_MAX_BATCH)
        return fail(nullptr, BELLMAN_EINVAL, "profile %u: replicas x max_batch > 64", i);
      if (p.prefill_mode != BELLMAN_PREFILL_NONBLOCKING || p.kv_cap_words != 0u)
        return fail(nullptr, BELLMAN_EINVAL, "profile %u: replicas > 1 needs prefill_mode 0 and no KV capacity", i);
    }
    if (p.tpw_q16 != 0u && (p.tpw_q16 < 16384u || p.tpw_q16 > 262144u))
      return fail(nullptr, BELLMAN_EINVAL, "profile %u: tpw_q16 not 0 or in 16384..262144 (0.25..4 tokens/word)", i);
    if (p.tpw_q16 != 0u) {  // inputs are 16-bit token counts on the device
      uint32_t max_in = 0;
      for (int k = 0; k < BELLMAN_TABLE_N; ++k) max_in = std::max(max_in, (uint32_t)m.I_words[k]);
      for (uint64_t k = 0; k < d->n_arrivals; ++k) max_in = std::max(max_in, d->arrivals[k].input_words);
      if ((((uint64_t)max_in * p.tpw_q16 + (1u << 15)) >> 16) > 65535u)
        return fail(nullptr, BELLMAN_EINVAL, "profile %u: an input of %u words is >= 65536 tokens", i, max_in);
    }
    if (!(p.e_in_j_per_word >= 0) || !(p.e_out_j_per_word >= 0) || !(p.p_idle_w >= 0))
      return fail(nullptr, BELLMAN_EINVAL, "profile %u: negative energy coefficient", i);
  }
  for (uint32_t i = 0; i < d->n_ctrls; ++i) {
    const bellman_ctrl &c = d->ctrls[i];
    if (c.law > BELLMAN_LAW_PCC) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: unknown law", i);
    if (c.signal > BELLMAN_SIG_UTIL) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: unknown signal", i);
    if (c.bypass_mask > 15u) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: bypass_mask has bits beyond 4 classes", i);
    if (c.window < 1 || c.window > 8) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: window not in 1..8", i);
    if (c.n_rungs > 8) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: more than 8 rungs", i);
    if (c.law == BELLMAN_LAW_CONST && c.r_const_bp > 5000) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: r_const > 5000 bp", i);
    if (c.law == BELLMAN_LAW_MAP || c.law == BELLMAN_LAW_STEP) {
      if (c.r_min_bp < 1 || c.r_min_bp > c.r_max_bp || c.r_max_bp > 5000)
        return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: need 0 < r_min <= r_max <= 5000 bp", i);
      if (!c.calibrated && c.t1 >= c.t2) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: need t1 < t2", i);
      if (c.law == BELLMAN_LAW_STEP && c.n_rungs == 0) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: STEP needs rungs", i);
      if (c.n_rungs) {
        for (uint32_t k = 1; k < c.n_rungs; ++k)
          if (c.rungs_bp[k] <= c.rungs_bp[k - 1]) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: rungs not ascending", i);
        if (c.rungs_bp[0] != c.r_min_bp || c.rungs_bp[c.n_rungs - 1] != c.r_max_bp)
          return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: rungs must span [r_min, r_max]", i);
      }
    }
    if (c.law >= BELLMAN_LAW_MPC) {  // NEXT-3 MPC / BBR / PCC
      if (c.r_min_bp < 1 || c.r_min_bp > c.r_max_bp || c.r_max_bp > 5000)
        return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: need 0 < r_min <= r_max <= 5000 bp", i);
      if (c.calibrated) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: calibration is for MAP / STEP only", i);
      if (c.w_lat > 65535u || c.w_q > 65535u || c.w_osc > 65535u)
        return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: cost weights must be <= 65535", i);
      if (c.n_rungs) {
        for (uint32_t k = 1; k < c.n_rungs; ++k)
          if (c.rungs_bp[k] <= c.rungs_bp[k - 1]) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: rungs not ascending", i);
        if (c.rungs_bp[0] != c.r_min_bp || c.rungs_bp[c.n_rungs - 1] != c.r_max_bp)
          return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: rungs must span [r_min, r_max]", i);
      }
      if (c.law == BELLMAN_LAW_MPC) {
        if (c.horizon_s > 16u) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: MPC horizon_s > 16", i);
        if (c.w_lat < 1u) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: MPC needs w_lat >= 1", i);
      } else if (c.law == BELLMAN_LAW_BBR) {
        if (c.signal != BELLMAN_SIG_TBT) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: BBR needs the TBT signal", i);
        if (!c.n_rungs && (c.step_bp < 1u || c.step_bp > 5000u))
          return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: BBR needs 1 <= step_bp <= 5000 or rungs", i);
      } else {
        if (c.n_rungs) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: PCC takes no rungs", i);
        if (c.step_bp < 1u || c.step_bp > 5000u) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: PCC needs 1 <= step_bp <= 5000", i);
        if (c.w_lat < 1u) return fail(nullptr, BELLMAN_EINVAL, "ctrl %u: PCC needs w_lat >= 1", i);
      }
    }
  }
  // per-scenario checks on host threads (C5: 2^20 scenarios, a memory-bound
  // pass over 64 MB); the message names the lowest failing scenario
  uint64_t bad = ~0ull;
  parallel_chunks(d->n_scenarios, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t s = lo; s < hi; ++s)
      if (check_scenario(d, s, false) != BELLMAN_OK) {
        std::lock_guard<std::mutex> lk(g_par_mu);
        if (s < bad) bad = s;
        return;
      }
  });
  if (bad != ~0ull) return check_scenario(d, bad, true);
  return BELLMAN_OK;
}

// ---------------------------------------------------------------------------
struct Layout {
  size_t off_sc, off_tr, off_seg, off_prof, off_ctrl, off_tab, off_log2, off_slot, off_soff, off_scap,
      off_sn, off_series, off_calib, off_stats, off_hist, off_cnt, off_dslot, off_doff, off_dcap, off_dn,
      off_drows, off_dctrl, off_arr, off_ord, off_sord, off_pre, off_lhist, off_lfifo, off_cmag, total;
  size_t in_end;              // [0, in_end): host-filled inputs, one staging copy at create
  size_t zero_beg, zero_end;  // [zero_beg, zero_end): zeroed at create (counters, stats, histograms)
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct HostPrep {
  std::vector<DevTrace> traces;
  std::vector<DevSeg> segs;
  std::vector<uint32_t> slot_of;   // per scenario
  std::vector<uint64_t> slot_off;  // per slot
  std::vector<uint32_t> slot_cap;
  uint64_t series_words = 0;
  std::vector<uint32_t> dbg_of;    // per scenario
  std::vector<uint64_t> dbg_off;   // per debug slot, in rows
  std::vector<uint32_t> dbg_cap;
  uint64_t dbg_rows = 0;
  std::vector<uint32_t> order;     // scenarios by decreasing expected arrivals (stable)
};

// Expected arrivals of a scenario: the integral of its trace's rate over
// [0, horizon) (kind 0) or the listed arrivals before the horizon (kind 1),
// capped by arrival_cap.  Used only to order the work (heavy scenarios first,
// so that the longest serial chains start at once and on distinct SM
// sub-partitions); results do not depend on the order.
static double expected_arrivals(const bellman_sim_desc *d, const bellman_scenario &sc) {
  const bellman_trace &tr = d->traces[sc.trace];
  const double H = (double)sc.horizon_us;
  double n = 0;
  if (tr.kind == 1) {
    const bellman_arrival *a = d->arrivals + tr.knot_offset;
    n = (double)(std::lower_bound(a, a + tr.n_knots, sc.horizon_us,
                                  [](const bellman_arrival &x, int64_t h) { return x.a_us < h; }) - a);
  } else {
    for (uint32_t k = 0; k + 1 < tr.n_knots; ++k) {
      const bellman_knot &a = d->knots[tr.knot_offset + k], &b = d->knots[tr.knot_offset + k + 1];
      const double ta = (double)a.t_us, tb = (double)b.t_us;
      if (tb <= ta || ta >= H) continue;
      const double te = tb < H ? tb : H;
      const double le = a.lam_mrps + ((double)b.lam_mrps - a.lam_mrps) * (te - ta) / (tb - ta);
      n += 0.5 * (a.lam_mrps + le) * (te - ta) * 1e-9;  // mRPS x µs
    }
  }
  if (tr.arrival_cap && n > tr.arrival_cap) n = tr.arrival_cap;
  return n;
}

static void prepare(const bellman_sim_desc *d, HostPrep &h) {
  h.segs.clear();
  h.slot_off.clear();
  h.slot_cap.clear();
  h.series_words = 0;
  h.dbg_off.clear();
  h.dbg_cap.clear();
  h.dbg_rows = 0;
  h.traces.resize(d->n_traces);
  for (uint32_t t = 0; t < d->n_traces; ++t) {
    const bellman_trace &tr = d->traces[t];
    if (tr.kind == 1) {  // replay: seg_off / n_seg index the device copy of desc->arrivals
      h.traces[t] = DevTrace{tr.knot_offset, tr.n_knots, tr.arrival_cap, 1u};
      continue;
    }
    DevTrace dt{(uint32_t)h.segs.size(), 0, tr.arrival_cap, 0};
    for (uint32_t k = 0; k + 1 < tr.n_knots; ++k) {
      const bellman_knot &a = d->knots[tr.knot_offset + k], &b = d->knots[tr.knot_offset + k + 1];
      const uint32_t lmax = a.lam_mrps > b.lam_mrps ? a.lam_mrps : b.lam_mrps;
      if (lmax == 0 || b.t_us <= a.t_us) continue;  // a zero-rate or empty phase draws no candidate
      DevSeg s{};
      s.ta = (uint64_t)a.t_us;
      s.tb = (uint64_t)b.t_us;
      s.span = s.tb - s.ta;
      s.M = (uint64_t)(((unsigned __int128)1000000000ull << 32) / lmax);  // mean gap 1e9/lmax µs, Q32
      s.la = a.lam_mrps;
      s.lb = b.lam_mrps;
      s.lmax = lmax;
      h.segs.push_back(s);
      dt.n_seg++;
    }
    h.traces[t] = dt;
  }
  // One pass over the scenario table (64 B per scenario: at C5's 2^20 the passes
  // are memory-bound, ~10 ms each): series slots (every recorded scenario and
  // every calibration source), debug-record slots, and the heavy-first cost rank.
  // The cost depends only on (trace, horizon): evaluated once per distinct pair.
  h.slot_of.assign(d->n_scenarios, BELLMAN_NONE);
  h.dbg_of.assign(d->n_scenarios, BELLMAN_NONE);
  // scratch reused across calls; bound to references here because the worker
  // threads below would otherwise name their own thread_local instances
  static thread_local std::vector<uint8_t> need_tls;
  static thread_local std::vector<uint32_t> rank_tls;
  std::vector<uint8_t> &need = need_tls;
  std::vector<uint32_t> &rank = rank_tls;
  need.assign(d->n_scenarios, 0);
  rank.resize(d->n_scenarios);
  std::vector<double> costs;  // distinct costs, in first-seen order
  {
    // on host threads, one chunk of scenarios each: the chunk's distinct
    // (trace << 44 | horizon) keys in first-seen order and chunk-local ranks;
    // merged below in chunk order, so the result is the sequential pass's
    struct Chunk {
      std::vector<uint64_t> keys;    // distinct keys, first-seen order
      std::vector<uint64_t> first;   // a scenario with that key
      std::vector<uint64_t> calib;   // calibration sources named by the chunk
      std::vector<uint64_t> dbg;     // debug-recorded scenarios of the chunk
    };
    std::vector<Chunk> ch(16);
    parallel_chunks(d->n_scenarios, [&](uint64_t lo, uint64_t hi, unsigned t) {
      Chunk &c = ch[t];
      std::unordered_map<uint64_t, uint32_t> memo;
      uint64_t last_key = ~0ull;  // consecutive scenarios usually share the key: skip the lookup
      uint32_t last_rank = 0;
      for (uint64_t s = lo; s < hi; ++s) {
        const bellman_scenario &sc = d->scenarios[s];
        if (sc.record & BELLMAN_RECORD_SIGNAL) need[s] = 1;
        const bellman_ctrl &cc = d->ctrls[sc.ctrl];
        if (cc.calibrated && (cc.law == BELLMAN_LAW_MAP || cc.law == BELLMAN_LAW_STEP)) c.calib.push_back(sc.calib_src);
        if (sc.record & BELLMAN_RECORD_SECONDS) c.dbg.push_back(s);
        const uint64_t key = ((uint64_t)sc.trace << 44) | (uint64_t)sc.horizon_us;  // horizon <= 2^43 (validated)
        if (key != last_key) {
          auto it = memo.find(key);
          if (it == memo.end()) {
            it = memo.emplace(key, (uint32_t)c.keys.size()).first;
            c.keys.push_back(key);
            c.first.push_back(s);
          }
          last_key = key;
          last_rank = it->second;
        }
        rank[s] = last_rank;  // chunk-local for now
      }
    });
    std::unordered_map<uint64_t, uint32_t> memo;  // key -> index into costs
    std::vector<std::vector<uint32_t>> remap(ch.size());
    for (size_t t = 0; t < ch.size(); ++t) {
      for (size_t k = 0; k < ch[t].keys.size(); ++k) {
        auto it = memo.find(ch[t].keys[k]);
        if (it == memo.end()) {
          it = memo.emplace(ch[t].keys[k], (uint32_t)costs.size()).first;
          costs.push_back(expected_arrivals(d, d->scenarios[ch[t].first[k]]));
        }
        remap[t].push_back(it->second);
      }
      for (uint64_t src : ch[t].calib) need[src] = 1;
      for (uint64_t s : ch[t].dbg) {
        h.dbg_of[s] = (uint32_t)h.dbg_off.size();
        const uint64_t cap = (uint64_t)d->scenarios[s].horizon_us / kUs + 2;
        h.dbg_off.push_back(h.dbg_rows);
        h.dbg_cap.push_back((uint32_t)cap);
        h.dbg_rows += cap;
      }
    }
    parallel_chunks(d->n_scenarios, [&](uint64_t lo, uint64_t hi, unsigned t) {
      const std::vector<uint32_t> &m = remap[t];
      for (uint64_t s = lo; s < hi; ++s) rank[s] = m[rank[s]];
    });
  }
  for (uint64_t s = 0; s < d->n_scenarios; ++s) {
    if (!need[s]) continue;
    h.slot_of[s] = (uint32_t)h.slot_off.size();
    const uint64_t cap = (uint64_t)d->scenarios[s].horizon_us / kUs + 2;
    h.slot_off.push_back(h.series_words);
    h.slot_cap.push_back((uint32_t)cap);
    h.series_words += cap;
  }
  std::vector<uint32_t> by_cost(costs.size());  // distinct cost indices by decreasing cost
  for (uint32_t i = 0; i < by_cost.size(); ++i) by_cost[i] = i;
  std::sort(by_cost.begin(), by_cost.end(), [&](uint32_t a, uint32_t b) { return costs[a] > costs[b]; });
  // equal costs (from different (trace, horizon) pairs) share one group, so ids
  // of equal cost keep their id order (the stable sort's tie rule)
  std::vector<uint32_t> group(costs.size());
  uint32_t ng = 0;
  for (uint32_t i = 0; i < by_cost.size(); ++i) {
    if (i && costs[by_cost[i]] != costs[by_cost[i - 1]]) ng++;
    group[by_cost[i]] = ng;
  }
  // counting sort by group, stable: per-chunk counts (host threads), the
  // chunks' offsets in chunk order, then each chunk scatters its ids
  h.order.resize(d->n_scenarios);
  if (!costs.empty()) {
    const uint32_t G = ng + 1;
    std::vector<std::vector<uint64_t>> cnt(16, std::vector<uint64_t>(G, 0));
    parallel_chunks(d->n_scenarios, [&](uint64_t lo, uint64_t hi, unsigned t) {
      std::vector<uint64_t> &c = cnt[t];
      for (uint64_t s = lo; s < hi; ++s) c[group[rank[s]]]++;
    });
    uint64_t at = 0;
    for (uint32_t g = 0; g < G; ++g)
      for (size_t t = 0; t < cnt.size(); ++t) {  // group-major, then chunk order: the stable order
        const uint64_t n = cnt[t][g];
        cnt[t][g] = at;
        at += n;
      }
    parallel_chunks(d->n_scenarios, [&](uint64_t lo, uint64_t hi, unsigned t) {
      std::vector<uint64_t> &c = cnt[t];
      for (uint64_t s = lo; s < hi; ++s) h.order[c[group[rank[s]]]++] = (uint32_t)s;
    });
  }
}

static Layout layout(const bellman_sim_desc *d, const HostPrep &h) {
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  const size_t ns = h.slot_off.size();
  const size_t nd = h.dbg_off.size();
  // host-filled inputs, contiguous: one H2D copy from a staging buffer
  L.off_sc = take(sizeof(bellman_scenario) * d->n_scenarios);
  L.off_tr = take(sizeof(DevTrace) * h.traces.size());
  L.off_seg = take(sizeof(DevSeg) * h.segs.size());
  L.off_prof = take(sizeof(bellman_profile) * d->n_profiles);
  L.off_ctrl = take(sizeof(bellman_ctrl) * d->n_ctrls);
  L.off_tab = take(sizeof(int32_t) * 6 * BELLMAN_TABLE_N);
  L.off_log2 = take(sizeof(uint2) * BELLMAN_TABLE_N);
  L.off_slot = take(sizeof(uint32_t) * d->n_scenarios);
  L.off_soff = take(sizeof(uint64_t) * ns);
  L.off_scap = take(sizeof(uint32_t) * ns);
  L.off_dslot = take(sizeof(uint32_t) * d->n_scenarios);
  L.off_doff = take(sizeof(uint64_t) * nd);
  L.off_dcap = take(sizeof(uint32_t) * nd);
  L.off_arr = take(sizeof(bellman_arrival) * d->n_arrivals);
  L.off_ord = take(sizeof(uint32_t) * d->n_scenarios);
  L.off_cmag = take(sizeof(uint64_t) * kCostMagicB * d->n_profiles);
  L.in_end = o;
  // zeroed at create, contiguous: one memset
  L.zero_beg = o;
  L.off_sn = take(sizeof(uint32_t) * ns);
  L.off_dn = take(sizeof(uint32_t) * 2 * nd);
  L.off_stats = take(sizeof(bellman_scenario_stats) * d->n_scenarios);
  L.off_hist = take(sizeof(uint64_t) * kSegWords * d->n_segments);
  L.off_cnt = take(sizeof(unsigned int) * 32);
  // K2L per-thread histograms: all-zero between scenarios (each epilogue
  // re-zeroes what its scenario touched), only when some scenario runs in K2L
  L.off_lhist = take(lane_possible(d) ? sizeof(uint32_t) * kLaneHistWords * kLaneMaxThreads : 0);
  L.zero_end = o;
  // written by the kernels before they are read
  L.off_series = take(sizeof(uint32_t) * h.series_words);
  L.off_calib = take(sizeof(uint32_t) * 4 * ns);
  L.off_drows = take(sizeof(bellman_second_row) * h.dbg_rows);
  L.off_dctrl = take(sizeof(bellman_ctrl_row) * h.dbg_rows);
  L.off_sord = take(sizeof(uint32_t) * d->n_scenarios);  // a strided shard's order, written by bellman_sim_run
  // NEXT-4 preemption scratch (per CTA: slot side state + the preempted stack),
  // only when some profile preempts
  bool pre = false;
  for (uint32_t i = 0; i < d->n_profiles; ++i)
    pre = pre || (d->profiles[i].kv_policy == BELLMAN_KV_PREEMPT && d->profiles[i].kv_cap_words > 0);
  L.off_pre = take(pre ? sizeof(PreScratch) * kMaxPreCtas : 0);
  // K2L per-thread arrival FIFOs (written before they are read)
  L.off_lfifo = take(lane_possible(d) ? sizeof(uint2) * 96u * kLaneMaxThreads : 0);
  L.total = o;
  return L;
}

// T[i] = round(2^32 * log2(1 + i/4096)) (reading R33), product-side evaluation
// (computed once per process: it depends on nothing).
static void log2_table_build(std::vector<uint2> &out) {
  out.resize(BELLMAN_TABLE_N);
  uint64_t prev = 0;
  for (int i = 0; i <= BELLMAN_TABLE_N; ++i) {
    const long double v = std::log2((long double)1.0 + (long double)i / 4096.0L) * 4294967296.0L;
    const uint64_t t = (uint64_t)std::floor(v + 0.5L);
    if (i > 0) out[i - 1] = make_uint2((uint32_t)prev, (uint32_t)(t - prev));
    prev = t;
  }
}

// K2L's leap reciprocals (bellman_internal.cuh): M = ceil(2^63 / c(B)) for
// B = 0 .. 64 of every profile whose kv-free cost law stays in [1, 2^31); 0
// elsewhere (such profiles never run in K2L's kv-free kernel).
static void cost_magic_build(const bellman_profile *pr, uint32_t n, std::vector<uint64_t> &out) {
  out.assign((size_t)kCostMagicB * n, 0);
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t b = 0; b < kCostMagicB; ++b) {
      const uint64_t c = (uint64_t)pr[i].t0_us + (uint64_t)pr[i].slope_us * (b > pr[i].knee ? b - pr[i].knee : 0u);
      if (c >= 1 && c < (1ull << 31)) out[(size_t)kCostMagicB * i + b] = ((1ull << 63) + c - 1) / c;
    }
}

extern "C" {

size_t bellman_sim_workspace_bytes(const bellman_sim_desc *desc) {
  if (validate(desc) != BELLMAN_OK) return 0;
  static thread_local HostPrep h;  // buffers reused across calls (C5: ~20 MB of per-scenario arrays)
  prepare(desc, h);
  return layout(desc, h).total;
}

bellman_status bellman_sim_create(const bellman_sim_desc *desc, void *workspace, size_t workspace_bytes, int device,
                                  void *stream, bellman_sim **out) {
  if (!out) return fail(nullptr, BELLMAN_EINVAL, "out is NULL");
  *out = nullptr;
  bellman_status st = validate(desc);
  if (st != BELLMAN_OK) return st;
  static thread_local HostPrep h;  // buffers reused across calls (C5: ~20 MB of per-scenario arrays)
  prepare(desc, h);
  const Layout L = layout(desc, h);
  if (!workspace || ((uintptr_t)workspace & 255u))
    return fail(nullptr, BELLMAN_EWORKSPACE, "workspace NULL or not 256-byte aligned");
  if (workspace_bytes < L.total)
    return fail(nullptr, BELLMAN_EWORKSPACE, "workspace too small: %zu < %zu", workspace_bytes, L.total);
  cudaError_t ce = cudaSetDevice(device);
  if (ce != cudaSuccess) return fail(nullptr, BELLMAN_ECUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(ce));
  cudaPointerAttributes pa{};
  ce = cudaPointerGetAttributes(&pa, workspace);
  if (ce != cudaSuccess || pa.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return fail(nullptr, BELLMAN_EWORKSPACE, "workspace is not device memory");
  }
  bellman_sim *sim = new (std::nothrow) bellman_sim();
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "out of host memory");
  sim->device = device;
  sim->n_scenarios = desc->n_scenarios;
  sim->n_segments = desc->n_segments;
  sim->n_slots = (uint32_t)h.slot_off.size();
  sim->grid = bellman_tick_grid(device);
  if (sim->grid <= 0) {
    delete sim;
    return fail(nullptr, BELLMAN_ECUDA, "occupancy query failed");
  }
  if (sim->grid > (int)kMaxPreCtas) sim->grid = (int)kMaxPreCtas;  // one preemption scratch per CTA
  sim->lane_grid = bellman_lane_grid(device);
  if (sim->lane_grid <= 0) {
    delete sim;
    return fail(nullptr, BELLMAN_ECUDA, "SM count query failed");
  }
  // one pass over the scenario table (host threads): calibrated scenarios and
  // which kernels have work
  sim->calibrated.assign(desc->n_scenarios, 0);
  sim->calib_src.assign(desc->n_scenarios, BELLMAN_NONE);
  {
    struct Flags {
      bool cal = false, kind[2][2][5] = {};
    };
    std::vector<Flags> fl(16);
    parallel_chunks(desc->n_scenarios, [&](uint64_t lo, uint64_t hi, unsigned t) {
      Flags &f = fl[t];
      for (uint64_t s = lo; s < hi; ++s) {
        const bellman_scenario &sc = desc->scenarios[s];
        const bellman_ctrl &c = desc->ctrls[sc.ctrl];
        if (c.calibrated) {
          sim->calibrated[s] = 1;
          f.cal = true;
          sim->calib_src[s] = sc.calib_src;
        }
        const uint32_t k1 = kind_of(desc, sc, 1u);
        const int dbg = (sc.record & BELLMAN_RECORD_SECONDS) ? 1 : 0;
        f.kind[1][dbg][k1] = true;
        f.kind[0][dbg][k1 >= 3u ? 0u : k1] = true;  // without K2L, its scenarios run in the TBT warp loop
      }
    });
    for (const Flags &f : fl) {
      sim->has_calibrated = sim->has_calibrated || f.cal;
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
          for (int k = 0; k < 5; ++k) sim->has_kind[a][b][k] = sim->has_kind[a][b][k] || f.kind[a][b][k];
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t *ws = (uint8_t *)workspace;
  Params &P = sim->params;
  P.sc = (const bellman_scenario *)(ws + L.off_sc);
  P.traces = (const DevTrace *)(ws + L.off_tr);
  P.segs = (const DevSeg *)(ws + L.off_seg);
  P.profs = (const bellman_profile *)(ws + L.off_prof);
  P.ctrls = (const bellman_ctrl *)(ws + L.off_ctrl);
  int32_t *tab = (int32_t *)(ws + L.off_tab);
  P.tabL = tab;
  P.tabI = tab + BELLMAN_TABLE_N;
  P.tabF = tab + 2 * BELLMAN_TABLE_N;
  P.tabN = tab + 3 * BELLMAN_TABLE_N;
  P.tabC = tab + 4 * BELLMAN_TABLE_N;
  P.tabQ = tab + 5 * BELLMAN_TABLE_N;
  P.q_inactive = desc->models.quality[0];
  P.q_active = desc->models.quality[1];
  P.q_floor = desc->models.quality[2];
  P.q_safe = desc->models.quality[3];
  P.q_end = desc->models.quality[4];
  P.class_cum0 = desc->models.class_cum[0];
  P.class_cum1 = desc->models.class_cum[1];
  P.class_cum2 = desc->models.class_cum[2];
  P.log2tab = (const uint2 *)(ws + L.off_log2);
  P.poly0 = desc->models.poly_q16[0];
  P.poly1 = desc->models.poly_q16[1];
  P.poly2 = desc->models.poly_q16[2];
  {  // N <= P < 2^17 and Fcomp <= 2^18: |poly| < 2^43 keeps poly * Fcomp inside int64
    const int64_t *c = desc->models.poly_q16;
    const unsigned __int128 b = (unsigned __int128)(c[0] < 0 ? -c[0] : c[0]) +
                                ((unsigned __int128)(c[1] < 0 ? -c[1] : c[1]) << 17) +
                                ((unsigned __int128)(c[2] < 0 ? -c[2] : c[2]) << 34);
    P.poly_fast = b < ((unsigned __int128)1 << 43) ? 1u : 0u;
  }
  P.series_slot = (const uint32_t *)(ws + L.off_slot);
  P.series_off = (const uint64_t *)(ws + L.off_soff);
  P.series_cap = (const uint32_t *)(ws + L.off_scap);
  P.series_n = (uint32_t *)(ws + L.off_sn);
  P.series = (uint32_t *)(ws + L.off_series);
  P.calib = (uint32_t *)(ws + L.off_calib);
  P.stats = (bellman_scenario_stats *)(ws + L.off_stats);
  P.seg_hist = (unsigned long long *)(ws + L.off_hist);
  sim->counters = (unsigned int *)(ws + L.off_cnt);
  P.dbg_slot = (const uint32_t *)(ws + L.off_dslot);
  P.dbg_off = (const uint64_t *)(ws + L.off_doff);
  P.dbg_cap = (const uint32_t *)(ws + L.off_dcap);
  P.dbg_n = (uint32_t *)(ws + L.off_dn);
  P.dbg_rows = (bellman_second_row *)(ws + L.off_drows);
  P.dbg_ctrl = (bellman_ctrl_row *)(ws + L.off_dctrl);
  P.arrivals = (const bellman_arrival *)(ws + L.off_arr);
  P.order = nullptr;
  P.pre = (PreScratch *)(ws + L.off_pre);
  P.lane_on = 0;  // set per run
  P.lane_hist = (uint32_t *)(ws + L.off_lhist);
  P.lane_fifo = (uint2 *)(ws + L.off_lfifo);
  P.cost_magic = (const uint64_t *)(ws + L.off_cmag);
  sim->lane_ok = lane_possible(desc);
  sim->order = (const uint32_t *)(ws + L.off_ord);
  sim->shard_order = (uint32_t *)(ws + L.off_sord);
  sim->host_order = h.order;
  sim->dbg_slot = h.dbg_of;
  sim->has_dbg = !h.dbg_off.empty();

  sim->dbg_off = h.dbg_off;
  sim->dbg_cap = h.dbg_cap;

  static const std::vector<uint2> l2 = [] {
    std::vector<uint2> t;
    log2_table_build(t);
    return t;
  }();
  {
    // the scenario table (64 B per scenario, the one large input) is copied
    // straight from the caller's array (a DMA when it is pinned); every other
    // input region is assembled in one pageable staging buffer laid out like
    // the rest of the workspace's input prefix: two H2D copies and one memset
    static_assert(sizeof(bellman_scenario) == 64, "scenario record");
    const size_t base = L.off_tr;  // the staging buffer starts here (off_sc = 0 precedes it)
    static thread_local std::vector<uint8_t> stage;  // reused across creates (no fresh pages per call)
    stage.assign(L.in_end - base, 0);
    auto put = [&](size_t off, const void *src, size_t bytes) {
      if (bytes) std::memcpy(stage.data() + (off - base), src, bytes);
    };
    put(L.off_tr, h.traces.data(), sizeof(DevTrace) * h.traces.size());
    put(L.off_seg, h.segs.data(), sizeof(DevSeg) * h.segs.size());
    put(L.off_prof, desc->profiles, sizeof(bellman_profile) * desc->n_profiles);
    put(L.off_ctrl, desc->ctrls, sizeof(bellman_ctrl) * desc->n_ctrls);
    const int32_t *tabs[6] = {desc->models.L_words, desc->models.I_words, desc->models.fvar_q16,
                              desc->models.noise,   desc->models.fcomp_q16, desc->models.qnoise};
    for (int k = 0; k < 6; ++k)
      put(L.off_tab + sizeof(int32_t) * BELLMAN_TABLE_N * k, tabs[k], sizeof(int32_t) * BELLMAN_TABLE_N);
    put(L.off_log2, l2.data(), sizeof(uint2) * BELLMAN_TABLE_N);
    put(L.off_slot, h.slot_of.data(), sizeof(uint32_t) * desc->n_scenarios);
    put(L.off_soff, h.slot_off.data(), sizeof(uint64_t) * h.slot_off.size());
    put(L.off_scap, h.slot_cap.data(), sizeof(uint32_t) * h.slot_cap.size());
    put(L.off_dslot, h.dbg_of.data(), sizeof(uint32_t) * desc->n_scenarios);
    put(L.off_doff, h.dbg_off.data(), sizeof(uint64_t) * h.dbg_off.size());
    put(L.off_dcap, h.dbg_cap.data(), sizeof(uint32_t) * h.dbg_cap.size());
    put(L.off_arr, desc->arrivals, sizeof(bellman_arrival) * desc->n_arrivals);
    put(L.off_ord, h.order.data(), sizeof(uint32_t) * desc->n_scenarios);
    {
      std::vector<uint64_t> cm;
      cost_magic_build(desc->profiles, desc->n_profiles, cm);
      put(L.off_cmag, cm.data(), sizeof(uint64_t) * cm.size());
    }
    auto body = [&]() -> bellman_status {
      if (desc->n_scenarios)
        CUDA_TRY(nullptr, cudaMemcpyAsync(ws + L.off_sc, desc->scenarios, sizeof(bellman_scenario) * desc->n_scenarios,
                                          cudaMemcpyHostToDevice, s));
      CUDA_TRY(nullptr, cudaMemcpyAsync(ws + base, stage.data(), L.in_end - base, cudaMemcpyHostToDevice, s));
      CUDA_TRY(nullptr, cudaMemsetAsync(ws + L.zero_beg, 0, L.zero_end - L.zero_beg, s));
      CUDA_TRY(nullptr, cudaStreamSynchronize(s));  // the staging buffer is freed on return (and the
                                                    // caller's scenario array may be reused)
      return BELLMAN_OK;
    };
    const bellman_status rc = body();
    if (rc != BELLMAN_OK) {
      delete sim;
      return rc;
    }
  }
  *out = sim;
  return BELLMAN_OK;
}

bellman_status bellman_sim_run(bellman_sim *sim, uint64_t first, uint64_t count, uint64_t stride, void *stream) {
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "sim is NULL");
  if (count == 0) {
    sim->last_launches = 0;
    sim->last_engines = 0;
    return BELLMAN_OK;
  }
  if (stride == 0) return fail(sim, BELLMAN_ESTATE, "stride must be >= 1");
  if (first >= sim->n_scenarios || (count - 1) > (sim->n_scenarios - 1 - first) / stride)
    return fail(sim, BELLMAN_ESTATE, "scenario range out of bounds");
  if (count > 0xFFFFFFFFull) return fail(sim, BELLMAN_ESTATE, "count too large");
  bool any_cal = false;
  if (sim->has_calibrated) {
    for (uint64_t k = 0; k < count; ++k) {
      const uint64_t id = first + k * stride;
      if (!sim->calibrated[id]) continue;
      any_cal = true;
      const uint64_t src = sim->calib_src[id];
      if (src < first || (src - first) % stride || (src - first) / stride >= count)
        return fail(sim, BELLMAN_ESTATE, "scenario %llu: calibration source %llu not in the run set",
                    (unsigned long long)id, (unsigned long long)src);
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(sim, cudaSetDevice(sim->device));
  Params P = sim->params;
  P.first = first;
  P.count = count;
  P.stride = stride;
  // every run takes its scenarios heavy-first: a whole-set run from the create-time
  // order, a shard (first + k stride, k < count) from that order filtered to the
  // shard (stable, so equal costs keep id order), uploaded once per distinct shard
  if (first == 0 && stride == 1 && count == sim->n_scenarios) {
    P.order = sim->order;
  } else {
    std::lock_guard<std::mutex> lk(g_shard_mu);
    auto it = g_shard_owner.find(sim->shard_order);
    const bool mine = it != g_shard_owner.end() && it->second == sim->shard_gen;
    if (!mine || sim->shard_key[0] != first || sim->shard_key[1] != stride || sim->shard_key[2] != count) {
      sim->host_shard.clear();
      sim->host_shard.reserve(count);
      for (uint32_t id : sim->host_order)
        if (id >= first && (id - first) % stride == 0 && (id - first) / stride < count) sim->host_shard.push_back(id);
      if (sim->host_shard.size() != count) return fail(sim, BELLMAN_ESTATE, "shard order: internal size mismatch");
      // the host vector outlives the copy (a member), and the copy is stream-ordered before the launch
      CUDA_TRY(sim, cudaMemcpyAsync(sim->shard_order, sim->host_shard.data(), sizeof(uint32_t) * count,
                                    cudaMemcpyHostToDevice, s));
      sim->shard_key[0] = first;
      sim->shard_key[1] = stride;
      sim->shard_key[2] = count;
      sim->shard_gen = ++g_shard_gen;
      g_shard_owner[sim->shard_order] = sim->shard_gen;
    }
    P.order = sim->shard_order;
  }
#ifdef BELLMAN_AB_NOORDER
  P.order = nullptr;
#endif
  CUDA_TRY(sim, cudaMemsetAsync(sim->counters, 0, 32 * sizeof(unsigned int), s));
  const uint64_t want = (count + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int grid = (int)(want < (uint64_t)sim->grid ? want : (uint64_t)sim->grid);
  sim->last_launches = 0;
  sim->last_engines = 0;
  // pass 1: non-calibrated scenarios.  One launch per kernel with work
  // (scenario_kind_of): K2L (kv = 0 / kv > 0), the TBT-specialised, generic and
  // multi-replica warp engines, debug-recorded or not; if no kernel has work
  // (an empty set) the TBT-specialised warp kernel runs once
  P.lane_on = (sim->lane_ok && (lane_mode() == 2 || count >= kLaneMinScenarios)) ? 1u : 0u;
  auto pass = [&](uint32_t pass_no, unsigned int *ctr) -> bellman_status {
    P.pass = pass_no;
    uint32_t n = 0;
    for (int dbg = 0; dbg < 2; ++dbg)
      for (int kind = 0; kind < 5; ++kind) {
        if (!sim->has_kind[P.lane_on][dbg][kind]) continue;
        P.counter = ctr + 5 * dbg + kind;
        if (kind >= 3) CUDA_TRY(sim, bellman_launch_lane(P, sim->lane_grid, kind, s));
        else CUDA_TRY(sim, bellman_launch_tick(P, grid, dbg != 0, kind, s));
        sim->last_engines |= 1u << kind;
        n++;
      }
    if (n == 0) {
      P.counter = ctr;
      CUDA_TRY(sim, bellman_launch_tick(P, grid, false, 0, s));
      sim->last_engines |= 1u;
      n++;
    }
    sim->last_launches += n;
    return BELLMAN_OK;
  };
  bellman_status rc = pass(1, sim->counters);
  if (rc != BELLMAN_OK) return rc;
  if (any_cal) {  // a10: calibration, then pass 2 over the calibrated scenarios
    CUDA_TRY(sim, bellman_launch_calibrate(P, sim->n_slots, s));
    sim->last_launches++;
    rc = pass(2, sim->counters + 16);
    if (rc != BELLMAN_OK) return rc;
  }
  return BELLMAN_OK;
}

bellman_status bellman_sim_stats(bellman_sim *sim, bellman_scenario_stats *dst, uint64_t first, uint64_t count,
                                 int dst_is_device, void *stream) {
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "sim is NULL");
  if (!dst) return fail(sim, BELLMAN_EINVAL, "dst is NULL");
  if (first > sim->n_scenarios || count > sim->n_scenarios - first)
    return fail(sim, BELLMAN_ESTATE, "stats range out of bounds");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(sim, cudaSetDevice(sim->device));
  CUDA_TRY(sim, cudaMemcpyAsync(dst, sim->params.stats + first, sizeof(bellman_scenario_stats) * count,
                                dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (!dst_is_device) CUDA_TRY(sim, cudaStreamSynchronize(s));
  return BELLMAN_OK;
}

bellman_status bellman_sim_stats_strided(bellman_sim *sim, bellman_scenario_stats *dst, uint64_t first,
                                         uint64_t count, uint64_t stride, int dst_is_device, void *stream) {
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "sim is NULL");
  if (!dst) return fail(sim, BELLMAN_EINVAL, "dst is NULL");
  if (stride == 0) return fail(sim, BELLMAN_ESTATE, "stride must be >= 1");
  if (count == 0) return BELLMAN_OK;
  if (first >= sim->n_scenarios || (count - 1) > (sim->n_scenarios - 1 - first) / stride)
    return fail(sim, BELLMAN_ESTATE, "stats range out of bounds");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(sim, cudaSetDevice(sim->device));
  const size_t rec = sizeof(bellman_scenario_stats);
  CUDA_TRY(sim, cudaMemcpy2DAsync(dst, rec, sim->params.stats + first, rec * stride, rec, count,
                                  dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (!dst_is_device) CUDA_TRY(sim, cudaStreamSynchronize(s));
  return BELLMAN_OK;
}

bellman_status bellman_sim_segment_hist(bellman_sim *sim, uint64_t *dst, int dst_is_device, void *stream) {
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "sim is NULL");
  if (!dst) return fail(sim, BELLMAN_EINVAL, "dst is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(sim, cudaSetDevice(sim->device));
  CUDA_TRY(sim, cudaMemcpyAsync(dst, sim->params.seg_hist, sizeof(uint64_t) * kSegWords * sim->n_segments,
                                dst_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  if (!dst_is_device) CUDA_TRY(sim, cudaStreamSynchronize(s));
  return BELLMAN_OK;
}

bellman_status bellman_sim_reset(bellman_sim *sim, void *stream) {
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "sim is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(sim, cudaSetDevice(sim->device));
  CUDA_TRY(sim, cudaMemsetAsync(sim->params.stats, 0, sizeof(bellman_scenario_stats) * sim->n_scenarios, s));
  CUDA_TRY(sim, cudaMemsetAsync(sim->params.seg_hist, 0, sizeof(uint64_t) * kSegWords * sim->n_segments, s));
  if (sim->n_slots) CUDA_TRY(sim, cudaMemsetAsync(sim->params.series_n, 0, sizeof(uint32_t) * sim->n_slots, s));
  if (sim->dbg_off.size())
    CUDA_TRY(sim, cudaMemsetAsync(sim->params.dbg_n, 0, sizeof(uint32_t) * 2 * sim->dbg_off.size(), s));
  return BELLMAN_OK;
}

bellman_status bellman_sim_series(bellman_sim *sim, uint64_t id, bellman_second_row *rows, uint64_t cap_rows,
                                  uint64_t *n_rows, bellman_ctrl_row *ctrl, uint64_t cap_ctrl, uint64_t *n_ctrl,
                                  void *stream) {
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "sim is NULL");
  if (id >= sim->n_scenarios || sim->dbg_slot[id] == BELLMAN_NONE)
    return fail(sim, BELLMAN_ESTATE, "scenario %llu is not debug-recorded", (unsigned long long)id);
  const uint32_t slot = sim->dbg_slot[id];
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(sim, cudaSetDevice(sim->device));
  uint32_t n[2] = {0, 0};
  CUDA_TRY(sim, cudaMemcpyAsync(n, sim->params.dbg_n + 2 * slot, sizeof(n), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(sim, cudaStreamSynchronize(s));
  if (n_rows) *n_rows = n[0];
  if (n_ctrl) *n_ctrl = n[1];
  const uint64_t nr = n[0] < cap_rows ? n[0] : cap_rows;
  const uint64_t nc = (n[1] < sim->dbg_cap[slot] ? n[1] : sim->dbg_cap[slot]);
  const uint64_t nc2 = nc < cap_ctrl ? nc : cap_ctrl;
  if (rows && nr)
    CUDA_TRY(sim, cudaMemcpyAsync(rows, sim->params.dbg_rows + sim->dbg_off[slot], sizeof(bellman_second_row) * nr,
                                  cudaMemcpyDeviceToHost, s));
  if (ctrl && nc2)
    CUDA_TRY(sim, cudaMemcpyAsync(ctrl, sim->params.dbg_ctrl + sim->dbg_off[slot], sizeof(bellman_ctrl_row) * nc2,
                                  cudaMemcpyDeviceToHost, s));
  CUDA_TRY(sim, cudaStreamSynchronize(s));
  return BELLMAN_OK;
}

// ---- fused summary exchange over peer memory (include/bellman_sim.h, §8(e))
static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");

bellman_status bellman_ipc_export(const void *dev_ptr, void *handle, uint64_t *offset) {
  if (!dev_ptr || !handle || !offset) return fail(nullptr, BELLMAN_EINVAL, "ipc_export: NULL argument");
  // base of the allocation containing dev_ptr (a caching allocator hands out
  // interior pointers): cuMemGetAddressRange, resolved through the runtime so
  // that the library does not link libcuda
  typedef CUresult (*range_fn)(CUdeviceptr *, size_t *, CUdeviceptr);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return fail(nullptr, BELLMAN_ECUDA, "ipc_export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (((range_fn)fn)(&base, &size, (CUdeviceptr)(uintptr_t)dev_ptr) != CUDA_SUCCESS)
    return fail(nullptr, BELLMAN_ECUDA, "ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
  if (e != cudaSuccess) return fail(nullptr, BELLMAN_ECUDA, "ipc_export: %s", cudaGetErrorString(e));
  std::memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return BELLMAN_OK;
}

bellman_status bellman_ipc_open(const void *handle, uint64_t offset, int device, void **base, void **dev_ptr) {
  if (!handle || !base || !dev_ptr) return fail(nullptr, BELLMAN_EINVAL, "ipc_open: NULL argument");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(nullptr, BELLMAN_ECUDA, "ipc_open: %s", cudaGetErrorString(e));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void *b = nullptr;
  e = cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(nullptr, BELLMAN_ECUDA, "ipc_open: %s", cudaGetErrorString(e));
  *base = b;
  *dev_ptr = (uint8_t *)b + offset;
  return BELLMAN_OK;
}

bellman_status bellman_ipc_close(void *base) {
  if (!base) return fail(nullptr, BELLMAN_EINVAL, "ipc_close: NULL base");
  const cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return fail(nullptr, BELLMAN_ECUDA, "ipc_close: %s", cudaGetErrorString(e));
  return BELLMAN_OK;
}

bellman_status bellman_sim_set_peers(bellman_sim *sim, void *const *peer_stats, uint32_t n_peers) {
  if (!sim) return fail(nullptr, BELLMAN_ESTATE, "sim is NULL");
  if (n_peers > BELLMAN_MAX_PEERS) return fail(sim, BELLMAN_EINVAL, "n_peers > %d", BELLMAN_MAX_PEERS);
  if (n_peers && !peer_stats) return fail(sim, BELLMAN_EINVAL, "peer_stats is NULL");
  for (uint32_t g = 0; g < n_peers; ++g)
    if (!peer_stats[g] || ((uintptr_t)peer_stats[g] & 15u))
      return fail(sim, BELLMAN_EINVAL, "peer %u: NULL or not 16-byte aligned", g);
  for (uint32_t g = 0; g < BELLMAN_MAX_PEERS; ++g)
    sim->params.peer[g] = g < n_peers ? (bellman_scenario_stats *)peer_stats[g] : nullptr;
  sim->params.n_peer = n_peers;
  return BELLMAN_OK;
}

uint32_t bellman_sim_last_launches(const bellman_sim *sim) { return sim ? sim->last_launches : 0; }
uint32_t bellman_sim_last_engines(const bellman_sim *sim) { return sim ? sim->last_engines : 0; }

void bellman_sim_destroy(bellman_sim *sim) { delete sim; }

const char *bellman_status_string(bellman_status s) {
  switch (s) {
    case BELLMAN_OK: return "ok";
    case BELLMAN_EINVAL: return "invalid descriptor";
    case BELLMAN_EIO: return "io error";
    case BELLMAN_EDEGENERATE: return "degenerate data";
    case BELLMAN_ECUDA: return "cuda error";
    case BELLMAN_EWORKSPACE: return "workspace error";
    case BELLMAN_ESTATE: return "invalid state or range";
  }
  return "unknown status";
}

const char *bellman_sim_last_error(const bellman_sim *sim) { return sim ? sim->err : g_err; }

}  // extern "C"

#ifdef BELLMAN_LANECHECK
// ---------------------------------------------------------------------------
// Development build only (-DBELLMAN_LANECHECK, never the product library): run
// K2L's per-scenario code on the CPU over every scenario it would take, with
// the calibration between the passes done here, so that the lane engine can be
// compared with the oracle (scripts/lanecheck.py) without a GPU.
namespace bellman {
void lane_host_run(const Params &p, uint64_t sid, uint32_t *smem_warp, uint32_t *hist, uint2 *fifo);
}
extern "C" int bellman_lanecheck(const bellman_sim_desc *d, bellman_scenario_stats *out, unsigned long long *seg,
                                 uint8_t *ran) {
  if (validate(d) != BELLMAN_OK) return -1;
  static thread_local HostPrep h;  // buffers reused across calls (C5: ~20 MB of per-scenario arrays)
  prepare(d, h);
  static std::vector<uint2> l2;
  if (l2.empty()) log2_table_build(l2);
  Params P{};
  P.sc = d->scenarios;
  P.traces = h.traces.data();
  P.segs = h.segs.data();
  P.profs = d->profiles;
  P.ctrls = d->ctrls;
  P.tabL = d->models.L_words;
  P.tabI = d->models.I_words;
  P.tabF = d->models.fvar_q16;
  P.tabN = d->models.noise;
  P.tabC = d->models.fcomp_q16;
  P.tabQ = d->models.qnoise;
  P.log2tab = l2.data();
  static thread_local std::vector<uint64_t> cm;
  cost_magic_build(d->profiles, d->n_profiles, cm);
  P.cost_magic = cm.data();
  P.poly0 = d->models.poly_q16[0];
  P.poly1 = d->models.poly_q16[1];
  P.poly2 = d->models.poly_q16[2];
  {
    const int64_t *c = d->models.poly_q16;
    const unsigned __int128 b = (unsigned __int128)(c[0] < 0 ? -c[0] : c[0]) +
                                ((unsigned __int128)(c[1] < 0 ? -c[1] : c[1]) << 17) +
                                ((unsigned __int128)(c[2] < 0 ? -c[2] : c[2]) << 34);
    P.poly_fast = b < ((unsigned __int128)1 << 43) ? 1u : 0u;
  }
  P.q_inactive = d->models.quality[0];
  P.q_active = d->models.quality[1];
  P.q_floor = d->models.quality[2];
  P.q_safe = d->models.quality[3];
  P.q_end = d->models.quality[4];
  P.class_cum0 = d->models.class_cum[0];
  P.class_cum1 = d->models.class_cum[1];
  P.class_cum2 = d->models.class_cum[2];
  std::vector<uint32_t> series(h.series_words + 1), series_n(h.slot_off.size() + 1), calib(4 * h.slot_off.size() + 4);
  P.series_slot = h.slot_of.data();
  P.series_off = h.slot_off.data();
  P.series_cap = h.slot_cap.data();
  P.series_n = series_n.data();
  P.series = series.data();
  P.calib = calib.data();
  P.stats = out;
  P.seg_hist = seg;
  P.lane_on = 1;
  std::vector<uint32_t> smem(kLaneWarpWords<false>), hist(kLaneHistWords, 0);
  std::vector<uint2> fifo(96);
  for (uint32_t pass = 1; pass <= 2; ++pass) {
    P.pass = pass;
    for (uint64_t s = 0; s < d->n_scenarios; ++s) {
      const bellman_scenario &sc = d->scenarios[s];
      if ((d->ctrls[sc.ctrl].calibrated != 0) != (pass == 2) || kind_of(d, sc, 1u) < 3u) continue;
      lane_host_run(P, s, smem.data(), hist.data(), fifo.data());
      ran[s] = 1;
    }
    if (pass == 1)
      for (size_t w = 0; w < h.slot_off.size(); ++w) {  // K5 on the host: nearest-rank p50 / p75
        const uint32_t n = std::min(series_n[w], h.slot_cap[w]);
        std::vector<uint32_t> x(series.begin() + h.slot_off[w], series.begin() + h.slot_off[w] + n);
        std::sort(x.begin(), x.end());
        uint32_t t1 = 0, t2 = 0, st = 1;
        if (n >= 4) {
          t1 = x[(50u * n + 99u) / 100u - 1u];
          t2 = x[(75u * n + 99u) / 100u - 1u];
          st = t1 == t2 ? 2u : 0u;
        }
        calib[4 * w] = t1;
        calib[4 * w + 1] = t2;
        calib[4 * w + 2] = st;
        calib[4 * w + 3] = n;
      }
  }
  for (uint32_t i = 0; i < kHistRing; ++i)
    if (hist[i]) return -2;  // every scenario's epilogue must leave its histograms zeroed
  return 0;
}
#endif

"""Seeded synthetic inputs for the beLLMan scenario simulator.

This module is the ONE place both the CPU oracle (``oracle/``) and the CUDA
path (``paper_2510_15330_b200/``) take their inputs from.  It holds none of the
method's arithmetic: no Philox, no -ln(U), no thinning, no cost law, no
controller, no statistics.  It only builds *descriptions* of experiments as
plain numpy column arrays:

* load traces as piecewise-linear knot tables of (µs, milli-RPS) integers
  ("Poisson process ... distinct phases when the request
  arrivals ramp up, stay put, and ramp down"; SPEC.md S:82 phase boundaries);
* workload distributions as 4096-entry quantile tables (SPEC.md S:84 and
  S:162-164 — the workload *provides* the distributions);
* serving cost profiles;
* controller configurations;
* the scenario list (seed x workload x controller) of each BASELINE.json config.

Every array is a pure function of the config name and its integer arguments.
Readings of silent/ambiguous passages are listed in DESIGN.md §3.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import ndtri

# ----------------------------------------------------------------------------
# enums shared *by value* with both implementations (documented in DESIGN.md)
# ----------------------------------------------------------------------------
LAW_OFF, LAW_CONST, LAW_MAP, LAW_STEP = 0, 1, 2, 3
LAW_MPC, LAW_BBR, LAW_PCC = 4, 5, 6  # NEXT-3, readings R41-R43
SIG_TBT, SIG_E2E, SIG_SLO, SIG_TTFT, SIG_INPUT, SIG_UTIL = 0, 1, 2, 3, 4, 5
MODE_CUTOFF, MODE_DRAIN = 0, 1

US = 1_000_000  # µs per second
TABLE_BITS = 12
TABLE_N = 1 << TABLE_BITS  # 4096 quantile entries, indexed by u32 >> 20

# ----------------------------------------------------------------------------
# cost profiles (readings R1, R2, R27)
# ----------------------------------------------------------------------------
PROFILES = {
    # SPEC.md S:248 literal defaults; used only to reproduce SPEC's worked examples.
    "spec-literal": dict(t0_us=50_000, knee=8, slope_us=6_000, kv_ns_per_word=0,
                         max_batch=64, prefill_ns_per_word=80_000,
                         e_in=0.05, e_out=0.5, p_idle=300.0),
    # Recalibrated so that saturation sits near the paper's 2.4 RPS.
    "P24": dict(t0_us=20_000, knee=1, slope_us=520, kv_ns_per_word=0,
                max_batch=64, prefill_ns_per_word=80_000,
                e_in=0.05, e_out=0.5, p_idle=300.0),
    # "Llama-3-8B-like decode cost model, 8xH100-equivalent capacity" (BJ C2; R27).
    "L8B": dict(t0_us=15_000, knee=1, slope_us=100, kv_ns_per_word=50,
                max_batch=64, prefill_ns_per_word=80_000,
                e_in=0.05, e_out=0.5, p_idle=300.0),
}


def _q(k):
    """Mid-point quantile level of table entry k: (k + 1/2) / 4096."""
    return (np.arange(TABLE_N, dtype=np.float64) + 0.5) / TABLE_N if k is None else (k + 0.5) / TABLE_N


def _round_half_up(x):
    return np.floor(np.asarray(x, dtype=np.float64) + 0.5).astype(np.int64)


def quantile_tables(L_mean=500.0, L_sd=80.0, L_lo=100, L_hi=1200,
                    in_median=9000.0, in_sigma=0.30, in_lo=2000, in_hi=20000,
                    var_sigma=0.0875, var_lo=0.75, var_hi=1.38,
                    pred_b=36.0, comp_rel_noise=0.05, sim_noise_pts=2.0):
    """Workload distributions as quantile tables.

    Entry k holds the distribution's quantile at level (k + 1/2)/4096; the
    simulator draws entry ``u >> 20`` of a uniform 32-bit word ``u``.

    * ``L``     unbounded output words ~ Normal(500, 80) clamped [100, 1200]
    * ``I``     input words ~ LogNormal(median 9000, sigma 0.30) clamped [2000, 20000]
                (sigma is reading R15)
    * ``fvar``  Q16 unbounded-variability factor, log ~ N(0, 0.0875) clipped to
                [ln 0.75, ln 1.38] (PAPER P:97 band, reading R14)
    * ``noise`` predictor error in words ~ Laplace(0, b=36) ("MAE 36";
                SPEC S:121)
    * ``fcomp`` Q16 compliance factor 1 + 0.05*z
    * ``qnoise`` similarity-score noise in centi-points ~ N(0, 2 points) (SPEC S:148,
                S:173 score_noise default 2.0; NEXT-2)
    """
    q = _q(None)
    z = ndtri(q)
    L = np.clip(_round_half_up(L_mean + L_sd * z), L_lo, L_hi)
    I = np.clip(_round_half_up(in_median * np.exp(in_sigma * z)), in_lo, in_hi)
    lf = np.clip(var_sigma * z, math.log(var_lo), math.log(var_hi))
    fvar = _round_half_up(65536.0 * np.exp(lf))
    lap = np.where(q < 0.5, pred_b * np.log(2.0 * q), -pred_b * np.log(2.0 * (1.0 - q)))
    noise = _round_half_up(lap)
    fcomp = np.maximum(_round_half_up(65536.0 * (1.0 + comp_rel_noise * z)), 0)
    qnoise = np.clip(_round_half_up(100.0 * sim_noise_pts * z), -2047, 2047)
    return {k: v.astype(np.int32) for k, v in
            dict(L=L, I=I, fvar=fvar, noise=noise, fcomp=fcomp, qnoise=qnoise).items()}


def constant_tables(L=500, I=9000, fvar=65536, noise=0, fcomp=65536, qnoise=0):
    """Degenerate (noise-free) tables, e.g. for closed-form queueing pins."""
    f = lambda v: np.full(TABLE_N, v, dtype=np.int32)
    return dict(L=f(L), I=f(I), fvar=f(fvar), noise=f(noise), fcomp=f(fcomp), qnoise=f(qnoise))


IDENTITY_POLY_Q16 = (0, 65536, 0)  # compliance realized = N (SPEC S:163 identity default)
# QualityModel (NEXT-2) in centi-points / basis points:
# inactive median 88 and active median 87, floor 65,
# safe window 20 %, linear decay to the floor at 40 %.
QUALITY = (8800, 8700, 6500, 2000, 4000)
# Request classes (NEXT-3): cumulative thresholds in 2^-20 units of the
# 20 low bits of the word that draws L; one class by default.
SINGLE_CLASS = (1 << 20,) * 4
# summarization 70 %, coding 20 %, short-form 10 % (an illustrative mix; the paper gives none)
MIXED_CLASSES = (int(0.7 * (1 << 20)), int(0.9 * (1 << 20)), 1 << 20, 1 << 20)

# ----------------------------------------------------------------------------
# traces (piecewise-linear lambda(t) knots; µs and milli-RPS integers)
# ----------------------------------------------------------------------------

def const_trace(rps: float, duration_s: float):
    lam = int(round(rps * 1000))
    return [(0, lam), (int(round(duration_s * US)), lam)]


# PAPER.md P:183 / SPEC.md S:82 (reading R16): the 22-minute two-peak trace.
PAPER_TRACE_KNOTS_S = [(0, 0.0), (60, 2.5), (150, 2.5), (210, 0.2), (840, 0.2),
                       (900, 1.5), (960, 1.5), (1020, 0.2), (1320, 0.2)]


def paper_trace(peak=2.5, peak_s=90, valley=0.2, second_peak=1.5):
    """Paper trace (R16) and its variants (R30: peak height/duration, valley)."""
    ramp_end = 60 + peak_s
    pts = [(0, 0.0), (60, peak), (ramp_end, peak), (ramp_end + 60, valley),
           (840, valley), (900, second_peak), (960, second_peak), (1020, valley), (1320, valley)]
    return [(int(s * US), int(round(r * 1000))) for s, r in pts]


def diurnal_trace(variant: int, days: float = 1.0):
    """24 h diurnal trace with congestion bursts (reading R29).

    lambda(t) = 1.2 + 0.8 sin(2 pi (t - 9h)/24h) RPS, knots every 15 min, plus
    8 bursts per day (60 s ramp up -> 90..300 s hold at 2.5..3.5 RPS -> 60 s
    ramp down), burst placement drawn from numpy's seeded Generator(variant).
    """
    rng = np.random.default_rng(1000 + variant)
    total_s = int(round(86400 * days))
    base = lambda t: 1.2 + 0.8 * math.sin(2 * math.pi * (t - 9 * 3600) / 86400.0)
    nb = int(round(8 * days))
    # non-overlapping bursts: one per equal slice of the day
    slice_s = total_s // nb
    bursts = []
    for b in range(nb):
        hold = int(rng.integers(90, 301))
        peak = float(rng.choice([2.5, 3.0, 3.5]))
        start = b * slice_s + int(rng.integers(900, slice_s - hold - 1200))
        bursts.append((start, hold, peak))
    knots = {}
    for t in range(0, total_s + 1, 900):
        knots[t] = base(t)
    for start, hold, peak in bursts:
        end = start + 60 + hold + 60
        for t in [t for t in knots if start <= t <= end]:
            del knots[t]
        knots[start] = base(start)
        knots[start + 60] = peak
        knots[start + 60 + hold] = peak
        knots[end] = base(end)
    return [(int(t) * US, int(round(r * 1000))) for t, r in sorted(knots.items())]


# ----------------------------------------------------------------------------
# controller configurations
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Ctrl:
    law: int = LAW_OFF
    signal: int = SIG_TBT
    window: int = 5           # P:193 "moving average over the last 5 seconds"
    r_min_bp: int = 500       # P:130 "between 5% and 20%"
    r_max_bp: int = 2000
    r_const_bp: int = 0
    t1: int = 0               # signal units: µs (TBT, E2E) or per-mille (SLO)
    t2: int = 0
    slo_us: int = 0
    calibrated: int = 0       # 1: t1/t2 = p50/p75 of the paired OFF run
    rungs_bp: tuple = ()      # word-limit ladder (reading R5), <= 8 ascending rungs
    bypass_mask: int = 0      # NEXT-3: bit c -> class c never rewritten ("coding tasks might use r=0")
    min_words_bypass: int = 0  # NEXT-3: predicted length below this is never rewritten
    horizon_s: int = 0        # NEXT-3 MPC: forecast horizon in seconds ("moving time horizon")
    w_lat: int = 0            # NEXT-3 MPC / PCC: cost per µs of signal above t1
    w_q: int = 0              # NEXT-3 MPC / PCC: cost per bp of r (quality and energy)
    w_osc: int = 0            # NEXT-3 MPC: cost per bp of |r change| ("avoid oscillations in r")
    step_bp: int = 0          # NEXT-3 BBR / PCC: r step (BBR without rungs) / experiment delta (PCC)


OFF = Ctrl()


def map_ctrl(t1_us, t2_us, r_min_bp=500, r_max_bp=2000, rungs=(), window=5, signal=SIG_TBT, slo_us=0):
    if rungs:
        r_min_bp, r_max_bp = rungs[0], rungs[-1]
    return Ctrl(LAW_MAP, signal, window, r_min_bp, r_max_bp, 0, int(t1_us), int(t2_us), slo_us, 0, tuple(rungs))


def step_ctrl(t1_us, t2_us, rungs, window=5, signal=SIG_TBT):
    return Ctrl(LAW_STEP, signal, window, rungs[0], rungs[-1], 0, int(t1_us), int(t2_us), 0, 0, tuple(rungs))


def mpc_ctrl(t1_us, horizon_s=3, w_lat=4, w_q=1, w_osc=2, r_min_bp=500, r_max_bp=2000, rungs=(), window=5,
             signal=SIG_TBT, slo_us=0):
    """NEXT-3 MPC (reading R41): forecast the signal horizon_s ahead and
    pick the r minimising w_lat (signal above t1) + w_q r + w_osc |dr|."""
    if rungs:
        r_min_bp, r_max_bp = rungs[0], rungs[-1]
    return Ctrl(LAW_MPC, signal, window, r_min_bp, r_max_bp, 0, int(t1_us), 0, slo_us, 0, tuple(rungs),
                horizon_s=horizon_s, w_lat=w_lat, w_q=w_q, w_osc=w_osc)


def bbr_ctrl(allow_us, step_bp=250, r_min_bp=500, r_max_bp=2000, rungs=(), window=5):
    """NEXT-3 BBR-style (reading R42): TBT signal; congested when the
    moving average exceeds the minimum TBT by allow_us; sheds / returns one step."""
    if rungs:
        r_min_bp, r_max_bp = rungs[0], rungs[-1]
    return Ctrl(LAW_BBR, SIG_TBT, window, r_min_bp, r_max_bp, 0, int(allow_us), 0, 0, 0, tuple(rungs),
                step_bp=0 if rungs else step_bp)


def pcc_ctrl(t1_us, delta_bp=250, w_lat=1, w_q=4, r_min_bp=500, r_max_bp=2000, window=5, signal=SIG_TBT,
             slo_us=0):
    """NEXT-3 PCC-style (reading R43): paired experiments r_base +- delta
    scored by the cost w_lat (signal above t1) + w_q r while MA >= t1."""
    return Ctrl(LAW_PCC, signal, window, r_min_bp, r_max_bp, 0, int(t1_us), 0, slo_us, 0, (),
                w_lat=w_lat, w_q=w_q, step_bp=delta_bp)


# ----------------------------------------------------------------------------
# scenario list -> column arrays
# ----------------------------------------------------------------------------
@dataclass
class Scenario:
    seed_index: int
    wid: int                  # Philox workload id (counter words 2,3); ON/OFF pairs share it
    trace: int
    profile: int
    ctrl: int
    segment: int
    mode: int
    horizon_us: int
    w0_us: int = 130 * US     # P:199 congestion window 130-500 s (reading R40)
    w1_us: int = 500 * US
    calib_src: int = 0xFFFFFFFF
    record: int = 0


@dataclass
class Workload:
    name: str
    traces: list = field(default_factory=list)      # list of (knots, arrival_cap)
    profiles: list = field(default_factory=list)    # list of dict
    ctrls: list = field(default_factory=list)       # list of Ctrl
    tables: dict = field(default_factory=dict)
    poly_q16: tuple = IDENTITY_POLY_Q16
    quality: tuple = QUALITY
    class_cum: tuple = SINGLE_CLASS
    scenarios: list = field(default_factory=list)
    n_segments: int = 1
    segment_names: list = field(default_factory=list)

    # ---- builders -------------------------------------------------------
    def add_trace(self, knots, cap=0):
        self.traces.append((list(knots), int(cap)))
        return len(self.traces) - 1

    def add_replay_trace(self, events, cap=0):
        """NEXT-4 replay: an explicit arrival list [(arrival_us, L, input, class), ...]
        sorted by arrival; per-request draws are keyed by the list index."""
        self.traces.append((("replay", [tuple(int(x) for x in e) for e in events]), int(cap)))
        return len(self.traces) - 1

    def add_profile(self, prof):
        p = PROFILES[prof] if isinstance(prof, str) else prof
        self.profiles.append(dict(p))
        return len(self.profiles) - 1

    def add_ctrl(self, c: Ctrl):
        if c in self.ctrls:
            return self.ctrls.index(c)
        self.ctrls.append(c)
        return len(self.ctrls) - 1

    # ---- columns --------------------------------------------------------
    def columns(self) -> dict:
        kt, kl, toff, tn, tcap, tkind = [], [], [], [], [], []
        ra, rL, rI, rC = [], [], [], []
        for knots, cap in self.traces:
            tcap.append(cap)
            if isinstance(knots, tuple) and knots and knots[0] == "replay":
                tkind.append(1)
                toff.append(len(ra))
                tn.append(len(knots[1]))
                for a, L, inp, cls in knots[1]:
                    ra.append(a)
                    rL.append(L)
                    rI.append(inp)
                    rC.append(cls)
                continue
            tkind.append(0)
            toff.append(len(kt))
            tn.append(len(knots))
            for t, lam in knots:
                kt.append(t)
                kl.append(lam)
        P = self.profiles
        C = self.ctrls
        rungs = np.zeros((max(len(C), 1), 8), dtype=np.uint32)
        for i, c in enumerate(C):
            for k, r in enumerate(c.rungs_bp):
                rungs[i, k] = r
        S = self.scenarios
        u32 = lambda xs: np.asarray(xs, dtype=np.uint32)
        i64 = lambda xs: np.asarray(xs, dtype=np.int64)
        f64 = lambda xs: np.asarray(xs, dtype=np.float64)
        cols = dict(
            knot_t=i64(kt), knot_lam=u32(kl),
            trace_knot_off=u32(toff), trace_n_knots=u32(tn), trace_cap=u32(tcap), trace_kind=u32(tkind),
            arr_a=i64(ra), arr_L=u32(rL), arr_input=u32(rI), arr_cls=u32(rC),
            prof_t0=u32([p["t0_us"] for p in P]), prof_knee=u32([p["knee"] for p in P]),
            prof_slope=u32([p["slope_us"] for p in P]), prof_kv=u32([p["kv_ns_per_word"] for p in P]),
            prof_maxb=u32([p["max_batch"] for p in P]), prof_prefill_ns=u32([p["prefill_ns_per_word"] for p in P]),
            prof_e_in=f64([p["e_in"] for p in P]), prof_e_out=f64([p["e_out"] for p in P]),
            prof_p_idle=f64([p["p_idle"] for p in P]),
            prof_kv_cap=u32([p.get("kv_cap_words", 0) for p in P]),
            prof_prefill_mode=u32([p.get("prefill_mode", 0) for p in P]),
            prof_kv_policy=u32([p.get("kv_policy", 0) for p in P]),
            prof_tpw=u32([p.get("tpw_q16", 0) for p in P]),
            prof_replicas=u32([p.get("replicas", 0) for p in P]), prof_route=u32([p.get("route", 0) for p in P]),
            ctrl_law=u32([c.law for c in C]), ctrl_signal=u32([c.signal for c in C]),
            ctrl_window=u32([c.window for c in C]), ctrl_rmin=u32([c.r_min_bp for c in C]),
            ctrl_rmax=u32([c.r_max_bp for c in C]), ctrl_rconst=u32([c.r_const_bp for c in C]),
            ctrl_t1=u32([c.t1 for c in C]), ctrl_t2=u32([c.t2 for c in C]),
            ctrl_slo_us=u32([c.slo_us for c in C]), ctrl_calibrated=u32([c.calibrated for c in C]),
            ctrl_nrungs=u32([len(c.rungs_bp) for c in C]), ctrl_rungs=rungs[:len(C)],
            ctrl_bypass_mask=u32([c.bypass_mask for c in C]), ctrl_min_words=u32([c.min_words_bypass for c in C]),
            ctrl_horizon=u32([c.horizon_s for c in C]), ctrl_wlat=u32([c.w_lat for c in C]),
            ctrl_wq=u32([c.w_q for c in C]), ctrl_wosc=u32([c.w_osc for c in C]), ctrl_step=u32([c.step_bp for c in C]),
            tab_L=self.tables["L"], tab_I=self.tables["I"], tab_fvar=self.tables["fvar"],
            tab_noise=self.tables["noise"], tab_fcomp=self.tables["fcomp"],
            poly_q16=i64(self.poly_q16),
            tab_qnoise=self.tables.get("qnoise", np.zeros(TABLE_N, dtype=np.int32)).astype(np.int32),
            quality=u32(self.quality), class_cum=u32(self.class_cum),
            sc_seed=u32([s.seed_index for s in S]), sc_wid=np.asarray([s.wid for s in S], dtype=np.uint64),
            sc_trace=u32([s.trace for s in S]), sc_profile=u32([s.profile for s in S]),
            sc_ctrl=u32([s.ctrl for s in S]), sc_segment=u32([s.segment for s in S]),
            sc_mode=u32([s.mode for s in S]), sc_horizon=i64([s.horizon_us for s in S]),
            sc_w0=i64([s.w0_us for s in S]), sc_w1=i64([s.w1_us for s in S]),
            sc_calib_src=u32([s.calib_src for s in S]), sc_record=u32([s.record for s in S]),
            n_segments=int(self.n_segments),
        )
        return cols

    @property
    def n_scenarios(self):
        return len(self.scenarios)


# ----------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------
C2_RATES_RPS = [0.5 * k for k in range(1, 17)]  # 0.5 .. 8.0 (BJ C2)
# Fixed C2 thresholds: nearest-rank p50/p75 of the per-second TBT samples pooled
# over the 64 OFF scenarios at 2.5 RPS.  Written by
# scripts/freeze_c2_thresholds.py, which calls only oracle/.
C2_T1_US = 50_810
C2_T2_US = 51_816

C3_T1_MS = (22, 24, 26, 28, 30, 34, 38, 42)
C3_DT_MS = (4, 8, 12, 16)
C3_LADDERS = (
    ("map", 500, 2000, ()), ("map", 500, 1500, ()), ("map", 200, 1000, ()),
    ("map", 500, 2500, ()), ("map", 1000, 3000, ()),
    ("map", 0, 0, (500, 1000, 1500, 2000)), ("map", 0, 0, (500, 2000)),
    ("map", 0, 0, (200, 400, 600, 800, 1000, 1500, 2000)),
    ("step", 0, 0, (500, 1000, 1500, 2000)),
    ("step", 0, 0, (200, 400, 600, 800, 1000, 1200, 1400, 1600)),
)


def _ladder_ctrl(lad, t1_us, t2_us):
    kind, rmin, rmax, rungs = lad
    if kind == "step":
        return step_ctrl(t1_us, t2_us, rungs)
    return map_ctrl(t1_us, t2_us, rmin, rmax, rungs)


def config_c1(tables=None, seed_index=0):
    """C1: one 2.5 RPS Poisson stream, 100 requests, 600 s, controller off vs on
    (thresholds calibrated from the off run), profile P24 (reading R28)."""
    w = Workload("C1")
    w.tables = tables or quantile_tables()
    tr = w.add_trace(const_trace(2.5, 600), cap=100)
    pr = w.add_profile("P24")
    off = w.add_ctrl(OFF)
    on = w.add_ctrl(Ctrl(LAW_MAP, SIG_TBT, 5, 500, 2000, 0, 0, 0, 0, 1, ()))
    w.scenarios = [
        Scenario(seed_index, wid=tr, trace=tr, profile=pr, ctrl=off, segment=0,
                 mode=MODE_CUTOFF, horizon_us=600 * US, record=1),
        Scenario(seed_index, wid=tr, trace=tr, profile=pr, ctrl=on, segment=1,
                 mode=MODE_CUTOFF, horizon_us=600 * US, calib_src=0),
    ]
    w.n_segments = 2
    w.segment_names = ["off", "on"]
    return w


def config_c2(n_seeds=64, rates=C2_RATES_RPS, horizon_s=600, seed_base=0, tables=None,
              t1_us=C2_T1_US, t2_us=C2_T2_US, profile="L8B"):
    """C2: arrival-rate sweep x seeds x {off, on}, L8B cost model (BJ configs[1])."""
    w = Workload("C2")
    w.tables = tables or quantile_tables()
    pr = w.add_profile(profile)
    off = w.add_ctrl(OFF)
    on = w.add_ctrl(map_ctrl(t1_us, t2_us))
    for ri, rps in enumerate(rates):
        tr = w.add_trace(const_trace(rps, horizon_s))
        for ci, c in enumerate((off, on)):
            seg = 2 * ri + ci
            for s in range(n_seeds):
                w.scenarios.append(Scenario(seed_base + s, wid=tr, trace=tr, profile=pr, ctrl=c,
                                            segment=seg, mode=MODE_CUTOFF, horizon_us=horizon_s * US))
    w.n_segments = 2 * len(rates)
    w.segment_names = [f"{r:g}rps/{m}" for r in rates for m in ("off", "on")]
    return w


def config_c3(n_seeds=32, tables=None, seed_base=0):
    """C3: controller grid (thresholds x ladders) x seeds on the paper trace, P24, drain."""
    w = Workload("C3")
    w.tables = tables or quantile_tables()
    tr = w.add_trace(paper_trace())
    pr = w.add_profile("P24")
    cells = [OFF]
    for t1 in C3_T1_MS:
        for dt in C3_DT_MS:
            for lad in C3_LADDERS:
                cells.append(_ladder_ctrl(lad, t1 * 1000, (t1 + dt) * 1000))
    for ci, c in enumerate(cells):
        k = w.add_ctrl(c)
        for s in range(n_seeds):
            w.scenarios.append(Scenario(seed_base + s, wid=tr, trace=tr, profile=pr, ctrl=k, segment=ci,
                                        mode=MODE_DRAIN, horizon_us=(1320 + 600) * US))
    w.n_segments = len(cells)
    return w


def config_c4(n_seeds=64, n_traces=16, days=1.0, tables=None):
    """C4: 24 h diurnal traces x 4 controllers x seeds, P24, drain (cap +1 h)."""
    w = Workload("C4")
    w.tables = tables or quantile_tables()
    pr = w.add_profile("P24")
    cells = [OFF, map_ctrl(26_000, 38_000), map_ctrl(26_000, 38_000, rungs=(500, 1000, 1500, 2000)),
             step_ctrl(26_000, 38_000, (500, 1000, 1500, 2000))]
    ks = [w.add_ctrl(c) for c in cells]
    cap = int(round(86400 * days)) + 3600
    for v in range(n_traces):
        tr = w.add_trace(diurnal_trace(v, days))
        for ci, k in enumerate(ks):
            for s in range(n_seeds):
                w.scenarios.append(Scenario(s, wid=tr, trace=tr, profile=pr, ctrl=k, segment=v * 4 + ci,
                                            mode=MODE_DRAIN, horizon_us=cap * US,
                                            w0_us=0, w1_us=cap * US))
    w.n_segments = n_traces * 4
    return w


def config_c5(n_seeds=4096, tables=None):
    """C5: 16 paper-trace variants x 16 controllers x 4096 seeds = 2^20 (reading R30)."""
    w = Workload("C5")
    w.tables = tables or quantile_tables()
    pr = w.add_profile("P24")
    grid = [OFF]
    for t1 in (26, 30, 34):
        for dt in (8, 12, 16):
            if len(grid) < 16:
                grid.append(map_ctrl(t1 * 1000, (t1 + dt) * 1000))
    for lad in C3_LADDERS[5:]:
        if len(grid) < 16:
            grid.append(_ladder_ctrl(lad, 26_000, 38_000))
    while len(grid) < 16:
        grid.append(map_ctrl(28_000, 40_000, 500, 1500))
    ks = [w.add_ctrl(c) for c in grid]
    vi = 0
    for peak in (2.0, 2.5, 3.0, 3.5):
        for dur in (90, 180):
            for valley in (0.2, 0.6):
                tr = w.add_trace(paper_trace(peak, dur, valley))
                for ci, k in enumerate(ks):
                    for s in range(n_seeds):
                        w.scenarios.append(Scenario(s, wid=tr, trace=tr, profile=pr, ctrl=k,
                                                    segment=vi * 16 + ci, mode=MODE_DRAIN,
                                                    horizon_us=(1320 + 600) * US))
                vi += 1
    w.n_segments = 256
    return w


def custom(traces, profiles, ctrls, scenarios, tables=None, poly_q16=IDENTITY_POLY_Q16, n_segments=None):
    """Free-form workload (used by unit tests and fixtures)."""
    w = Workload("custom")
    w.tables = tables if tables is not None else quantile_tables()
    w.poly_q16 = tuple(poly_q16)
    for t in traces:
        if isinstance(t, dict) and "replay" in t:
            w.add_replay_trace(t["replay"], t.get("cap", 0))
        elif isinstance(t, tuple) and len(t) == 2 and isinstance(t[1], int) and isinstance(t[0], list):
            w.add_trace(t[0], t[1])
        else:
            w.add_trace(t)
    for p in profiles:
        w.add_profile(p)
    w.ctrls = list(ctrls)
    w.scenarios = list(scenarios)
    w.n_segments = n_segments or (max((s.segment for s in scenarios), default=0) + 1)
    return w


def shard(n_scenarios: int, rank: int, world: int):
    """Scenario ids owned by ``rank``: interleaved (id % world == rank), SURVEY §8(e)."""
    return np.arange(rank, n_scenarios, world, dtype=np.int64)


CONFIGS = {"C1": config_c1, "C2": config_c2, "C3": config_c3, "C4": config_c4, "C5": config_c5}


def config_paper_pair(seed_index=0, tables=None, peak=2.5, peak_s=90, valley=0.2, profile="P24"):
    """The paper's headline experiment (P:183-199, S:495 A4): unbounded run on
    the 22-minute trace, then the bounded run with T1/T2 calibrated from it
    (P:185); both debug-recorded (per-second rows + controller log, NEXT-1)."""
    w = Workload("paper-pair")
    w.tables = tables or quantile_tables()
    tr = w.add_trace(paper_trace(peak, peak_s, valley))
    pr = w.add_profile(profile)
    off = w.add_ctrl(OFF)
    on = w.add_ctrl(Ctrl(LAW_MAP, SIG_TBT, 5, 500, 2000, 0, 0, 0, 0, 1, ()))
    H = (1320 + 600) * US
    w.scenarios = [
        Scenario(seed_index, wid=tr, trace=tr, profile=pr, ctrl=off, segment=0, mode=MODE_DRAIN, horizon_us=H,
                 record=3),
        Scenario(seed_index, wid=tr, trace=tr, profile=pr, ctrl=on, segment=1, mode=MODE_DRAIN, horizon_us=H,
                 calib_src=0, record=2),
    ]
    w.n_segments = 2
    w.segment_names = ["unbounded", "bounded"]
    return w


CONFIGS["paper-pair"] = config_paper_pair


# ----------------------------------------------------------------------------
# trace files (NEXT-4 replay)
# ----------------------------------------------------------------------------
TRACE_HEADER = "id,arrival_ms,input_words,unbounded_output_words,class"
CLASS_NAMES = ("summarization", "coding", "short-form", "other")


class TraceFormatError(ValueError):
    """Malformed or unsorted trace file; the message names the line."""


def write_trace(path, events, comments=()):
    """events: iterable of (id, arrival_ms, input_words, unbounded_output_words, class_index)."""
    with open(path, "w", encoding="utf-8") as f:
        for c in comments:
            f.write(f"# {c}\n")
        f.write(TRACE_HEADER + "\n")
        for e in events:
            i, a, inp, out, cls = e
            f.write(f"{int(i)},{int(a)},{int(inp)},{int(out)},{CLASS_NAMES[int(cls)]}\n")


def read_trace(path):
    """Parse a trace file; returns a list of (id, arrival_ms, input, output, class_index).
    Errors: malformed line -> TraceFormatError naming the line number;
    arrival_ms decreasing -> TraceFormatError citing the later line."""
    out = []
    seen_header = False
    last = None
    with open(path, encoding="utf-8") as f:
        for ln, raw in enumerate(f, 1):
            line = raw.rstrip("\n")
            if not seen_header:
                if line.startswith("#") or not line.strip():
                    continue
                if line.strip() != TRACE_HEADER:
                    raise TraceFormatError(f"line {ln}: expected header '{TRACE_HEADER}'")
                seen_header = True
                continue
            parts = line.split(",")
            if len(parts) != 5:
                raise TraceFormatError(f"line {ln}: expected 5 fields, got {len(parts)}")
            try:
                i, a, inp, o = (int(x) for x in parts[:4])
            except ValueError:
                raise TraceFormatError(f"line {ln}: non-integer field") from None
            name = parts[4].strip()
            if name not in CLASS_NAMES:
                raise TraceFormatError(f"line {ln}: unknown class '{name}'")
            if a < 0 or inp < 1 or o < 1 or inp > 65535 or o > 65535:
                raise TraceFormatError(f"line {ln}: field out of range")
            if last is not None and a < last:
                raise TraceFormatError(f"line {ln}: arrival_ms decreases (sortedness, S:77)")
            last = a
            out.append((i, a, inp, o, CLASS_NAMES.index(name)))
    if not seen_header:
        raise TraceFormatError("missing header")
    ids = [e[0] for e in out]
    if len(set(ids)) != len(ids):
        raise TraceFormatError("duplicate request ids (S:43)")
    return out

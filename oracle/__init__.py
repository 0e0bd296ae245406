"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding to ``oracle/liboracle.so`` (plain C, see ``oracle/oracle.h``).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  It shares no code with the
CUDA path; both consume the column arrays built by ``workloads``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = ["rng.c", "arrivals.c", "sim.c", "batch.c"]

NONE = 0xFFFFFFFF
HIST_LAT = 896
HIST_R = 512


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math, no FP contraction)."""
    srcs = [os.path.join(_HERE, s) for s in _SRCS] + [os.path.join(_HERE, "oracle.h")]
    if not force and os.path.exists(_SO) and all(os.path.getmtime(_SO) >= os.path.getmtime(s) for s in srcs):
        return _SO
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-ffp-contract=off", "-fPIC", "-shared", "-o", _SO]
    cmd += [os.path.join(_HERE, s) for s in _SRCS] + ["-lm", "-lpthread"]
    subprocess.run(cmd, check=True)
    return _SO


P = C.POINTER
u32p, u64p, i64p, i32p, f64p = P(C.c_uint32), P(C.c_uint64), P(C.c_int64), P(C.c_int32), P(C.c_double)


class Inputs(C.Structure):
    _fields_ = [
        ("knot_t", i64p), ("knot_lam", u32p),
        ("trace_knot_off", u32p), ("trace_n_knots", u32p), ("trace_cap", u32p),
        ("trace_kind", u32p), ("arr_a", i64p), ("arr_L", u32p), ("arr_input", u32p), ("arr_cls", u32p),
        ("prof_t0", u32p), ("prof_knee", u32p), ("prof_slope", u32p), ("prof_kv", u32p),
        ("prof_maxb", u32p), ("prof_prefill_ns", u32p), ("prof_kv_cap", u32p), ("prof_prefill_mode", u32p),
        ("prof_kv_policy", u32p), ("prof_tpw", u32p), ("prof_replicas", u32p), ("prof_route", u32p),
        ("prof_e_in", f64p), ("prof_e_out", f64p), ("prof_p_idle", f64p),
        ("ctrl_law", u32p), ("ctrl_signal", u32p), ("ctrl_window", u32p), ("ctrl_rmin", u32p),
        ("ctrl_rmax", u32p), ("ctrl_rconst", u32p),
        ("ctrl_t1", u32p), ("ctrl_t2", u32p), ("ctrl_slo_us", u32p), ("ctrl_calibrated", u32p),
        ("ctrl_nrungs", u32p), ("ctrl_rungs", u32p), ("ctrl_bypass_mask", u32p), ("ctrl_min_words", u32p),
        ("ctrl_horizon", u32p), ("ctrl_wlat", u32p), ("ctrl_wq", u32p), ("ctrl_wosc", u32p), ("ctrl_step", u32p),
        ("tab_L", i32p), ("tab_I", i32p), ("tab_fvar", i32p), ("tab_noise", i32p), ("tab_fcomp", i32p),
        ("poly_q16", i64p), ("tab_qnoise", i32p), ("quality", u32p), ("class_cum", u32p),
        ("sc_seed", u32p), ("sc_wid", u64p),
        ("sc_trace", u32p), ("sc_profile", u32p), ("sc_ctrl", u32p), ("sc_segment", u32p), ("sc_mode", u32p),
        ("sc_horizon", i64p), ("sc_w0", i64p), ("sc_w1", i64p),
        ("sc_calib_src", u32p), ("sc_record", u32p),
        ("n_scenarios", C.c_uint64),
    ]


class Request(C.Structure):
    _fields_ = [("a_us", C.c_uint64), ("j", C.c_uint32), ("L", C.c_uint32), ("input", C.c_uint32),
                ("U", C.c_uint32), ("P", C.c_uint32), ("fcomp_q16", C.c_int32), ("qnoise", C.c_int32),
                ("cls", C.c_uint32)]


class Profile(C.Structure):
    _fields_ = [("t0_us", C.c_uint32), ("knee", C.c_uint32), ("slope_us", C.c_uint32),
                ("kv_ns_per_word", C.c_uint32), ("max_batch", C.c_uint32), ("prefill_ns_per_word", C.c_uint32),
                ("e_in", C.c_double), ("e_out", C.c_double), ("p_idle", C.c_double), ("kv_cap_words", C.c_uint32),
                ("prefill_mode", C.c_uint32), ("kv_policy", C.c_uint32), ("tpw_q16", C.c_uint32),
                ("replicas", C.c_uint32), ("route", C.c_uint32)]


class Ctrl(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("law", "signal", "window", "r_min_bp", "r_max_bp", "r_const_bp",
                                           "t1", "t2", "slo_us", "calibrated", "n_rungs")] + \
               [("rungs_bp", C.c_uint32 * 8), ("bypass_mask", C.c_uint32), ("min_words_bypass", C.c_uint32)] + \
               [(n, C.c_uint32) for n in ("horizon_s", "w_lat", "w_q", "w_osc", "step_bp")]


class RunCfg(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("horizon_us", C.c_int64), ("w0_us", C.c_int64), ("w1_us", C.c_int64),
                ("poly_q16", C.c_int64 * 3), ("quality", C.c_uint32 * 5), ("record", C.c_uint32)]


RESULT_U64 = ["ticks", "candidates", "arrivals", "admitted", "served", "rewritten",
              "words_in", "words_out", "idle_us", "end_us", "queued_end", "inflight_end",
              "win_served", "win_words_in", "win_words_out", "win_idle_us",
              "sum_queue_us", "sum_ttft_us", "sum_e2e_us", "slo_violations"]
RESULT_U32 = ["e2e_p50_ms", "e2e_p99_ms", "ttft_p50_ms", "ttft_p99_ms", "median_r_bp",
              "t1", "t2", "activations", "first_act_s", "last_deact_s", "active_ingests", "flags"]
RESULT_F64 = ["energy_j", "win_energy_j"]
RESULT_Q = ["sim_active_p50", "sim_inactive_p50", "scored_active", "scored_inactive", "bypassed", "preemptions"]
RESULT_P = ["recompute_words"]
HIST_Q = 201
RESULT_EXTRA = ["e2e_exact_p50_us", "e2e_exact_p99_us", "ttft_exact_p50_us", "ttft_exact_p99_us",
                "int_system_us", "int_queue_us", "sum_sojourn_us", "tbt_samples", "tbt_sum_us", "tbt_max_us"]
SUMMARY_FIELDS = RESULT_U64 + RESULT_U32 + RESULT_F64 + RESULT_Q + RESULT_P


class Result(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in RESULT_U64] + [(n, C.c_uint32) for n in RESULT_U32] + \
               [(n, C.c_double) for n in RESULT_F64] + [(n, C.c_uint32) for n in RESULT_Q] + \
               [(n, C.c_uint64) for n in RESULT_P] + \
               [(n, C.c_uint64) for n in RESULT_EXTRA] + \
               [("hist_e2e", C.c_uint32 * HIST_LAT), ("hist_ttft", C.c_uint32 * HIST_LAT),
                ("hist_r", C.c_uint32 * HIST_R), ("hist_q_active", C.c_uint32 * HIST_Q),
                ("hist_q_inactive", C.c_uint32 * HIST_Q), ("n_series", C.c_uint32)]


class ReqLog(C.Structure):
    _fields_ = [("admit_us", C.c_uint64), ("first_us", C.c_uint64), ("done_us", C.c_uint64),
                ("R", C.c_uint32), ("r_bp", C.c_uint32), ("n_gaps", C.c_uint32), ("_pad", C.c_uint32)]


class CtrlLog(C.Structure):
    _fields_ = [("second", C.c_uint32), ("sample", C.c_uint32), ("k", C.c_uint32), ("r_bp", C.c_uint32),
                ("active", C.c_uint32), ("_pad", C.c_uint32), ("A", C.c_uint64)]


SECOND_ROW = np.dtype([("arrivals", "<u4"), ("admitted", "<u4"), ("first_tokens", "<u4"), ("completions", "<u4"),
                       ("tbt_count", "<u4"), ("idle_us", "<u4"), ("words_in", "<u4"), ("words_out", "<u4"),
                       ("sum_queue_us", "<u8"), ("sum_ttft_us", "<u8"), ("sum_e2e_us", "<u8"),
                       ("sum_tbt_us", "<u8")])


class SecondRow(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("arrivals", "admitted", "first_tokens", "completions", "tbt_count",
                                           "idle_us", "words_in", "words_out")] + \
               [(n, C.c_uint64) for n in ("sum_queue_us", "sum_ttft_us", "sum_e2e_us", "sum_tbt_us")]


class Log(C.Structure):
    _fields_ = [("req", P(ReqLog)), ("gaps", u64p), ("cap_gaps", C.c_uint64), ("n_gaps", C.c_uint64),
                ("ctrl", P(CtrlLog)), ("cap_ctrl", C.c_uint64), ("n_ctrl", C.c_uint64),
                ("series", u32p), ("cap_series", C.c_uint64),
                ("rows", P(SecondRow)), ("cap_rows", C.c_uint64), ("n_rows", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.orc_philox.argtypes = [C.c_uint32, C.c_uint32, u32p, u32p]
        L.orc_neglog_q32.argtypes = [C.c_uint32]
        L.orc_neglog_q32.restype = C.c_uint64
        L.orc_log2_table.argtypes = [C.c_uint32]
        L.orc_log2_table.restype = C.c_uint64
        L.orc_lat_bin.argtypes = [C.c_uint64]
        L.orc_lat_bin.restype = C.c_uint32
        L.orc_lat_edge.argtypes = [C.c_uint32]
        L.orc_lat_edge.restype = C.c_uint64
        L.orc_arrivals.argtypes = [P(Inputs), C.c_uint64, P(Request), C.c_uint64]
        L.orc_arrivals.restype = C.c_int64
        L.orc_simulate.argtypes = [P(Request), C.c_uint64, P(Profile), P(Ctrl), P(RunCfg), P(Result), P(Log)]
        L.orc_simulate_replicas.argtypes = [P(Request), C.c_uint64, P(Profile), P(Ctrl), P(RunCfg), P(Result), P(Log)]
        L.orc_run_scenario.argtypes = [P(Inputs), C.c_uint64, P(Result), P(Log)]
        L.orc_percentile_u32.argtypes = [u32p, C.c_uint64, C.c_uint32]
        L.orc_percentile_u32.restype = C.c_uint32
        L.orc_calibrate.argtypes = [u32p, C.c_uint64, u32p, u32p]
        L.orc_map_rate.argtypes = [C.c_uint64, C.c_uint32, P(Ctrl)]
        L.orc_map_rate.restype = C.c_uint32
        L.orc_run_batch.argtypes = [P(Inputs), u64p, C.c_uint64, P(Result), C.c_int]
        L.orc_similarity.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int32, u32p]
        L.orc_similarity.restype = C.c_uint32
        L.orc_ctrl_trace.argtypes = [P(Ctrl), u32p, u32p, u32p, C.c_uint64, P(Result), P(CtrlLog)]
        _lib = L
    return _lib


# ---------------------------------------------------------------------------
def philox(k0: int, k1: int, ctr) -> tuple:
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    o = (C.c_uint32 * 4)()
    lib().orc_philox(k0 & 0xFFFFFFFF, k1 & 0xFFFFFFFF, c, o)
    return tuple(o)


def neglog_q32(u: int) -> int:
    return lib().orc_neglog_q32(u)


def log2_table(i: int) -> int:
    return lib().orc_log2_table(i)


def lat_bin(ms: int) -> int:
    return lib().orc_lat_bin(ms)


def lat_edge(b: int) -> int:
    return lib().orc_lat_edge(b)


def percentile(values, p: int) -> int:
    a = np.ascontiguousarray(values, dtype=np.uint32)
    return lib().orc_percentile_u32(a.ctypes.data_as(u32p), len(a), p)


def calibrate(series):
    a = np.ascontiguousarray(series, dtype=np.uint32)
    t1, t2 = C.c_uint32(), C.c_uint32()
    st = lib().orc_calibrate(a.ctypes.data_as(u32p), len(a), C.byref(t1), C.byref(t2))
    return st, t1.value, t2.value


def make_ctrl(law=0, signal=0, window=5, r_min_bp=500, r_max_bp=2000, r_const_bp=0, t1=0, t2=0,
              slo_us=0, calibrated=0, rungs=(), bypass_mask=0, min_words_bypass=0, horizon_s=0, w_lat=0, w_q=0,
              w_osc=0, step_bp=0):
    c = Ctrl(law, signal, window, r_min_bp, r_max_bp, r_const_bp, t1, t2, slo_us, calibrated, len(rungs))
    c.bypass_mask = bypass_mask
    c.min_words_bypass = min_words_bypass
    c.horizon_s, c.w_lat, c.w_q, c.w_osc, c.step_bp = horizon_s, w_lat, w_q, w_osc, step_bp
    for i, r in enumerate(rungs):
        c.rungs_bp[i] = r
    return c


def map_rate(A: int, k: int, ctrl: Ctrl) -> int:
    return lib().orc_map_rate(A, k, C.byref(ctrl))


def ctrl_trace(ctrl: Ctrl, samples, words=None, seconds=None) -> dict:
    """The controller alone (every law) over per-second samples: returns the
    per-ingest log (r_bp, active, k, A) and the transition summary."""
    n = len(samples)
    x = np.ascontiguousarray(samples, dtype=np.uint32)
    sec = np.ascontiguousarray(range(n) if seconds is None else seconds, dtype=np.uint32)
    w = np.ascontiguousarray(np.zeros(n) if words is None else words, dtype=np.uint32)
    r = Result()
    log = (CtrlLog * max(n, 1))()
    rc = lib().orc_ctrl_trace(C.byref(ctrl), sec.ctypes.data_as(u32p), x.ctypes.data_as(u32p),
                              w.ctypes.data_as(u32p), n, C.byref(r), log)
    if rc != 0:
        raise RuntimeError("oracle ctrl_trace failed")
    return dict(r=[e.r_bp for e in log[:n]], active=[e.active for e in log[:n]], k=[e.k for e in log[:n]],
                A=[e.A for e in log[:n]], activations=r.activations, first_act_s=r.first_act_s,
                last_deact_s=r.last_deact_s, active_ingests=r.active_ingests)


class Bound:
    """Column arrays pinned in memory + the orc_inputs struct pointing at them."""

    _SPEC = [("knot_t", np.int64), ("knot_lam", np.uint32), ("trace_knot_off", np.uint32),
             ("trace_n_knots", np.uint32), ("trace_cap", np.uint32), ("trace_kind", np.uint32),
             ("arr_a", np.int64), ("arr_L", np.uint32), ("arr_input", np.uint32), ("arr_cls", np.uint32),
             ("prof_t0", np.uint32), ("prof_knee", np.uint32), ("prof_slope", np.uint32), ("prof_kv", np.uint32),
             ("prof_maxb", np.uint32), ("prof_prefill_ns", np.uint32), ("prof_kv_cap", np.uint32),
             ("prof_prefill_mode", np.uint32), ("prof_kv_policy", np.uint32), ("prof_tpw", np.uint32),
             ("prof_replicas", np.uint32), ("prof_route", np.uint32),
             ("prof_e_in", np.float64), ("prof_e_out", np.float64), ("prof_p_idle", np.float64),
             ("ctrl_law", np.uint32), ("ctrl_signal", np.uint32), ("ctrl_window", np.uint32),
             ("ctrl_rmin", np.uint32), ("ctrl_rmax", np.uint32), ("ctrl_rconst", np.uint32),
             ("ctrl_t1", np.uint32), ("ctrl_t2", np.uint32), ("ctrl_slo_us", np.uint32),
             ("ctrl_calibrated", np.uint32), ("ctrl_nrungs", np.uint32), ("ctrl_rungs", np.uint32),
             ("ctrl_bypass_mask", np.uint32), ("ctrl_min_words", np.uint32),
             ("ctrl_horizon", np.uint32), ("ctrl_wlat", np.uint32), ("ctrl_wq", np.uint32), ("ctrl_wosc", np.uint32),
             ("ctrl_step", np.uint32),
             ("tab_L", np.int32), ("tab_I", np.int32), ("tab_fvar", np.int32), ("tab_noise", np.int32),
             ("tab_fcomp", np.int32), ("poly_q16", np.int64), ("tab_qnoise", np.int32), ("quality", np.uint32),
             ("class_cum", np.uint32),
             ("sc_seed", np.uint32), ("sc_wid", np.uint64), ("sc_trace", np.uint32), ("sc_profile", np.uint32),
             ("sc_ctrl", np.uint32), ("sc_segment", np.uint32), ("sc_mode", np.uint32),
             ("sc_horizon", np.int64), ("sc_w0", np.int64), ("sc_w1", np.int64),
             ("sc_calib_src", np.uint32), ("sc_record", np.uint32)]
    _CT = {np.int64: i64p, np.uint32: u32p, np.int32: i32p, np.float64: f64p, np.uint64: u64p}

    def __init__(self, cols: dict):
        self.arrays = {}
        kw = {}
        for name, dt in self._SPEC:
            a = np.ascontiguousarray(cols[name], dtype=dt)
            if a.size == 0:
                a = np.zeros(1, dtype=dt)
            self.arrays[name] = a
            kw[name] = a.ctypes.data_as(self._CT[dt])
        self.n = len(cols["sc_seed"])
        self.st = Inputs(n_scenarios=self.n, **kw)


def _result_dict(r: Result, hist=True) -> dict:
    d = {n: getattr(r, n) for n in SUMMARY_FIELDS + RESULT_EXTRA}
    d["n_series"] = r.n_series
    if hist:
        d["hist_e2e"] = np.frombuffer(r.hist_e2e, dtype=np.uint32).copy()
        d["hist_ttft"] = np.frombuffer(r.hist_ttft, dtype=np.uint32).copy()
        d["hist_r"] = np.frombuffer(r.hist_r, dtype=np.uint32).copy()
        d["hist_q_active"] = np.frombuffer(r.hist_q_active, dtype=np.uint32).copy()
        d["hist_q_inactive"] = np.frombuffer(r.hist_q_inactive, dtype=np.uint32).copy()
    return d


def arrivals(cols_or_bound, sid: int) -> np.ndarray:
    b = cols_or_bound if isinstance(cols_or_bound, Bound) else Bound(cols_or_bound)
    n = lib().orc_arrivals(C.byref(b.st), sid, None, 0)
    buf = (Request * max(n, 1))()
    m = lib().orc_arrivals(C.byref(b.st), sid, buf, n)
    assert m == n
    dt = np.dtype(Request)  # field layout and padding of orc_request
    return np.frombuffer(buf, dtype=dt, count=n).copy()


def run_scenario(cols_or_bound, sid: int, hist=True, ctrl_log_cap=0, series_cap=0, rows_cap=0) -> dict:
    """One scenario.  ctrl_log_cap / series_cap / rows_cap > 0 return the
    controller log, the recorded signal series and (record & 2) the per-second rows."""
    b = cols_or_bound if isinstance(cols_or_bound, Bound) else Bound(cols_or_bound)
    r = Result()
    log = Log()
    clog = (CtrlLog * max(ctrl_log_cap, 1))()
    ser = (C.c_uint32 * max(series_cap, 1))()
    rws = (SecondRow * max(rows_cap, 1))()
    if rows_cap:
        log.rows = rws
        log.cap_rows = rows_cap
    if ctrl_log_cap:
        log.ctrl = clog
        log.cap_ctrl = ctrl_log_cap
    if series_cap:
        log.series = ser
        log.cap_series = series_cap
    rc = lib().orc_run_scenario(C.byref(b.st), sid, C.byref(r), C.byref(log))
    if rc != 0:
        raise RuntimeError(f"oracle failed on scenario {sid}")
    d = _result_dict(r, hist)
    if ctrl_log_cap:
        d["ctrl_log"] = [dict(second=c.second, sample=c.sample, k=c.k, r_bp=c.r_bp, active=c.active, A=c.A)
                         for c in clog[:min(log.n_ctrl, ctrl_log_cap)]]
    if series_cap:
        d["series"] = np.frombuffer(ser, dtype=np.uint32, count=min(r.n_series, series_cap)).copy()
    if rows_cap:
        d["rows"] = np.frombuffer(rws, dtype=SECOND_ROW, count=min(log.n_rows, rows_cap)).copy()
    d["n_ctrl"] = log.n_ctrl
    return d


def run_batch(cols_or_bound, sids=None, nthreads=None) -> list:
    b = cols_or_bound if isinstance(cols_or_bound, Bound) else Bound(cols_or_bound)
    if sids is None:
        sids = np.arange(b.n, dtype=np.uint64)
    sids = np.ascontiguousarray(sids, dtype=np.uint64)
    res = (Result * max(len(sids), 1))()
    nt = nthreads or os.cpu_count() or 1
    rc = lib().orc_run_batch(C.byref(b.st), sids.ctypes.data_as(u64p), len(sids), res, nt)
    if rc != 0:
        raise RuntimeError("oracle batch failed")
    return [_result_dict(res[i], hist=False) for i in range(len(sids))]


QUALITY_DEFAULT = (8800, 8700, 6500, 2000, 4000)


def similarity(U: int, R: int, active: bool, noise: int = 0, q=QUALITY_DEFAULT) -> int:
    qq = (C.c_uint32 * 5)(*q)
    return lib().orc_similarity(U, R, 1 if active else 0, noise, qq)


def simulate(requests, profile: dict, ctrl: Ctrl | None = None, mode=0, horizon_us=10**12,
             w0_us=0, w1_us=2**62, poly_q16=(0, 65536, 0), record=0, gap_cap=100000, ctrl_log_cap=10000,
             quality=QUALITY_DEFAULT, multi=False):
    """Run the DES on an explicit request list (hand fixtures, brute-force pins).

    ``requests``: iterable of dicts with a_us, input, U and optionally L, P, fcomp_q16, j.
    """
    reqs = list(requests)
    n = len(reqs)
    rq = (Request * max(n, 1))()
    for i, q in enumerate(reqs):
        rq[i] = Request(int(q["a_us"]), int(q.get("j", i)), int(q.get("L", q["U"])), int(q["input"]),
                        int(q["U"]), int(q.get("P", q.get("L", q["U"]))), int(q.get("fcomp_q16", 65536)),
                        int(q.get("qnoise", 0)), int(q.get("cls", 0)))
    pr = Profile(profile["t0_us"], profile["knee"], profile["slope_us"], profile.get("kv_ns_per_word", 0),
                 profile["max_batch"], profile["prefill_ns_per_word"], profile.get("e_in", 0.05),
                 profile.get("e_out", 0.5), profile.get("p_idle", 300.0), profile.get("kv_cap_words", 0),
                 profile.get("prefill_mode", 0), profile.get("kv_policy", 0), profile.get("tpw_q16", 0),
                 profile.get("replicas", 0), profile.get("route", 0))
    c = ctrl if ctrl is not None else make_ctrl()
    cfg = RunCfg(mode, horizon_us, w0_us, w1_us, (C.c_int64 * 3)(*poly_q16), (C.c_uint32 * 5)(*quality), record)
    r = Result()
    log = Log()
    reqlog = (ReqLog * max(n, 1))()
    gaps = (C.c_uint64 * (2 * gap_cap))()
    clog = (CtrlLog * max(ctrl_log_cap, 1))()
    ser = (C.c_uint32 * 200000)()
    log.req = reqlog
    log.gaps = gaps
    log.cap_gaps = gap_cap
    log.ctrl = clog
    log.cap_ctrl = ctrl_log_cap
    log.series = ser
    log.cap_series = 200000
    fn = lib().orc_simulate_replicas if multi else lib().orc_simulate  # multi: the replica DES at any count
    rc = fn(rq, n, C.byref(pr), C.byref(c), C.byref(cfg), C.byref(r), C.byref(log))
    if rc != 0:
        raise RuntimeError("oracle simulate failed")
    d = _result_dict(r)
    d["requests"] = [dict(admit_us=x.admit_us, first_us=x.first_us, done_us=x.done_us, R=x.R, r_bp=x.r_bp,
                          n_gaps=x.n_gaps) for x in reqlog[:n]]
    g = np.frombuffer(gaps, dtype=np.uint64, count=2 * min(log.n_gaps, gap_cap)).reshape(-1, 2)
    d["gaps"] = [[] for _ in range(n)]
    for m, gap in g:
        d["gaps"][int(m)].append(int(gap))
    d["ctrl_log"] = [dict(second=x.second, sample=x.sample, k=x.k, r_bp=x.r_bp, active=x.active, A=x.A)
                     for x in clog[:min(log.n_ctrl, ctrl_log_cap)]]
    d["series"] = np.frombuffer(ser, dtype=np.uint32, count=min(r.n_series, 200000)).copy()
    return d

"""ctypes mirror of include/bellman_sim.h (argument marshalling only).

Loads the in-tree ``libbellman_sim.so``.  There is no fallback: if the library
is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbellman_sim.so")

TABLE_N = 4096
HIST_LAT = 896
HIST_R = 512
HIST_Q = 201
SEG_HIST_WORDS = 2 * HIST_LAT + HIST_R + 2 * HIST_Q
NONE = 0xFFFFFFFF
MAX_PEERS = 8
FLAG_TRUNCATED, FLAG_DEGENERATE_CALIB, FLAG_SERIES_OVERFLOW, FLAG_DONE = 0x1, 0x2, 0x4, 0x100

KNOT = np.dtype([("t_us", "<i8"), ("lam_mrps", "<u4"), ("_pad", "<u4")])
TRACE = np.dtype([("knot_offset", "<u4"), ("n_knots", "<u4"), ("arrival_cap", "<u4"), ("kind", "<u4")])
ARRIVAL = np.dtype([("a_us", "<i8"), ("L_words", "<u4"), ("input_words", "<u4"), ("cls", "<u4"), ("_pad", "<u4")])
PROFILE = np.dtype([("t0_us", "<u4"), ("knee", "<u4"), ("slope_us", "<u4"), ("kv_ns_per_word", "<u4"),
                    ("max_batch", "<u4"), ("prefill_ns_per_word", "<u4"), ("kv_cap_words", "<u4"), ("prefill_mode", "<u4"),
                    ("kv_policy", "<u4"), ("tpw_q16", "<u4"), ("e_in_j_per_word", "<f8"), ("e_out_j_per_word", "<f8"), ("p_idle_w", "<f8"),
                    ("replicas", "<u4"), ("route", "<u4")])
CTRL = np.dtype([(n, "<u4") for n in ("law", "signal", "window", "r_min_bp", "r_max_bp", "r_const_bp", "t1", "t2",
                                       "slo_us", "calibrated", "n_rungs")] + [("rungs_bp", "<u4", (8,))] +
                [("bypass_mask", "<u4"), ("min_words_bypass", "<u4")] +
                [(n, "<u4") for n in ("horizon_s", "w_lat", "w_q", "w_osc", "step_bp")])
SCENARIO = np.dtype([("seed_index", "<u4"), ("trace", "<u4"), ("wid", "<u8"), ("profile", "<u4"), ("ctrl", "<u4"),
                     ("segment", "<u4"), ("mode", "<u4"), ("horizon_us", "<i8"), ("w0_us", "<i8"),
                     ("w1_us", "<i8"), ("calib_src", "<u4"), ("record", "<u4")])
STATS_U64 = ["scenario_id", "ticks", "candidates", "arrivals", "admitted", "served", "rewritten",
             "words_in", "words_out", "idle_us", "end_us", "queued_end", "inflight_end",
             "win_served", "win_words_in", "win_words_out", "win_idle_us",
             "sum_queue_us", "sum_ttft_us", "sum_e2e_us", "slo_violations"]
STATS_U32 = ["e2e_p50_ms", "e2e_p99_ms", "ttft_p50_ms", "ttft_p99_ms", "median_r_bp",
             "t1", "t2", "activations", "first_act_s", "last_deact_s", "active_ingests", "flags",
             "segment", "bypassed"]
STATS_Q = ["sim_active_p50", "sim_inactive_p50", "scored_active", "scored_inactive"]
STATS = np.dtype([(n, "<u8") for n in STATS_U64] + [(n, "<u4") for n in STATS_U32] +
                 [("energy_j", "<f8"), ("win_energy_j", "<f8")] + [(n, "<u4") for n in STATS_Q] +
                 [("preemptions", "<u4"), ("_pad2", "<u4"), ("recompute_words", "<u8")])
SECOND_ROW = np.dtype([(n, "<u4") for n in ("arrivals", "admitted", "first_tokens", "completions", "tbt_count",
                                              "idle_us", "words_in", "words_out")] +
                      [(n, "<u8") for n in ("sum_queue_us", "sum_ttft_us", "sum_e2e_us", "sum_tbt_us")])
CTRL_ROW = np.dtype([("second", "<u4"), ("sample", "<u4"), ("k", "<u4"), ("r_bp", "<u4"), ("active", "<u4"),
                     ("_pad", "<u4"), ("A", "<u8")])
RECORD_SIGNAL, RECORD_SECONDS = 0x1, 0x2
assert SECOND_ROW.itemsize == 64 and CTRL_ROW.itemsize == 32
assert ARRIVAL.itemsize == 24
assert KNOT.itemsize == 16 and TRACE.itemsize == 16 and PROFILE.itemsize == 72
assert CTRL.itemsize == 104 and SCENARIO.itemsize == 64 and STATS.itemsize == 272


class Models(C.Structure):
    _fields_ = [("L_words", C.c_void_p), ("I_words", C.c_void_p), ("fvar_q16", C.c_void_p),
                ("noise", C.c_void_p), ("fcomp_q16", C.c_void_p), ("poly_q16", C.c_int64 * 3),
                ("qnoise", C.c_void_p), ("quality", C.c_uint32 * 5), ("class_cum", C.c_uint32 * 4),
                ("_pad", C.c_uint32 * 3)]


class Desc(C.Structure):
    _fields_ = [("knots", C.c_void_p), ("n_knots", C.c_uint32),
                ("traces", C.c_void_p), ("n_traces", C.c_uint32),
                ("profiles", C.c_void_p), ("n_profiles", C.c_uint32),
                ("ctrls", C.c_void_p), ("n_ctrls", C.c_uint32),
                ("models", Models),
                ("scenarios", C.c_void_p), ("n_scenarios", C.c_uint64),
                ("n_segments", C.c_uint32), ("_pad", C.c_uint32),
                ("arrivals", C.c_void_p), ("n_arrivals", C.c_uint64)]


EXPORTS = {
    "bellman_sim_workspace_bytes": (C.c_size_t, [C.POINTER(Desc)]),
    "bellman_sim_create": (C.c_int, [C.POINTER(Desc), C.c_void_p, C.c_size_t, C.c_int, C.c_void_p,
                                     C.POINTER(C.c_void_p)]),
    "bellman_sim_run": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]),
    "bellman_sim_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_void_p]),
    "bellman_sim_stats_strided": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                            C.c_void_p]),
    "bellman_sim_segment_hist": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "bellman_sim_reset": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bellman_sim_series": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                     C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p]),
    "bellman_sim_last_launches": (C.c_uint32, [C.c_void_p]),
    "bellman_sim_last_engines": (C.c_uint32, [C.c_void_p]),
    "bellman_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    "bellman_ipc_open": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "bellman_ipc_close": (C.c_int, [C.c_void_p]),
    "bellman_sim_set_peers": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_uint32]),
    "bellman_sim_destroy": (None, [C.c_void_p]),
    "bellman_status_string": (C.c_char_p, [C.c_int]),
    "bellman_sim_last_error": (C.c_char_p, [C.c_void_p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libbellman_sim.so (raises if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -c 'import __graft_entry__ as g; g.build()')")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class BellmanError(RuntimeError):
    pass


def check(status: int, handle=None):
    if status != 0:
        L = lib()
        msg = L.bellman_sim_last_error(handle).decode(errors="replace")
        raise BellmanError(f"{L.bellman_status_string(status).decode()}: {msg}")

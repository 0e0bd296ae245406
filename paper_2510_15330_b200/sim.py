"""Thin Python front end of the C ABI (argument marshalling only).

Every step of the simulation runs in the CUDA kernels of libbellman_sim.so;
this module only packs the column arrays produced by ``workloads`` into the
ABI structs of include/bellman_sim.h, owns the device workspace (a torch
uint8 tensor) and forwards calls.  PyTorch provides device memory and streams.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _abi as A


def pack(cols: dict, pinned: bool = False) -> dict:
    """Column arrays -> ABI structured arrays (host memory, optionally pinned)."""

    def alloc(dtype, n):
        n = max(int(n), 1)
        if pinned:
            t = torch.empty(n * dtype.itemsize, dtype=torch.uint8, pin_memory=True)
            return t.numpy().view(dtype), t
        return np.zeros(n, dtype=dtype), None

    keep = []
    out = {}
    nk = len(cols["knot_t"])
    knots, k = alloc(A.KNOT, nk)
    keep.append(k)
    knots[:nk]["t_us"] = cols["knot_t"]
    knots[:nk]["lam_mrps"] = cols["knot_lam"]
    nt = len(cols["trace_knot_off"])
    traces, k = alloc(A.TRACE, nt)
    keep.append(k)
    traces[:nt]["knot_offset"] = cols["trace_knot_off"]
    traces[:nt]["n_knots"] = cols["trace_n_knots"]
    traces[:nt]["arrival_cap"] = cols["trace_cap"]
    traces[:nt]["kind"] = cols.get("trace_kind", np.zeros(nt, dtype=np.uint32))
    na = len(cols.get("arr_a", ()))
    arrs, k = alloc(A.ARRIVAL, na)
    keep.append(k)
    if na:
        arrs[:na]["a_us"] = cols["arr_a"]
        arrs[:na]["L_words"] = cols["arr_L"]
        arrs[:na]["input_words"] = cols["arr_input"]
        arrs[:na]["cls"] = cols["arr_cls"]
    npf = len(cols["prof_t0"])
    profs, k = alloc(A.PROFILE, npf)
    keep.append(k)
    for f, c in (("t0_us", "prof_t0"), ("knee", "prof_knee"), ("slope_us", "prof_slope"),
                 ("kv_ns_per_word", "prof_kv"), ("max_batch", "prof_maxb"),
                 ("prefill_ns_per_word", "prof_prefill_ns"), ("kv_cap_words", "prof_kv_cap"), ("prefill_mode", "prof_prefill_mode"),
                 ("kv_policy", "prof_kv_policy"), ("tpw_q16", "prof_tpw"), ("replicas", "prof_replicas"),
                 ("route", "prof_route"),
                 ("e_in_j_per_word", "prof_e_in"),
                 ("e_out_j_per_word", "prof_e_out"), ("p_idle_w", "prof_p_idle")):
        profs[:npf][f] = cols[c]
    nc = len(cols["ctrl_law"])
    ctrls, k = alloc(A.CTRL, nc)
    keep.append(k)
    for f, c in (("law", "ctrl_law"), ("signal", "ctrl_signal"), ("window", "ctrl_window"),
                 ("r_min_bp", "ctrl_rmin"), ("r_max_bp", "ctrl_rmax"), ("r_const_bp", "ctrl_rconst"),
                 ("t1", "ctrl_t1"), ("t2", "ctrl_t2"), ("slo_us", "ctrl_slo_us"),
                 ("calibrated", "ctrl_calibrated"), ("n_rungs", "ctrl_nrungs"), ("bypass_mask", "ctrl_bypass_mask"),
                 ("min_words_bypass", "ctrl_min_words"), ("horizon_s", "ctrl_horizon"), ("w_lat", "ctrl_wlat"),
                 ("w_q", "ctrl_wq"), ("w_osc", "ctrl_wosc"), ("step_bp", "ctrl_step")):
        ctrls[:nc][f] = cols[c]
    ctrls[:nc]["rungs_bp"] = np.asarray(cols["ctrl_rungs"]).reshape(nc, 8)
    ns = len(cols["sc_seed"])
    scs, k = alloc(A.SCENARIO, ns)
    keep.append(k)
    for f, c in (("seed_index", "sc_seed"), ("trace", "sc_trace"), ("wid", "sc_wid"), ("profile", "sc_profile"),
                 ("ctrl", "sc_ctrl"), ("segment", "sc_segment"), ("mode", "sc_mode"),
                 ("horizon_us", "sc_horizon"), ("w0_us", "sc_w0"), ("w1_us", "sc_w1"),
                 ("calib_src", "sc_calib_src"), ("record", "sc_record")):
        scs[:ns][f] = cols[c]
    tabs = {}
    for name in ("tab_L", "tab_I", "tab_fvar", "tab_noise", "tab_fcomp", "tab_qnoise"):
        t, k = alloc(np.dtype("<i4"), A.TABLE_N)
        keep.append(k)
        t[:] = cols[name]
        tabs[name] = t
    out.update(knots=knots, n_knots=nk, traces=traces, n_traces=nt, profiles=profs, n_profiles=npf,
               arrivals=arrs, n_arrivals=na,
               ctrls=ctrls, n_ctrls=nc, scenarios=scs, n_scenarios=ns, tables=tabs,
               poly_q16=np.asarray(cols["poly_q16"], dtype=np.int64), n_segments=int(cols["n_segments"]),
               quality=np.asarray(cols["quality"], dtype=np.uint32),
               class_cum=np.asarray(cols["class_cum"], dtype=np.uint32),
               _keep=keep)
    return out


def make_desc(pk: dict) -> A.Desc:
    t = pk["tables"]
    m = A.Models(t["tab_L"].ctypes.data, t["tab_I"].ctypes.data, t["tab_fvar"].ctypes.data,
                 t["tab_noise"].ctypes.data, t["tab_fcomp"].ctypes.data,
                 (C.c_int64 * 3)(*[int(x) for x in pk["poly_q16"]]), t["tab_qnoise"].ctypes.data,
                 (C.c_uint32 * 5)(*[int(x) for x in pk["quality"]]),
                 (C.c_uint32 * 4)(*[int(x) for x in pk["class_cum"]]), (C.c_uint32 * 3)(0, 0, 0))
    return A.Desc(pk["knots"].ctypes.data, pk["n_knots"], pk["traces"].ctypes.data, pk["n_traces"],
                  pk["profiles"].ctypes.data, pk["n_profiles"], pk["ctrls"].ctypes.data, pk["n_ctrls"], m,
                  pk["scenarios"].ctypes.data, pk["n_scenarios"], pk["n_segments"], 0,
                  pk["arrivals"].ctypes.data, pk["n_arrivals"])


def workspace_bytes(pk: dict) -> int:
    d = make_desc(pk)
    n = A.lib().bellman_sim_workspace_bytes(C.byref(d))
    if n == 0:
        raise A.BellmanError(A.lib().bellman_sim_last_error(None).decode())
    return int(n)


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


class Simulator:
    """One simulator handle bound to one CUDA device (one process per GPU)."""

    def __init__(self, cols: dict | None = None, device: int = 0, stream=None, packed: dict | None = None,
                 workspace: torch.Tensor | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("bellman_sim needs a CUDA device (there is no CPU fallback)")
        self.device = device
        self.pk = packed if packed is not None else pack(cols)
        self.n_scenarios = self.pk["n_scenarios"]
        self.n_segments = self.pk["n_segments"]
        desc = make_desc(self.pk)
        nbytes = self.pk.get("_ws_bytes") or workspace_bytes(self.pk)  # validated once per packed set
        self.pk["_ws_bytes"] = nbytes
        if workspace is None or workspace.numel() < nbytes:
            workspace = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        self.ws = workspace
        self.ws_bytes = nbytes
        h = C.c_void_p()
        A.check(A.lib().bellman_sim_create(C.byref(desc), C.c_void_p(workspace.data_ptr()), nbytes, device,
                                           C.c_void_p(_stream_ptr(stream)), C.byref(h)))
        self.h = h

    def run(self, first: int = 0, count: int | None = None, stride: int = 1, stream=None):
        if count is None:
            count = (self.n_scenarios - first + stride - 1) // stride
        A.check(A.lib().bellman_sim_run(self.h, first, count, stride, C.c_void_p(_stream_ptr(stream))), self.h)

    @property
    def last_launches(self) -> int:
        return int(A.lib().bellman_sim_last_launches(self.h))

    @property
    def last_engines(self) -> int:
        """Bit mask of the engines the last run launched (BELLMAN_ENGINE_*: 1/2/4 the
        warp-per-scenario loops, 8/16 the lane-per-scenario kernel K2L)."""
        return int(A.lib().bellman_sim_last_engines(self.h))

    def stats_device(self, out: torch.Tensor, first: int = 0, count: int | None = None, stream=None):
        count = self.n_scenarios - first if count is None else count
        assert out.is_cuda and out.numel() * out.element_size() >= count * A.STATS.itemsize
        A.check(A.lib().bellman_sim_stats(self.h, C.c_void_p(out.data_ptr()), first, count, 1,
                                          C.c_void_p(_stream_ptr(stream))), self.h)
        return out

    def stats(self, first: int = 0, count: int | None = None, out: np.ndarray | None = None, stream=None):
        count = self.n_scenarios - first if count is None else count
        if out is None:
            out = np.zeros(count, dtype=A.STATS)
        A.check(A.lib().bellman_sim_stats(self.h, C.c_void_p(out.ctypes.data), first, count, 0,
                                          C.c_void_p(_stream_ptr(stream))), self.h)
        return out

    def stats_shard(self, first: int, stride: int, count: int | None = None, out: np.ndarray | None = None,
                    stream=None):
        """Records of scenarios first, first+stride, ... (a rank's shard), packed, to host memory."""
        if count is None:
            count = (self.n_scenarios - first + stride - 1) // stride
        if out is None:
            out = np.zeros(count, dtype=A.STATS)
        assert out.nbytes >= count * A.STATS.itemsize
        A.check(A.lib().bellman_sim_stats_strided(self.h, C.c_void_p(out.ctypes.data), first, count, stride, 0,
                                                  C.c_void_p(_stream_ptr(stream))), self.h)
        return out

    def segment_hist(self, stream=None) -> np.ndarray:
        out = np.zeros((self.n_segments, A.SEG_HIST_WORDS), dtype=np.uint64)
        A.check(A.lib().bellman_sim_segment_hist(self.h, C.c_void_p(out.ctypes.data), 0,
                                                 C.c_void_p(_stream_ptr(stream))), self.h)
        return out

    def segment_hist_device(self, out: torch.Tensor, stream=None):
        A.check(A.lib().bellman_sim_segment_hist(self.h, C.c_void_p(out.data_ptr()), 1,
                                                 C.c_void_p(_stream_ptr(stream))), self.h)
        return out

    def series(self, sid: int, cap: int | None = None, stream=None):
        """Debug record mode (scenario.record & RECORD_SECONDS): the per-second
        rows and the controller log of scenario `sid` (host numpy arrays)."""
        if cap is None:
            cap = int(self.pk["scenarios"][sid]["horizon_us"] // 1_000_000 + 2)
        rows = np.zeros(cap, dtype=A.SECOND_ROW)
        ctrl = np.zeros(cap, dtype=A.CTRL_ROW)
        nr, nc = C.c_uint64(), C.c_uint64()
        A.check(A.lib().bellman_sim_series(self.h, sid, C.c_void_p(rows.ctypes.data), cap, C.byref(nr),
                                           C.c_void_p(ctrl.ctypes.data), cap, C.byref(nc),
                                           C.c_void_p(_stream_ptr(stream))), self.h)
        return rows[: min(nr.value, cap)], ctrl[: min(nc.value, cap)]

    def set_peers(self, ptrs: list):
        """Fused exchange (include/bellman_sim.h): later runs also
        store every record they finish into these device record arrays (every
        rank's full-size array, mapped into this process); [] turns it off."""
        arr = (C.c_void_p * max(len(ptrs), 1))(*[C.c_void_p(int(x)) for x in ptrs])
        A.check(A.lib().bellman_sim_set_peers(self.h, arr, len(ptrs)), self.h)
        self._peers = list(ptrs)

    def reset(self, stream=None):
        A.check(A.lib().bellman_sim_reset(self.h, C.c_void_p(_stream_ptr(stream))), self.h)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            A.lib().bellman_sim_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stats_to_dicts(arr: np.ndarray) -> list:
    names = A.STATS.names
    return [{n: (arr[i][n].item() if np.ndim(arr[i][n]) == 0 else arr[i][n]) for n in names} for i in range(len(arr))]

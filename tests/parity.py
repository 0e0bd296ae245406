"""Helpers comparing the CUDA path (through the C ABI) with the CPU oracle."""
from __future__ import annotations

import numpy as np

import oracle

ENERGY_RTOL = 1e-9  # BASELINE.json north_star: "within 1e-9 relative error for fp64 energy"
INT_FIELDS = [f for f in oracle.SUMMARY_FIELDS if f not in ("energy_j", "win_energy_j")]


def run_gpu(cols, first=0, count=None, stride=1, per_scenario_segments=False):
    import torch

    from paper_2510_15330_b200 import Simulator

    if per_scenario_segments:
        cols = dict(cols)
        cols["sc_segment"] = np.arange(len(cols["sc_seed"]), dtype=np.uint32)
        cols["n_segments"] = len(cols["sc_seed"])
    sim = Simulator(cols, device=0)
    sim.run(first=first, count=count, stride=stride)
    torch.cuda.synchronize()
    st = sim.stats()
    hist = sim.segment_hist() if per_scenario_segments else None
    launches = sim.last_launches
    sim.close()
    return st, hist, launches


def compare(gpu_rec, orc: dict, sid: int, hist_row=None):
    """Bit-exact on every integer field, energy within 1e-9 relative."""
    errs = []
    for k in INT_FIELDS:
        g = int(gpu_rec[k])
        if k == "flags":
            g &= 0xFF
        if g != int(orc[k]):
            errs.append(f"{k}: gpu={g} oracle={orc[k]}")
    for k in ("energy_j", "win_energy_j"):
        g, o = float(gpu_rec[k]), float(orc[k])
        if abs(g - o) > ENERGY_RTOL * max(abs(o), 1e-300):
            errs.append(f"{k}: gpu={g!r} oracle={o!r}")
    if int(gpu_rec["scenario_id"]) != sid:
        errs.append(f"scenario_id {int(gpu_rec['scenario_id'])} != {sid}")
    if not (int(gpu_rec["flags"]) & 0x100):
        errs.append("record not written (FLAG_DONE missing)")
    if hist_row is not None:
        for name, lo, hi in (("hist_e2e", 0, 896), ("hist_ttft", 896, 1792), ("hist_r", 1792, 2304),
                             ("hist_q_active", 2304, 2505), ("hist_q_inactive", 2505, 2706)):
            if not np.array_equal(hist_row[lo:hi].astype(np.int64), orc[name].astype(np.int64)):
                d = np.nonzero(hist_row[lo:hi].astype(np.int64) != orc[name].astype(np.int64))[0][:5]
                errs.append(f"{name} differs at bins {d.tolist()}")
    return errs


def check_all(cols, sids=None, per_scenario_segments=True, nthreads=None):
    n = len(cols["sc_seed"])
    st, hist, _ = run_gpu(cols, per_scenario_segments=per_scenario_segments)
    sids = range(n) if sids is None else sids
    b = oracle.Bound(cols)
    bad = []
    for sid in sids:
        o = oracle.run_scenario(b, sid)
        e = compare(st[sid], o, sid, hist[sid] if hist is not None else None)
        if e:
            bad.append((sid, e))
    return bad, st

"""Throughput of the code paths on a C5-shaped workload (1/16 of C5: 65,536
scenarios, the same traces, seeds and controller grid), one launch each:
the TBT-specialised KV-free loop (C5 as is), the generic loop (token costs),
the NEXT-3 laws (MPC / BBR / PCC instead of the grid), and the multi-replica
loop (4 replicas x 16 slots, least loaded).  Prints ticks/s per variant and
the roofline fraction bench.py would report for it (SURVEY 8(d) algorithmic
warp-instructions / kernel time / the nominal issue peak at 1965 MHz)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2510_15330_b200 import Simulator  # noqa: E402

import bench  # noqa: E402  (the algorithmic-work formula of the bench line)


def variant(name):
    w = W.config_c5(n_seeds=256)
    if name == "tokens":
        w.profiles = [dict(p, tpw_q16=65536) for p in w.profiles]  # 1 token/word: same work, generic loop
    elif name == "next3_laws":
        laws = [W.mpc_ctrl(24_000), W.bbr_ctrl(3_000), W.pcc_ctrl(24_000)]
        w.ctrls = [w.ctrls[0]] + [laws[i % 3] for i in range(1, len(w.ctrls))]
    elif name in ("mpc", "bbr", "pcc", "map_generic"):
        c = {"mpc": W.mpc_ctrl(24_000), "bbr": W.bbr_ctrl(3_000), "pcc": W.pcc_ctrl(24_000),
             "map_generic": W.map_ctrl(24_000, 40_000)}[name]
        w.ctrls = [w.ctrls[0]] + [c] * (len(w.ctrls) - 1)
        if name == "map_generic":
            w.profiles = [dict(p, tpw_q16=65536) for p in w.profiles]
    elif name == "replicas4x16":
        w.profiles = [dict(p, replicas=4, max_batch=16) for p in w.profiles]
    elif name == "replicas4x16_kv":  # with a KV term (L8B's 50 ns per context word): the stepped leap
        w.profiles = [dict(p, replicas=4, max_batch=16, kv_ns_per_word=50) for p in w.profiles]
    return w


def main():
    out = {}
    names = sys.argv[1:] or ["c5_as_is", "tokens", "map_generic", "mpc", "bbr", "pcc", "replicas4x16",
                             "replicas4x16_kv"]
    for name in names:
        w = variant(name)
        sim = Simulator(w.columns())
        best = None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sim.run()
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        st = sim.stats()
        ticks = int(st["ticks"].astype(np.int64).sum())
        ops = bench.algorithmic_ops(st)  # SURVEY 8(d) per-unit counts x units, as bench.py
        peak = 148 * 4 * 1965e6  # nominal issue peak, warp-inst/s (bench.py's roofline denominator)
        out[name] = {"ms": round(best, 2), "ticks": ticks, "ticks_per_s": ticks / (best / 1e3),
                     "roofline_frac": ops / (best / 1e3) / peak}
        sim.close()
        print(name, out[name], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

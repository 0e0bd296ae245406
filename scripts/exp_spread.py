"""Development: is C2 latency-bound by its heaviest scenarios?  Kernel time and
scenario-ticks/s for C2 subsets and for more seeds (library from argv[1] if given)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2510_15330_b200 import _abi, sim  # noqa: E402

if len(sys.argv) > 1:
    _abi.LIB_PATH = sys.argv[1]


def t(w, reps=7):
    s = sim.Simulator(w.columns())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(reps + 1):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.run()
        b.record()
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    st = s.stats()
    ticks = st["ticks"].astype(np.int64)
    s.close()
    ms = statistics.median(ts)
    return ms, int(ticks.sum()), int(ticks.max()), len(ticks)


for name, w in [("C2", W.config_c2()),
                ("rate8 only", W.config_c2(rates=[8.0])),
                ("rate0.5 only", W.config_c2(rates=[0.5])),
                ("rates<=4", W.config_c2(rates=W.C2_RATES_RPS[:8])),
                ("C2 x4 seeds", W.config_c2(n_seeds=256)),
                ("C2 x16 seeds", W.config_c2(n_seeds=1024))]:
    ms, tk, tmax, n = t(w)
    print(f"{name:14s} n={n:6d} {ms:8.3f} ms  ticks={tk:.3e} max/scen={tmax}  {tk / ms / 1e6:8.3f} Gticks/s")

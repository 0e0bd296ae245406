"""One-off evidence: BASELINE configs[4] (C5, all 2^20 scenarios) in bench's
N = 1 launch configuration, EVERY record compared with the CPU oracle (bit-exact
integer fields, energy within 1e-9 relative), on the GPU box's host cores.
(The -m gpu suite samples id % 64 == 0; this covers the rest once.)"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_2510_15330_b200 import Simulator  # noqa: E402
from tests.parity import compare  # noqa: E402


def main():
    w = W.config_c5()
    cols = w.columns()
    sim = Simulator(cols)
    sim.run()
    torch.cuda.synchronize()
    st = sim.stats()
    print(f"engines mask {sim.last_engines} (8/16 = K2L lane-per-scenario, 1 = K2 warp-per-scenario)", flush=True)
    b = oracle.Bound(cols)
    n = w.n_scenarios
    bad, t0, chunk = 0, time.time(), 1 << 15
    ticks = 0
    for lo in range(0, n, chunk):
        sids = np.arange(lo, min(n, lo + chunk), dtype=np.uint64)
        rs = oracle.run_batch(b, sids)
        for s, o in zip(sids, rs):
            e = compare(st[int(s)], o, int(s))
            ticks += o["ticks"]
            if e:
                bad += 1
                if bad <= 10:
                    print("MISMATCH", int(s), e[:3], flush=True)
        print(f"{lo + len(sids)} / {n} records compared, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
    print(f"C5 full parity: {n} records, {ticks} oracle ticks (GPU {int(st['ticks'].astype(np.int64).sum())}), "
          f"{bad} mismatches, {os.cpu_count()} host cores, {time.time() - t0:.0f} s")
    assert bad == 0


if __name__ == "__main__":
    main()

"""Development A/B timing: kernel time of C2 for several builds of the library
(paths given on the command line), same process, alternating, median of N."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes  # noqa: E402

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2510_15330_b200 import _abi, sim  # noqa: E402


def main(paths, reps=15):
    reps = int(os.environ.get("AB_REPS", reps))
    # AB_WL: Python expression over W building the workload (default C2)
    cols = eval(os.environ.get("AB_WL", "W.config_c2()"), {"W": W}).columns()
    pk = sim.pack(cols)
    libs = []
    for p in paths:
        _abi._lib = None
        _abi.LIB_PATH = p
        libs.append(_abi.lib())
    res = {p: [] for p in paths}
    sims = []
    for p, L in zip(paths, libs):
        _abi._lib = L
        pk.pop("_ws_bytes", None)  # builds may lay the workspace out differently
        sims.append(sim.Simulator(packed=pk))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for it in range(reps + 2):
        for p, L, s in zip(paths, libs, sims):
            _abi._lib = L
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s.run()
            b.record()
            torch.cuda.synchronize()
            if it >= 2:
                res[p].append(a.elapsed_time(b))
    # every build's records of the last run, byte for byte, against the first build's
    recs = []
    for p, L, s in zip(paths, libs, sims):
        _abi._lib = L
        recs.append(s.stats().view("u1"))
    for p, r in zip(paths, recs):
        same = "records == first build" if (r == recs[0]).all() else "RECORDS DIFFER from the first build"
        print(f"{os.path.basename(p):40s} median {statistics.median(res[p]):7.3f} ms  min {min(res[p]):7.3f}  {same}")


if __name__ == "__main__":
    main(sys.argv[1:])

"""Development: run a workload once (after one warm-up) with the library at
argv[1] (for ncu A/B).  argv[2] (optional) is a Python expression over W
building the workload, default W.config_c2()."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2510_15330_b200 import _abi, sim  # noqa: E402

_abi.LIB_PATH = sys.argv[1]
w = eval(sys.argv[2], {"W": W}) if len(sys.argv) > 2 else W.config_c2()
s = sim.Simulator(w.columns())
for _ in range(2):
    s.run()
torch.cuda.synchronize()

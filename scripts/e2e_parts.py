"""Development: where the e2e step's time goes (create / run / stats), C2."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2510_15330_b200 import Simulator, _abi, pack  # noqa: E402

cols = W.config_c2().columns()
pk = pack(cols, pinned=True)
n = len(cols["sc_seed"])
host = torch.empty((n, _abi.STATS.itemsize), dtype=torch.uint8, pin_memory=True).numpy().view(_abi.STATS).reshape(-1)
sim0 = Simulator(packed=pk)
ws = sim0.ws
s = torch.cuda.current_stream()
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim = Simulator(packed=pk, workspace=ws, stream=s)
    t1 = time.perf_counter()
    sim.run(stream=s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    sim.stats(out=host, stream=s)
    t3 = time.perf_counter()
    sim.close()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.3f} ms  run {1e3*(t2-t1):.3f}  stats {1e3*(t3-t2):.3f}  close {1e3*(t4-t3):.3f}")

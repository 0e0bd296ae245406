#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small configs.
set -u
cd "$(dirname "$0")/.."
cat > /tmp/san_run.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, workloads as W
from paper_2510_15330_b200 import Simulator
pre = W.config_paper_pair(1)  # NEXT-4 preemption (global scratch, re-admission stack)
pre.profiles = [dict(p, kv_cap_words=150_000, kv_policy=1) for p in pre.profiles]
# round 2: NEXT-3 laws, NEXT-4 token costs and multi-replica routing
r2 = W.custom([W.paper_trace(), W.const_trace(4.0, 200)],
              [dict(W.PROFILES["P24"], replicas=4, max_batch=16, route=1, tpw_q16=85197),
               dict(W.PROFILES["L8B"], replicas=2, max_batch=8), dict(W.PROFILES["P24"], tpw_q16=49152)],
              [W.OFF, W.mpc_ctrl(24_000), W.bbr_ctrl(3_000), W.pcc_ctrl(24_000)],
              [W.Scenario(k, wid=k % 2, trace=k % 2, profile=k % 3, ctrl=k % 4, segment=0, mode=k % 2,
                          horizon_us=900 * W.US) for k in range(24)])
for w in (W.config_c1(), W.config_c2(n_seeds=1, rates=[0.5, 4.0], horizon_s=120), W.config_paper_pair(0), pre, r2):
    for s in w.scenarios[:2]:
        s.record |= 2
    sim = Simulator(w.columns())
    full = torch.zeros((w.n_scenarios, 272), dtype=torch.uint8, device='cuda')
    sim.set_peers([full.data_ptr()])  # the fused exchange's peer stores (a local array here)
    sim.run(); torch.cuda.synchronize()
    st = sim.stats()
    print(w.name, int(st['ticks'].sum()), flush=True)
PY
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_run.py 2>&1 | tail -6
  echo "exit $?"
done
# K2L (the lane-per-scenario kernel) on the same workloads: BELLMAN_LANE=2 takes
# it for runs of any size (its scenarios; the rest stay in the warp engines)
for tool in memcheck racecheck synccheck; do
  echo "== $tool (K2L)"
  BELLMAN_LANE=2 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_run.py 2>&1 | tail -6
  echo "exit $?"
done

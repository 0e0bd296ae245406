"""bench.py's N > 1 path end to end — two ranks under torch.distributed.run,
sharing one B200 (BELLMAN_BENCH_SHARE_GPU=1, gloo): strong-scaling shards, the
fused peer-memory summary exchange (checked inside bench.py byte for byte
against the all-gather of the same records), max-over-ranks timing, one JSON
line from rank 0.  A reduced C2 (16 seeds) keeps it to seconds."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra,lane", [([], "1"), (["--nccl-gather"], "1"), ([], "2")],
                         ids=["fused", "gather", "fused-K2L"])
def test_bench_two_ranks_one_gpu(extra, lane):
    """fused-K2L: the same with K2L forced at this size (BELLMAN_LANE=2): the
    lane kernel's peer stores and bench.py's lane roofline."""
    env = dict(os.environ, BELLMAN_BENCH_SHARE_GPU="1", BELLMAN_LANE=lane)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", "C2", "--seeds", "16", "--e2e-steps", "1", "--no-peak", "--no-cpu-baseline", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["scenarios"] == 2 * d["config"]["scenarios_per_gpu"] == 16 * 16 * 2
    assert d["value"] > 0 and d["gpu_launches"] > 0
    want = "fused" if not extra else "NCCL all-gather"
    assert d["exchange"].startswith(want), d["exchange"]
    assert d["e2e"]["d2h_bytes_per_step"] == d["config"]["scenarios_per_gpu"] * 272  # the rank's shard only
    if lane == "2":
        assert d["engines"]["mask"] & 0x18 and d["roofline"]["unit"] == "G int-lane-ops/s"

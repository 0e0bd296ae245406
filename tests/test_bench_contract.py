"""bench.py's reference arm runs on a GPU-less host (it times the oracle) and
prints the contract's JSON line: the product arm's metric, unit and config,
plus `impl`, `cpu_baseline` and `e2e`.  Checked here on a 2-seed C2 so that it
finishes in seconds; the driver runs it at full size."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench_line(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    sys.path.insert(0, ROOT)
    import bench

    d = _bench_line("--impl", "reference", "--steps", "2", "--warmup", "1", "--workload", "C2", "--seeds", "2")
    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["higher_is_better"] is True and d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["scaling"] == "strong"
    # the same config object the product arm prints at this N (the driver compares them)
    assert d["config"] == bench.config_dict("C2", 16 * 2 * 2, 1, 2)  # 16 rates x 2 seeds x {off, on}
    assert d["ticks_per_step"] > 0
    assert d["value"] > 0 and d["value"] == d["cpu_baseline"]["value"] == d["e2e"]["value"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--workload", "C2", "--seeds", "2"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_default_workload_is_c5_strong_scaled():
    """the bench line is BASELINE configs[4] (2^20 scenarios), the
    same scenario set at every N, sharded 2^20 / N per GPU."""
    sys.path.insert(0, ROOT)
    import bench

    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        args = bench.parse()
    finally:
        sys.argv = old
    assert args.workload == "C5" and args.warmup >= 3
    assert bench.config_dict("C5", 1 << 20, 8)["scenarios_per_gpu"] == 131072
    assert bench.config_dict("C5", 1 << 20, 1) != bench.config_dict("C5", 1 << 20, 2)

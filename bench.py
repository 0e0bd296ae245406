#!/usr/bin/env python
"""Benchmark: simulated scenario-ticks/s of the beLLMan simulator on B200.

Workload (BASELINE.json configs[4], the default): the
1M-scenario Monte Carlo sweep — 16 paper-trace variants x 16 controller
configs (OFF + 15 of C3's grid) x 4096 seeds = 2^20 scenarios, P24 decode-cost
model, drained.  Strong scaling: the job is the config's fixed scenario set at
every N; rank r of N runs ids r, r+N, ... (2^20 / N per GPU), heavy-first
inside its shard.  The one exchange step is the summary all-gather (fused into
the tick kernel's epilogue over peer memory, or NCCL all_gather with
--nccl-gather) plus the NCCL all_reduce of the integer segment histograms.
`--workload C2|C3|C4` times another BASELINE config the same way.

A step = one pass of the whole hot path (arrival generation, draws, decode
iterations, controller, accounting, histograms, percentiles) over the shard,
plus the exchange.  Inputs are resident in HBM when the timed region starts
(value); `e2e` repeats the step through the C ABI with host buffers
(descriptor H2D in bellman_sim_create, the rank's summaries D2H).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "simulated scenario-ticks/sec"
UNIT = "scenario-ticks/s"

# Survey §8(d) algorithmic integer work per unit (warp-instructions): a0 per
# tick, 130 per candidate and per admission (Philox-10 + -ln/table draws +
# thinning), 12 per completion, 40 per ingested second, 6 per prefill end.
A_TICK, A_CAND, A_ADMIT, A_DONE, A_SEC, A_PF = 12, 130, 130, 12, 40, 6
# Algorithmic HBM bytes per scenario: the 64 B descriptor read
# once and the 272 B summary record written once.
B_DESC, B_REC = 64, 272


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--nccl-gather", action="store_true",
                    help="N > 1: exchange summaries with a separate NCCL all-gather instead of the fused kernel stores")
    ap.add_argument("--workload", default="C5", choices=["C2", "C3", "C4", "C5"],
                    help="BASELINE config; C5 (configs[4], 2^20 scenarios) is the reported bench line")
    ap.add_argument("--no-peak", action="store_true", help="skip the integer-issue microbenchmark")
    ap.add_argument("--seeds", type=int, default=None,
                    help="tests only: override the config's seed count (the line then names the reduced set)")
    return ap.parse_args()


WORKLOAD_DESC = {
    "C2": "C2 rate sweep 0.5-8 RPS x 64 seeds x {off,on} = 2048 scenarios, L8B cost model, 600 s cutoff",
    "C3": "C3 controller grid (32 threshold pairs x 10 ladders + OFF) x 32 seeds = 10272 scenarios, paper trace, "
          "P24, drain",
    "C4": "C4 diurnal 24 h, 16 traces x 4 ctrls x 64 seeds = 4096 scenarios, P24, drain",
    "C5": "C5 Monte Carlo 16 trace variants x 16 ctrls x 4096 seeds = 2^20 scenarios, P24, drain",
}


def workload(name: str = "C5", seeds: int | None = None):
    """The BASELINE config as SURVEY §8(d) fixes it: the same scenario set at
    every N (strong scaling; ranks shard it).  `seeds` (tests only) shrinks it."""
    kw = {} if seeds is None else {"n_seeds": seeds}
    if name == "C3":
        return W.config_c3(**kw)
    if name == "C4":
        return W.config_c4(**kw)
    if name == "C2":
        return W.config_c2(**kw)
    return W.config_c5(**kw)


def config_dict(name: str, n_total: int, world: int, seeds: int | None = None) -> dict:
    """The `config` object of both arms' JSON lines (identical at equal N)."""
    desc = WORKLOAD_DESC[name] + ("" if seeds is None else f" [reduced: {seeds} seeds]")
    return {"workload": desc, "scenarios": n_total,
            "scenarios_per_gpu": (n_total + world - 1) // world,
            "parallelism": f"scenario-sharded x{world} (rank r runs ids r, r+{world}, ...)",
            "l2": "flushed between steps (256 MiB write)"}


def algorithmic_ops(st) -> float:
    """Survey §8(d) per-unit counts x the units the launch processed."""
    ticks = st["ticks"].astype(np.float64).sum()
    cand = st["candidates"].astype(np.float64).sum()
    adm = st["admitted"].astype(np.float64).sum()
    done = st["served"].astype(np.float64).sum()
    secs = (st["end_us"].astype(np.float64) // 1e6).sum()
    return A_TICK * ticks + A_CAND * cand + A_ADMIT * adm + A_DONE * done + A_SEC * secs + A_PF * adm


def latency_floor(w, pk, ws, local, stream, kernel_ms):
    """The launch's lower bound from serial latency: every segment's scenarios
    (<= 148, contiguous ids) launched alone — one warp per SM, no co-runners —
    and the slowest such launch taken.  No launch of the whole set can finish
    before its longest serial chain does.  None where segments are larger."""
    import torch

    from paper_2510_15330_b200 import Simulator

    seg = np.array([s.segment for s in w.scenarios])
    groups = []
    for g in range(w.n_segments):
        ids = np.nonzero(seg == g)[0]
        if len(ids) == 0:
            continue
        if len(ids) > 148 or ids[-1] - ids[0] + 1 != len(ids):
            return None
        groups.append((g, int(ids[0]), len(ids)))
    s3 = Simulator(packed=pk, device=local, stream=stream, workspace=ws)
    worst = (0.0, None)
    for g, first, cnt in groups:
        best = None
        for _ in range(2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s3.run(first=first, count=cnt, stride=1, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        if best > worst[0]:
            worst = (best, g)
    s3.close()
    names = getattr(w, "segment_names", None)
    return {"critical_ms": worst[0], "kernel_ms": kernel_ms, "frac": worst[0] / kernel_ms,
            "critical_segment": names[worst[1]] if names else worst[1],
            "note": "each segment's scenarios launched alone (one warp per SM): the slowest such launch is the "
                    "serial-latency floor of the whole launch; frac = floor / measured kernel time"}


def ncu_traffic(name: str, engine: str):
    """DRAM bytes (read + write) per launch of the dominant kernel (engine
    "lane" = K2L, "warp" = the warp-per-scenario tick kernel) on this
    workload, from the committed summary of one `ncu --set full` capture
    (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)[f"{name}/{engine}"]
        return int(t["dram_bytes_read"]) + int(t["dram_bytes_write"]), t["source"]
    except Exception:
        return None, None


def peaks():
    p = {"hbm_gbs": 6457.7, "sm_max_mhz": 1965.0, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update(hbm_gbs=m["hbm_gbs"], sm_max_mhz=m["sm_max_mhz"], src="measured")
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(cols, budget_s=12.0):
    """The oracle as it stands, on this host's cores, over a bounded sample of
    the same workload: whole passes (or a stride subsample of large configs)
    repeated until ~budget_s of CPU work."""
    import oracle

    b = oracle.Bound(cols)
    n = len(cols["sc_seed"])
    stride = max(1, n // 4096)
    sids = np.arange(0, n, stride, dtype=np.uint64)
    nthreads = os.cpu_count() or 1
    ticks, reps = 0, 0
    t0 = time.perf_counter()
    while True:
        rs = oracle.run_batch(b, sids=sids, nthreads=nthreads)
        ticks += sum(r["ticks"] for r in rs)
        reps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    what = "the full" if stride == 1 else f"a stride-{stride} subsample ({len(sids)} scenarios) of the"
    return {"value": ticks / dt, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"{reps} x {what} {n}-scenario workload ({ticks} scenario-ticks, {dt:.1f} s)"}


def run_reference(args):
    """The reference arm: the oracle as it stands on this host's cores, on this
    arm's workload (--workload), each step one bounded sample of it — the full
    scenario set for C2, a stride subsample of the larger configs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload(args.workload, args.seeds)
    cols = w.columns()
    import oracle

    b = oracle.Bound(cols)
    n = len(cols["sc_seed"])
    stride = max(1, n // 4096)
    sids = np.arange(0, n, stride, dtype=np.uint64)
    nthreads = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.run_batch(b, sids=sids, nthreads=nthreads)
    times, ticks = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        rs = oracle.run_batch(b, sids=sids, nthreads=nthreads)
        times.append(time.perf_counter() - t0)
        ticks = sum(r["ticks"] for r in rs)
    tot = sum(times)
    value = ticks * args.steps / tot
    what = "the full" if stride == 1 else f"a stride-{stride} subsample ({len(sids)} scenarios, id % {stride} == 0) of the"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": config_dict(args.workload, n, args.gpus, args.seeds),
            "ticks_per_step": int(ticks),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                             "sample": f"{args.steps} steps x {what} {n}-scenario workload"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def outputs(st_all, seg_hist, n_segments):
    """The metric's outputs (BASELINE.json: p50/p99 E2E latency, energy) over
    the whole job: nearest-rank p50/p99 on the merged E2E histogram (lower bin
    edge, ms; R13), served, energy.  Reporting only (not parity)."""
    def edge(b):  # log-linear bins, 32 per octave above 32 ms (DESIGN §2 a9)
        return b if b < 32 else (32 + b % 32) << (b // 32 - 1)

    def nr(h, p):
        n = int(h.sum())
        if n == 0:
            return None
        k = max(1, -(-p * n // 100))
        return edge(int(np.searchsorted(np.cumsum(h), k)))

    h = seg_hist[:, :896].sum(axis=0)
    seg = st_all["segment"].astype(np.int64)
    served = np.bincount(seg, weights=st_all["served"].astype(np.float64), minlength=n_segments)
    energy = np.bincount(seg, weights=st_all["energy_j"], minlength=n_segments)
    per_seg = [[g, nr(seg_hist[g, :896], 50), nr(seg_hist[g, :896], 99), int(served[g]), round(float(energy[g]), 1)]
               for g in range(n_segments)]
    return {"e2e_p50_ms": nr(h, 50), "e2e_p99_ms": nr(h, 99), "served": int(st_all["served"].sum()),
            "energy_j": float(st_all["energy_j"].sum()), "win_energy_j": float(st_all["win_energy_j"].sum()),
            "segments": {"columns": ["segment", "e2e_p50_ms", "e2e_p99_ms", "served", "energy_j"], "rows": per_seg},
            "note": f"job totals over {len(st_all)} scenarios / {n_segments} segments, and per segment; p50/p99 = "
                    "lower edge of the merged E2E histogram bin holding the nearest rank (R13)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2510_15330_b200 import Simulator, _abi, pack
    from paper_2510_15330_b200 import parallel as PAR

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: BELLMAN_BENCH_SHARE_GPU=1 folds ranks onto the visible GPUs (two
    # ranks on one B200 exercise the N > 1 path; gloo, since NCCL wants one GPU per rank)
    share = os.environ.get("BELLMAN_BENCH_SHARE_GPU") == "1"
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    w = workload(args.workload, args.seeds)
    cols = w.columns()
    n = w.n_scenarios
    mine = W.shard(n, rank, world)
    count = len(mine)
    stream = torch.cuda.current_stream()
    sim = Simulator(cols, device=local, stream=stream)
    stats_dev = torch.zeros((n, _abi.STATS.itemsize), dtype=torch.uint8, device=dev)
    full_dev = torch.zeros((n, _abi.STATS.itemsize), dtype=torch.uint8, device=dev)
    seg_dev = torch.zeros((w.n_segments, _abi.SEG_HIST_WORDS), dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    # N > 1: the summary all-gather is fused into the tick kernel — every record
    # is stored into every rank's full_dev over peer memory as it is finished
    # (CUDA IPC mappings over NVLink / NVSwitch); --nccl-gather times the
    # separate NCCL all-gather instead.  The segment-histogram sum stays NCCL.
    fused = world > 1 and not args.nccl_gather
    peers, fused_err = None, None
    if fused:
        peers, fused_err = PAR.open_peer_records(full_dev, rank, world, local)
        if peers is not None:
            sim.set_peers(peers.ptrs)
        else:
            fused = False
            print(f"bench: fused exchange unavailable ({fused_err}); using the NCCL all-gather",
                  file=sys.stderr, flush=True)

    def step():
        sim.reset(stream)
        sim.run(first=rank, count=count, stride=world, stream=stream)
        k_end = torch.cuda.Event(enable_timing=True)
        k_end.record(stream)
        if world > 1 and not fused:
            sim.stats_device(stats_dev, stream=stream)
            PAR.gather_summaries(PAR.shard_rows(stats_dev, rank, world), n, rank, world, out=full_dev)
        sim.segment_hist_device(seg_dev, stream=stream)
        PAR.reduce_segments(seg_dev)
        return k_end

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kends = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (untimed)
            starts[i].record(stream)
            kends.append(step())
            ends[i].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = [s.elapsed_time(k) for s, k in zip(starts, kends)]
    tot_ms = sum(step_ms)
    t = torch.tensor([tot_ms, sum(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, kern_tot = float(t[0]), float(t[1])
    # correctness-carrying unit count: ticks from the summaries of this step
    sim.stats_device(stats_dev, stream=stream)
    if fused:  # the fused exchange must equal the NCCL all-gather of the same records
        chk = PAR.gather_summaries(PAR.shard_rows(stats_dev, rank, world), n, rank, world)
        torch.cuda.synchronize()
        dist.barrier()
        assert torch.equal(chk, full_dev), "fused peer-memory exchange differs from the NCCL all-gather"
    st_local = stats_dev.cpu().numpy().view(_abi.STATS).reshape(-1)
    st_mine = st_local[mine]
    local_ticks = int(st_mine["ticks"].astype(np.int64).sum())
    local_ops = algorithmic_ops(st_mine)
    tt = torch.tensor([local_ticks, local_ops], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt)
    ticks_all, ops_all = float(tt[0]), float(tt[1])
    value = ticks_all * args.steps / (tot_ms / 1e3)
    launches = sim.last_launches
    engines = sim.last_engines
    lane_engine = bool(engines & 0x18)  # BELLMAN_ENGINE_LANE_KV0 | BELLMAN_ENGINE_LANE_KV
    if world > 1:
        st_all = (full_dev if fused else PAR.gather_summaries(PAR.shard_rows(stats_dev, rank, world), n, rank,
                                                              world)).cpu().numpy().view(_abi.STATS).reshape(-1)
    else:
        st_all = st_local
    outs = outputs(st_all, seg_dev.cpu().numpy().view(np.uint64), w.n_segments)

    # ---- e2e through the C ABI with host buffers (pinned): descriptors H2D,
    # the rank's shard simulated, the rank's records D2H ----
    pk = pack(cols, pinned=True)
    host_stats = torch.empty((count, _abi.STATS.itemsize), dtype=torch.uint8,
                             pin_memory=True).numpy().view(_abi.STATS).reshape(-1)
    e2e_ms = []
    for i in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s2 = Simulator(packed=pk, device=local, stream=stream, workspace=sim.ws)
        s2.run(first=rank, count=count, stride=world, stream=stream)
        if world == 1:
            s2.stats(out=host_stats, stream=stream)
        else:
            s2.stats_shard(rank, world, count, out=host_stats, stream=stream)
        b.record(stream)
        torch.cuda.synchronize()
        s2.close()
        if i > 0:
            e2e_ms.append(a.elapsed_time(b))
    e = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
    e2e_value = ticks_all * len(e2e_ms) / (float(e[0]) / 1e3) if e2e_ms else None
    h2d = int(sum(v.nbytes for k, v in pk.items() if isinstance(v, np.ndarray)) +
              sum(v.nbytes for v in pk["tables"].values()) + 8 * W.TABLE_N + 4 * n)
    d2h = int(count * _abi.STATS.itemsize)
    if peers is not None:  # every rank's kernels are done: unmap the peers' arrays
        torch.cuda.synchronize()
        dist.barrier()
        sim.set_peers([])
        peers.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    lat = latency_floor(w, pk, sim.ws, local, stream, kern_tot / args.steps) if world == 1 else None
    pk_ = peaks()
    clocks = clk.summary()
    mhz = pk_["sm_max_mhz"]
    kern_s = kern_tot / 1e3 / args.steps
    achieved = ops_all / max(world, 1) / kern_s / 1e9  # per GPU, G algorithmic int ops/s
    issue_peak = 148 * 4 * mhz * 1e6 / 1e9  # R_issue: 4 warp-instructions / clk / SM
    # R_lane from the guide's unit counts: 4 SMSPs x (alu + fma pipes, each one
    # warp-instruction / 2 clk) x 32 lanes = 128 integer lanes / clk / SM
    lane_peak = 148 * 128 * mhz * 1e6 / 1e9
    engine = "lane" if lane_engine else "warp"
    traffic, traffic_src = ncu_traffic(args.workload, engine)
    if lane_engine:
        # K2L: one thread per scenario, so an algorithmic op is one lane-op and
        # the binding roof is the SM's integer lanes (SURVEY 8(d) R_lane)
        roof = {"bound": "alu", "achieved": achieved, "peak": lane_peak, "unit": "G int-lane-ops/s",
                "frac": achieved / lane_peak, "traffic": traffic, "kernel": "bellman_lane_kernel (K2L)",
                "note": f"survey 8(d) algorithmic integer ops per launch (per-unit counts x the units processed) / "
                        f"kernel time (max over ranks, per GPU); K2L runs one scenario per lane, so the roof is R_lane "
                        f"= 148 SM x 128 int lanes/clk (4 SMSP x alu + fma pipes x 16 lanes/clk, guide) x {mhz:.0f} "
                        f"MHz ({pk_['src']} sm_max); traffic = DRAM bytes per launch ({traffic_src or 'no capture'})"}
        roof["issue_model"] = {"peak": issue_peak, "unit": "Gwarp-inst/s", "frac": achieved / issue_peak,
                               "note": "R_issue of SURVEY 8(d) (one warp per scenario: every algorithmic op takes a "
                                       "warp issue slot); K2L issues one instruction for up to 32 scenarios, so it "
                                       "runs above that ceiling"}
    else:
        roof = {"bound": "alu", "achieved": achieved, "peak": issue_peak, "unit": "Gwarp-inst/s",
                "frac": achieved / issue_peak, "traffic": traffic, "kernel": "bellman_tick_kernel (K2)",
                "note": f"survey 8(d) algorithmic warp-instructions per launch / kernel time (max over ranks, per "
                        f"GPU); peak = 148 SM x 4 issue/clk x {mhz:.0f} MHz ({pk_['src']} sm_max); traffic = DRAM "
                        f"bytes per launch ({traffic_src or 'no capture'})"}
    if not args.no_peak:
        # measured integer issue / lane throughput (microbenchmark, after the timed region)
        from paper_2510_15330_b200 import peak as PEAK

        mb = PEAK.measure(local)
        best = max(v for k, v in mb.items() if "warp_inst" in k)
        issue_meas = 148 * best * mhz * 1e6 / 1e9
        l_int = max(mb["mixed_lanes_per_clk_sm"], mb["alu_lanes_per_clk_sm"], mb["fma_lanes_per_clk_sm"])
        lane_meas = 148 * l_int * mhz * 1e6 / 1e9
        roof["issue_measured"] = {"peak": issue_meas, "frac": achieved / issue_meas,
                                  "warp_inst_per_clk_sm": {k.split("_warp")[0]: round(v, 3) for k, v in mb.items()
                                                           if "warp_inst" in k},
                                  "note": "peak = the best measured integer issue rate x 148 SM x clock"}
        roof["lane"] = {"L_int": l_int, "peak": lane_meas, "unit": "G int-lane-ops/s", "frac": achieved / lane_meas,
                        "note": "R_lane (SURVEY 8(d)) with L_int measured (integer lanes / clk / SM, microbenchmark)"}
    # HBM (BASELINE north_star asks for achieved GB/s): algorithmic bytes = descriptor in + record out
    # per scenario of the launch; ncu bytes = the committed capture's DRAM read + write
    alg_bytes = (B_DESC + B_REC) * count
    roof["hbm"] = {"algorithmic_bytes": alg_bytes, "achieved_gbs": alg_bytes / kern_s / 1e9,
                   "ncu_bytes": traffic, "ncu_gbs": (traffic / kern_s / 1e9) if traffic else None,
                   "peak_gbs": pk_["hbm_gbs"], "frac": alg_bytes / kern_s / 1e9 / pk_["hbm_gbs"]}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cols)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": config_dict(args.workload, n, world, args.seeds),
        "ticks_per_step": int(ticks_all),
        "exchange": ("none (1 GPU)" if world == 1 else "NCCL all-gather" if not fused else
                     "fused: records stored to every rank over peer memory by the tick kernel; "
                     "segment histograms NCCL all-reduce"),
        "roofline": roof,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches * args.steps,
        "engines": {"mask": engines, "dominant": "K2L lane-per-scenario" if lane_engine else "K2 warp-per-scenario"},
        "clocks": clocks,
        "kernel_ms_per_step": kern_tot / args.steps,
        "outputs": outs,
    }
    if lat is not None:
        line["latency_floor"] = lat
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

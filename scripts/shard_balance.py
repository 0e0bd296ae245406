"""Strong-scaling projection on one GPU: each rank's shard of BASELINE
configs[4] (C5, 2^20 scenarios; rank r of N runs ids r, r+N, ... heavy-first)
launched alone on the whole B200, timed with CUDA events.  At N GPUs the job
time is the slowest rank's shard, so  max_r t(r, N) x N / t(whole)  is the
projected strong-scaling inefficiency of the data path (the summary exchange
excluded; it overlaps inside the kernel).  Also reports id-order shards
(BELLMAN_AB_NOORDER build, if given) to show what heavy-first ordering buys.

  python scripts/shard_balance.py [lib_noorder.so]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2510_15330_b200 import _abi, sim  # noqa: E402


def times(pk, reps=3):
    s = sim.Simulator(packed=pk)
    n = s.n_scenarios
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def t(first, count, stride):
        best = None
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s.run(first=first, count=count, stride=stride)
            b.record()
            torch.cuda.synchronize()
            v = a.elapsed_time(b)
            best = v if best is None else min(best, v)
        return best

    out = {"whole_ms": t(0, n, 1)}
    for N in (2, 4, 8):
        per = [t(r, (n - r + N - 1) // N, N) for r in range(N)]
        out[f"N{N}"] = {"shard_ms": per, "max_ms": max(per),
                        "projected_efficiency": out["whole_ms"] / (N * max(per))}
    s.close()
    return out


def main():
    pk = sim.pack(W.config_c5().columns())
    res = {"heavy_first": times(pk)}
    if len(sys.argv) > 1:
        _abi._lib = None
        _abi.LIB_PATH = sys.argv[1]
        res["id_order"] = times(pk)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

"""Development check of K2L (the lane-per-scenario kernel) on the CPU.

Builds build/liblanecheck.so — bellman_host.cu + bellman_lane.cu with
-DBELLMAN_LANECHECK, whose entry runs K2L's per-scenario code (the same
__host__ __device__ functions the kernel runs) on the host — and compares its
records and segment histograms with the oracle, field by field.  Development
only: the product library never contains this entry, and no test, bench or
product path loads this library.

usage: python scripts/lanecheck.py [C1|C2|C3|C5|...] [stride] [max]
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_2510_15330_b200 import _abi as A  # noqa: E402
from paper_2510_15330_b200 import sim as S  # noqa: E402
from parity import compare  # noqa: E402

CSRC = os.path.join(ROOT, "paper_2510_15330_b200", "csrc")
OUT = os.path.join(ROOT, "build", "liblanecheck.so")


def build() -> str:
    srcs = [os.path.join(CSRC, f) for f in ("bellman_host.cu", "bellman_lane.cu", "bellman_kernels.cu")]
    deps = srcs + [os.path.join(CSRC, f) for f in ("bellman_internal.cuh", "bellman_lane.cuh")]
    if os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(s) for s in deps):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    # LANECHECK_FLAGS: extra -D flags (a K2L variant under test)
    extra = os.environ.get("LANECHECK_FLAGS", "").split()
    cmd = ["nvcc", "-DBELLMAN_LANECHECK", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-o", OUT] + extra + srcs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return OUT


def run(cols):
    lib = C.CDLL(build())
    lib.bellman_lanecheck.restype = C.c_int
    lib.bellman_lanecheck.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    pk = S.pack(cols)
    d = S.make_desc(pk)
    n = pk["n_scenarios"]
    out = np.zeros(n, dtype=A.STATS)
    seg = np.zeros(pk["n_segments"] * A.SEG_HIST_WORDS, dtype=np.uint64)
    ran = np.zeros(n, dtype=np.uint8)
    t = time.time()
    rc = lib.bellman_lanecheck(C.byref(d), out.ctypes.data, seg.ctypes.data, ran.ctypes.data)
    dt = time.time() - t
    if rc:
        raise RuntimeError(f"bellman_lanecheck rc={rc}")
    return out, seg.reshape(pk["n_segments"], A.SEG_HIST_WORDS), ran, dt


def check(cols, stride=1, limit=None, segs=False):
    out, seg, ran, dt = run(cols)
    n = len(cols["sc_seed"])
    sids = [s for s in range(0, n, stride) if ran[s]]
    if limit:
        sids = sids[:limit]
    rs = oracle.run_batch(oracle.Bound(cols), np.array(sids, dtype=np.uint64))
    bad = []
    for s, o in zip(sids, rs):
        e = compare(out[s], o, s)
        if e:
            bad.append((s, e))
    print(f"lane host run {dt:.1f}s; {int(ran.sum())}/{n} scenarios in K2L; compared {len(sids)}; bad {len(bad)}")
    for s, e in bad[:8]:
        print("  sid", s, e[:6])
    if segs and stride == 1 and not limit and ran.all():
        b = oracle.Bound(cols)
        want = np.zeros_like(seg, dtype=np.int64)
        for s in range(n):
            o = oracle.run_scenario(b, s)
            g = cols["sc_segment"][s]
            want[g, :896] += o["hist_e2e"]
            want[g, 896:1792] += o["hist_ttft"]
            want[g, 1792:2304] += o["hist_r"]
            want[g, 2304:2505] += o["hist_q_active"]
            want[g, 2505:2706] += o["hist_q_inactive"]
        print("segment histograms equal:", np.array_equal(seg.astype(np.int64), want))
    return bad


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    stride = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    limit = int(sys.argv[3]) if len(sys.argv) > 3 else None
    w = getattr(W, "config_" + name.lower())()
    bad = check(w.columns(), stride, limit, segs=True)
    sys.exit(1 if bad else 0)

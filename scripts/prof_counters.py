"""Development tool: build the tick kernel with BELLMAN_PROFILE_COUNTERS into a
separate library, run C2 once and print event-trip counters.  Never used by
the product path, the tests or the bench."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_15330_b200 import _abi, build as B  # noqa: E402

NAMES = ["trips", "mid_iteration_trips", "iter_end", "iter_end_with_completion", "prefill_end_event", "admit",
         "leap_calls", "leaped_ticks", "join_starts", "cyc_advance", "cyc_iteration_end", "cyc_prefill_end",
         "cyc_admit", "cyc_leap", "cyc_start_iteration", "cyc_event_loop", "lazy_prefill_batches", "quiet_join_ends", "cyc_admit_select", "cyc_admit_requests", "cyc_admit_reduce", "cyc_admit_head", "cyc_epilogue_queued", "cyc_epilogue_pct_merge"]


def main():
    out = os.path.join(ROOT, "build", "ab", "libbellman_sim_prof.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    if not os.environ.get("PROF_NO_BUILD"):  # PROF_NO_BUILD=1: use the library built beforehand
        cmd = [B.nvcc()] + [f for f in B.NVCC_FLAGS if f != "-v" and f != "-Xptxas"] + \
              ["-DBELLMAN_PROFILE_COUNTERS", "-o", out] + [os.path.join(B.CSRC, s) for s in B.SOURCES]
        subprocess.run(cmd, check=True)
    _abi.LIB_PATH = out
    import workloads as W
    from paper_2510_15330_b200 import Simulator

    cols = (eval(sys.argv[1], {"W": W}) if len(sys.argv) > 1 else W.config_c2()).columns()
    sim = Simulator(cols)
    sim.run()
    torch.cuda.synchronize()
    st = sim.stats()
    lib = _abi.lib()
    vals = np.zeros(24, dtype=np.uint64)
    assert lib.bellman_debug_prof(ctypes.c_void_p(vals.ctypes.data)) == 0
    print("ticks", int(st["ticks"].sum()), "admitted", int(st["admitted"].sum()), "served", int(st["served"].sum()))
    for n, v in zip(NAMES, vals):
        print(f"{n:26s} {int(v):12d}")
    ns = len(st)
    span = np.zeros(2 * ns, dtype=np.uint64)
    assert lib.bellman_debug_span(ctypes.c_void_p(span.ctypes.data), ctypes.c_uint(ns)) == 0
    t0 = span[0::2].astype(np.int64)
    t1 = span[1::2].astype(np.int64)
    base = t0.min()
    seg = st["segment"].astype(np.int64)
    tk = st["ticks"].astype(np.int64)
    print(f"kernel span {(t1.max() - base) / 1e3:.1f} us")
    print("segment  n   dur_mean_us dur_max_us start_max_us end_max_us  ticks_mean  ns/tick")
    for g in np.unique(seg):
        m = seg == g
        d = (t1[m] - t0[m]) / 1e3
        print(f"{g:5d} {m.sum():5d} {d.mean():11.1f} {d.max():10.1f} {(t0[m].max() - base) / 1e3:12.1f} "
              f"{(t1[m].max() - base) / 1e3:10.1f} {tk[m].mean():11.0f} {1e3 * d.mean() / max(tk[m].mean(), 1):8.1f}")


if __name__ == "__main__":
    main()

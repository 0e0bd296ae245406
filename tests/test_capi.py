"""The C-ABI library builds for sm_100a, loads on a GPU-less host, and exports
every entry point include/bellman_sim.h declares; the ctypes mirror matches the
header's struct sizes.  (No compute calls: there is no GPU here.)"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "bellman_sim.h")).read()
    return sorted(set(re.findall(r"\b(bellman_\w+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2510_15330_b200 import build as B

    path = B.build()
    lib = ctypes.CDLL(path)
    names = _declared()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n


def test_peak_library_exports_header_symbols():
    """The roofline microbenchmark (include/bellman_peak.h) builds and exports its entry point."""
    from paper_2510_15330_b200 import build as B

    B.build()
    lib = ctypes.CDLL(B.PEAK_OUT)
    src = open(os.path.join(ROOT, "include", "bellman_peak.h")).read()
    names = sorted(set(re.findall(r"\b(bellman_\w+)\s*\(", src)))
    assert names == ["bellman_peak_int"]
    for n in names:
        assert hasattr(lib, n), n


def test_struct_sizes_and_validation():
    from paper_2510_15330_b200 import _abi as A, sim
    import workloads as W

    A.lib()
    pk = sim.pack(W.config_c2(n_seeds=1, rates=[1.0]).columns())
    assert sim.workspace_bytes(pk) > 0
    bad = W.config_c2(n_seeds=1, rates=[1.0]).columns()
    bad["prof_maxb"] = bad["prof_maxb"].copy()
    bad["prof_maxb"][0] = 65          # S:185 max_batch in 1..64
    with pytest.raises(A.BellmanError, match="max_batch"):
        sim.workspace_bytes(sim.pack(bad))
    bad = W.config_c2(n_seeds=1, rates=[1.0]).columns()
    bad["ctrl_t2"] = bad["ctrl_t1"].copy()  # S:269 t1 < t2
    with pytest.raises(A.BellmanError, match="t1 < t2"):
        sim.workspace_bytes(sim.pack(bad))
    # the kernel's iteration counter is 32-bit: horizon / t0 must allow < 2^32 iterations
    bad = W.config_c2(n_seeds=1, rates=[1.0]).columns()
    bad["prof_t0"] = bad["prof_t0"].copy()
    bad["prof_t0"][:] = 1
    bad["sc_horizon"] = bad["sc_horizon"].copy()
    bad["sc_horizon"][:] = 1 << 32
    with pytest.raises(A.BellmanError, match="2\\^32 iterations"):
        sim.workspace_bytes(sim.pack(bad))
    bad["sc_horizon"][:] = (1 << 32) - 3  # ticks <= H / t0 + 1 < 2^32: accepted
    assert sim.workspace_bytes(sim.pack(bad)) > 0


def test_kv_policy_validation_and_scratch():
    """NEXT-4 preemption: unknown policies, preemption with contending prefill
    and recompute prefills that could outgrow the 32-bit event clock are
    rejected; a preempting profile adds the per-CTA scratch to the workspace."""
    from paper_2510_15330_b200 import _abi as A, sim
    import workloads as W

    def cols(**prof):
        c = W.config_c2(n_seeds=1, rates=[1.0]).columns()
        for k, v in prof.items():
            c[k] = c[k].copy()
            c[k][0] = v
        return c

    base = sim.workspace_bytes(sim.pack(cols(prof_kv_cap=50_000)))
    pre = sim.workspace_bytes(sim.pack(cols(prof_kv_cap=50_000, prof_kv_policy=1)))
    assert pre - base >= 4096 * 3584
    assert sim.workspace_bytes(sim.pack(cols(prof_kv_cap=0, prof_kv_policy=1))) == \
        sim.workspace_bytes(sim.pack(cols(prof_kv_cap=0)))  # no capacity: nothing to preempt
    with pytest.raises(A.BellmanError, match="unknown kv_policy"):
        sim.workspace_bytes(sim.pack(cols(prof_kv_policy=2)))
    with pytest.raises(A.BellmanError, match="needs prefill_mode 0"):
        sim.workspace_bytes(sim.pack(cols(prof_kv_cap=50_000, prof_kv_policy=1, prof_prefill_mode=1)))
    with pytest.raises(A.BellmanError, match="prefill of the capacity"):
        sim.workspace_bytes(sim.pack(cols(prof_kv_cap=2**28, prof_kv_policy=1)))


def test_sass_sm100a_warp_level_no_transcendentals():
    """Kernel built for sm_100a; the tick kernel's SASS uses warp vote/shuffle/
    reduce instructions (the warp-level design), and no kernel evaluates a
    transcendental (R33: no libm on the sampling path — -ln U and the quantile
    draws are integer tables): the only MUFU forms are the reciprocal seeds of
    integer / IEEE division (RCP, RCP64H), never EX2 / LG2 / SIN / COS / SQRT / RSQ.
    (Floating point that does appear: the energy epilogue's IEEE fp64 ops and
    the quality decay's and K2L's MAP-law quotient's fp32 estimates with an
    exact integer fix-up.)"""
    import re as _re
    import subprocess

    from paper_2510_15330_b200 import build as B

    path = B.build()
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper() or "arch = sm_100a" in out
    for mnemonic in ("VOTE", "SHFL", "REDUX"):
        assert mnemonic in out, mnemonic
    mufu = set(_re.findall(r"MUFU\.(\w+)", out))
    assert mufu <= {"RCP", "RCP64H"}, mufu


def test_next3_law_validation():
    """NEXT-3 laws: BBR needs the TBT signal, PCC a delta and no rungs, MPC a
    bounded horizon and w_lat >= 1; weights <= 65535; no calibration."""
    from paper_2510_15330_b200 import _abi as A, sim
    import workloads as W

    def cols(c):
        w = W.config_c2(n_seeds=1, rates=[1.0])
        w.ctrls = [c] + w.ctrls[1:]
        return w.columns()

    assert sim.workspace_bytes(sim.pack(cols(W.mpc_ctrl(24_000)))) > 0
    assert sim.workspace_bytes(sim.pack(cols(W.bbr_ctrl(3_000)))) > 0
    assert sim.workspace_bytes(sim.pack(cols(W.pcc_ctrl(24_000)))) > 0
    bad = [
        (W.bbr_ctrl(3_000).__class__(**{**W.bbr_ctrl(3_000).__dict__, "signal": W.SIG_E2E}), "BBR needs the TBT"),
        (W.Ctrl(**{**W.pcc_ctrl(24_000).__dict__, "step_bp": 0}), "PCC needs 1 <= step_bp"),
        (W.Ctrl(**{**W.pcc_ctrl(24_000).__dict__, "rungs_bp": (500, 2000)}), "PCC takes no rungs"),
        (W.mpc_ctrl(24_000, horizon_s=17), "horizon_s > 16"),
        (W.mpc_ctrl(24_000, w_lat=0), "MPC needs w_lat"),
        (W.mpc_ctrl(24_000, w_q=70000), "weights must be <= 65535"),
        (W.Ctrl(**{**W.mpc_ctrl(24_000).__dict__, "calibrated": 1}), "calibration is for MAP"),
        (W.Ctrl(**{**W.bbr_ctrl(3_000).__dict__, "step_bp": 0}), "BBR needs 1 <= step_bp"),
        (W.Ctrl(**{**W.mpc_ctrl(24_000).__dict__, "law": 7}), "unknown law"),
    ]
    for c, msg in bad:
        with pytest.raises(A.BellmanError, match=msg):
            sim.workspace_bytes(sim.pack(cols(c)))


def test_replica_validation():
    """NEXT-4 multi-replica profiles: <= 8 replicas, replicas x max_batch <= 64,
    known route, non-blocking prefill and no KV capacity."""
    from paper_2510_15330_b200 import _abi as A, sim
    import workloads as W

    def cols(**prof):
        c = W.config_c2(n_seeds=1, rates=[1.0]).columns()
        for k, v in prof.items():
            c[k] = c[k].copy()
            c[k][0] = v
        return c

    assert sim.workspace_bytes(sim.pack(cols(prof_replicas=8, prof_maxb=8, prof_knee=1))) > 0
    for kw, msg in ((dict(prof_replicas=9, prof_maxb=4, prof_knee=1), "replicas > 8"),
                    (dict(prof_replicas=2, prof_maxb=33, prof_knee=1), "replicas x max_batch > 64"),
                    (dict(prof_replicas=2, prof_maxb=8, prof_knee=1, prof_route=2), "unknown route"),
                    (dict(prof_replicas=2, prof_maxb=8, prof_knee=1, prof_prefill_mode=1), "needs prefill_mode 0"),
                    (dict(prof_replicas=2, prof_maxb=8, prof_knee=1, prof_kv_cap=10_000), "needs prefill_mode 0")):
        with pytest.raises(A.BellmanError, match=msg):
            sim.workspace_bytes(sim.pack(cols(**kw)))


def test_lane_engine_workspace_and_sass(monkeypatch):
    """K2L (the lane-per-scenario kernel): a descriptor with >= 65,536
    scenarios in its bounds gets the per-thread histogram and FIFO regions in
    its workspace, unless BELLMAN_LANE=0; BELLMAN_LANE=2 adds them to small
    sets too.  Both K2L instantiations are in the library, built for sm_100a
    with no local-memory spills."""
    import workloads as W
    from paper_2510_15330_b200 import build as B
    from paper_2510_15330_b200 import sim

    path = B.build()
    lane_bytes = 40960 * (2760 * 4 + 96 * 8)  # kLaneMaxThreads x (histograms + FIFO)
    big = sim.pack(W.config_c5(n_seeds=256).columns())  # 65,536 scenarios
    small = sim.pack(W.config_c2(n_seeds=1).columns())
    monkeypatch.delenv("BELLMAN_LANE", raising=False)
    auto_big, auto_small = sim.workspace_bytes(big), sim.workspace_bytes(small)
    monkeypatch.setenv("BELLMAN_LANE", "0")
    off_big, off_small = sim.workspace_bytes(big), sim.workspace_bytes(small)
    monkeypatch.setenv("BELLMAN_LANE", "2")
    on_small = sim.workspace_bytes(small)
    assert auto_big - off_big >= lane_bytes
    assert auto_small == off_small and on_small - off_small >= lane_bytes
    info = open(os.path.join(os.path.dirname(path), "ptxas_info.txt")).read()
    blocks = info.split("Compiling entry function")
    lane = [b for b in blocks if "bellman_lane_kernel" in b.split("\n")[0]]
    assert len(lane) == 2, "two K2L instantiations (kv = 0, kv > 0)"
    for b in lane:
        assert "sm_100a" in b.split("\n")[0]
        assert "0 bytes spill stores, 0 bytes spill loads" in b


def test_parallel_validation_names_the_lowest_bad_scenario():
    """Per-scenario validation runs on host threads in chunks (bellman_host.cu
    parallel_chunks): with invalid scenarios in several chunks the message must
    still name the lowest one, as a sequential pass would, and workspace
    sizing must be a pure function of the descriptor."""
    import numpy as np

    from paper_2510_15330_b200 import _abi as A, sim
    import workloads as W

    cols = W.config_c5(n_seeds=256).columns()  # 65,536 scenarios: chunked on any multi-core host
    n = len(cols["sc_seed"])
    pk = sim.pack(cols)
    a, b = sim.workspace_bytes(pk), sim.workspace_bytes(sim.pack(cols))
    assert a == b > 0
    bad = dict(cols)
    bad["sc_w0"] = np.asarray(cols["sc_w0"]).copy()
    bad["sc_w1"] = np.asarray(cols["sc_w1"]).copy()
    for s in (n - 5, n // 2 + 7, 40_000, 12_345):  # w0 > w1 in four different chunks
        bad["sc_w0"][s], bad["sc_w1"][s] = 10, 5
    with pytest.raises(A.BellmanError, match="scenario 12345: w0 > w1"):
        sim.workspace_bytes(sim.pack(bad))

"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): bit-exact for every integer field (ticks,
arrivals, words, served, latencies sums, percentiles, controller logs, flags)
and for the E2E / TTFT / r histograms; fp64 energy within 1e-9 relative.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from tests.parity import check_all, compare, run_gpu

pytestmark = pytest.mark.gpu


def _assert_ok(bad):
    assert not bad, "\n".join(f"scenario {sid}: {e}" for sid, e in bad[:10])


def test_c1_full():
    bad, st = check_all(W.config_c1().columns())
    _assert_ok(bad)
    assert st[1]["activations"] >= 1 and st[1]["rewritten"] > 0


def test_c2_reduced_all_rates():
    bad, _ = check_all(W.config_c2(n_seeds=2).columns())
    _assert_ok(bad)


def test_c3_reduced_controller_grid():
    bad, _ = check_all(W.config_c3(n_seeds=1).columns())
    _assert_ok(bad)


def test_c4_reduced_diurnal():
    bad, _ = check_all(W.config_c4(n_seeds=2, n_traces=2, days=0.25).columns())
    _assert_ok(bad)


def test_c5_reduced_variants():
    bad, _ = check_all(W.config_c5(n_seeds=1).columns())
    _assert_ok(bad)


def _edge_workload():
    """Degenerate and ragged cases: empty traces, ragged max_batch around the
    32-lane boundary, knee 0, heavy KV term, 1-µs prefill, realized length 1,
    queue far beyond one 32-entry buffer, arrival caps around 32, E2E/SLO
    signals, every law, every window, a degenerate calibration, odd windows."""
    tabs = W.quantile_tables()
    traces = [
        W.const_trace(0.0, 100),                                     # 0: no arrivals
        W.const_trace(2.5, 300),                                     # 1
        W.const_trace(30.0, 120),                                    # 2: deep queue
        [(0, 0), (50 * W.US, 4000), (50 * W.US, 500), (80 * W.US, 0), (200 * W.US, 1500)],  # 3: ramps + jump
        (W.const_trace(5.0, 200), 31), (W.const_trace(5.0, 200), 32), (W.const_trace(5.0, 200), 33),  # 4-6: caps
        (W.const_trace(5.0, 200), 1),                                # 7: single request
        W.paper_trace(3.5, 180, 0.6),                                # 8
    ]
    profs = [
        W.PROFILES["P24"], W.PROFILES["L8B"], W.PROFILES["spec-literal"],
        dict(W.PROFILES["P24"], max_batch=1, knee=0), dict(W.PROFILES["P24"], max_batch=31, knee=0),
        dict(W.PROFILES["P24"], max_batch=32, knee=32), dict(W.PROFILES["P24"], max_batch=33, knee=7),
        dict(W.PROFILES["L8B"], max_batch=63, kv_ns_per_word=900),
        dict(W.PROFILES["P24"], prefill_ns_per_word=0, t0_us=1, slope_us=0),  # 1 µs prefills, 1 µs iterations
        dict(W.PROFILES["P24"], replicas=8, max_batch=8, route=0),         # round 2: all 64 slots in replicas
        dict(W.PROFILES["L8B"], replicas=7, max_batch=9, knee=3, route=1),  # 63 slots, ragged
        dict(W.PROFILES["P24"], replicas=2, max_batch=1, knee=0, prefill_ns_per_word=0, t0_us=1, slope_us=0),
    ]
    ctrls = [
        W.OFF,
        W.map_ctrl(30_000, 45_000),
        W.map_ctrl(20_000, 60_000, rungs=(300, 700, 1900)),
        W.step_ctrl(25_000, 40_000, (500, 1000, 1500, 2000)),
        W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 1200),
        W.map_ctrl(5_000_000, 20_000_000, signal=W.SIG_E2E, window=3),
        W.map_ctrl(200, 900, signal=W.SIG_SLO, slo_us=20_000_000, window=1),
        W.map_ctrl(30_000, 31_000, window=8, r_min_bp=1, r_max_bp=5000),
        W.Ctrl(W.LAW_MAP, W.SIG_TBT, 5, 500, 2000, 0, 0, 0, 0, 1, ()),  # calibrated
    ]
    sc = []
    sid = 0
    rng = np.random.default_rng(42)
    for ti in range(len(traces)):
        for pi in range(len(profs)):
            ci = int(rng.integers(0, len(ctrls) - 1))
            mode = int(rng.integers(0, 2))
            H = int(rng.choice([1, 60 * W.US, 700 * W.US, 2000 * W.US]))
            w0 = int(rng.integers(0, 200)) * W.US
            sc.append(W.Scenario(int(rng.integers(0, 1000)), wid=ti, trace=ti, profile=pi, ctrl=ci, segment=0,
                                 mode=mode, horizon_us=H, w0_us=w0, w1_us=w0 + int(rng.integers(0, 300)) * W.US))
            sid += 1
    # calibrated pairs: one healthy (paper trace), one degenerate (empty trace)
    for ti in (8, 0, 7):
        src = len(sc)
        sc.append(W.Scenario(3, wid=ti, trace=ti, profile=0, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                             horizon_us=2000 * W.US, record=1))
        sc.append(W.Scenario(3, wid=ti, trace=ti, profile=0, ctrl=8, segment=0, mode=W.MODE_DRAIN,
                             horizon_us=2000 * W.US, calib_src=src))
    return W.custom(traces, profs, ctrls, sc, tables=tabs)


def test_edge_cases():
    w = _edge_workload()
    bad, st = check_all(w.columns())
    _assert_ok(bad)
    assert any(int(r["flags"]) & 2 for r in st)  # a degenerate calibration occurred


def test_short_outputs_and_tiny_tables():
    """Realized length 1 and 2 dominate (R9), compliance noise maximal."""
    t = W.quantile_tables(L_mean=2.0, L_sd=1.5, L_lo=1, L_hi=6, in_median=50, in_lo=1, in_hi=200,
                          pred_b=2.0, comp_rel_noise=0.4)
    scs = [W.Scenario(s, wid=0, trace=0, profile=p, ctrl=c, segment=0, mode=s % 2, horizon_us=40 * W.US)
           for s in range(6) for p in range(2) for c in range(3)]
    w = W.custom([W.const_trace(40.0, 30)],
                 [dict(W.PROFILES["P24"], prefill_ns_per_word=3000, max_batch=5, knee=2),
                  dict(W.PROFILES["spec-literal"], t0_us=900, prefill_ns_per_word=1000)],
                 [W.OFF, W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 3000), W.map_ctrl(1_000, 9_000, window=2)],
                 scs, tables=t, poly_q16=(3 * 65536, 50000, 20))
    bad, _ = check_all(w.columns())
    _assert_ok(bad)


def test_sharded_runs_match_single_run():
    """Interleaved shards (first = rank, stride = world) write the same records
    as one run over all scenarios (determinism contract)."""
    cols = W.config_c2(n_seeds=2, rates=[1.0, 3.0, 6.0]).columns()
    full, _, _ = run_gpu(cols)
    for world in (2, 3):
        import torch

        from paper_2510_15330_b200 import Simulator

        sim = Simulator(cols)
        n = len(cols["sc_seed"])
        for rank in range(world):
            sim.run(first=rank, count=len(range(rank, n, world)), stride=world)
        torch.cuda.synchronize()
        st = sim.stats()
        assert np.array_equal(st.view(np.uint8), full.view(np.uint8))


def _full_size_sampled(w, stride, sim=None):
    """A BASELINE config at full size in bench.py's launch configuration (one
    whole-set launch, heavy-first order): the records with id % stride == 0
    (SURVEY §8(d)'s deterministic stride subsample) vs the oracle, and on every
    record the properties that hold at any size — written, arrivals = admitted
    + queued, admitted = served + in flight, a drained run leaves nothing
    behind, energy is the fp64 formula of the record's own integers (R19)."""
    import torch

    from paper_2510_15330_b200 import Simulator

    cols = w.columns()
    sim = sim or Simulator(cols)
    sim.run()
    torch.cuda.synchronize()
    st = sim.stats()
    assert sim.last_launches == 1
    n = w.n_scenarios
    sids = np.arange(0, n, stride, dtype=np.uint64)
    rs = oracle.run_batch(oracle.Bound(cols), sids)
    bad = [(int(s), e) for s, o in zip(sids, rs) for e in [compare(st[int(s)], o, int(s))] if e]
    _assert_ok(bad)
    _invariants(st, cols, n)
    return st


def _invariants(st, cols, n, ids=None):
    ids = np.arange(n) if ids is None else ids
    assert np.all(st["flags"] & 0x100)
    assert np.array_equal(st["scenario_id"], ids)
    assert np.array_equal(st["arrivals"], st["admitted"] + st["queued_end"])
    assert np.array_equal(st["admitted"], st["served"] + st["inflight_end"])
    drained = (st["flags"] & 1) == 0
    assert np.all(st["queued_end"][drained] == 0) and np.all(st["inflight_end"][drained] == 0)
    prof = cols["prof_e_in"][0], cols["prof_e_out"][0], cols["prof_p_idle"][0]
    assert np.all(cols["prof_e_in"] == prof[0]) and np.all(cols["prof_e_out"] == prof[1])
    e = (prof[0] * st["words_in"].astype(np.float64) + prof[1] * st["words_out"].astype(np.float64)) + \
        prof[2] * st["idle_us"].astype(np.float64) / 1e6
    assert np.array_equal(e, st["energy_j"])


def test_c5_full_size_stride64_and_strong_scaled_shard():
    """BASELINE configs[4] (2^20 scenarios) in bench.py's N = 1 launch
    configuration: the 16,384 records with id % 64 == 0 vs the oracle
    (SURVEY §8(d)), invariants on all 2^20.  Then one rank's shard of the
    strong-scaled 8-GPU run (first = 5, stride = 8, 131,072 scenarios, in the
    shard's own heavy-first order): every record byte-equal to the whole-set
    run's, and the 16,384 with id % 64 == 5 vs the oracle."""
    import torch

    from paper_2510_15330_b200 import Simulator

    w = W.config_c5()
    cols = w.columns()
    sim = Simulator(cols)
    st = _full_size_sampled(w, 64, sim)
    assert int(st["ticks"].sum()) > 5e10
    sim.reset()
    sim.run(first=5, count=(w.n_scenarios - 5 + 7) // 8, stride=8)
    torch.cuda.synchronize()
    sh = sim.stats_shard(5, 8)
    assert len(sh) == 131072
    assert np.array_equal(sh.view(np.uint8), np.ascontiguousarray(st[5::8]).view(np.uint8))
    sids = np.arange(5, w.n_scenarios, 64, dtype=np.uint64)
    rs = oracle.run_batch(oracle.Bound(cols), sids)
    bad = [(int(s), e) for s, o in zip(sids, rs) for e in [compare(sh[(int(s) - 5) // 8], o, int(s))] if e]
    _assert_ok(bad)
    untouched = sim.stats(first=0, count=5)  # ids outside the shard stay zero after reset
    assert not untouched.view(np.uint8).any()


def test_c4_full_size_every_record():
    """BASELINE configs[3]: 24 h diurnal traces with bursts, 4096 scenarios,
    every record vs the oracle."""
    st = _full_size_sampled(W.config_c4(), 1)
    assert int(st["ticks"].max()) > 10**6


def test_c3_full_size_every_record():
    """BASELINE configs[2] at full size (321 controllers x 32 seeds = 10,272
    scenarios, one launch): every record vs the oracle."""
    st = _full_size_sampled(W.config_c3(), 1)
    assert len(st) == 10272


def test_c2_full_bench_config():
    """BASELINE configs[1] at full size, in the launch configuration bench.py
    times: every one of the 2048 records vs the oracle, and the per-segment
    histograms vs the sum of the oracle's per-scenario histograms."""
    w = W.config_c2()
    cols = w.columns()
    import torch

    from paper_2510_15330_b200 import Simulator

    sim = Simulator(cols)
    sim.run()
    torch.cuda.synchronize()
    st = sim.stats()
    seg = sim.segment_hist()
    b = oracle.Bound(cols)
    want_seg = np.zeros_like(seg, dtype=np.int64)
    bad = []
    for sid in range(w.n_scenarios):
        o = oracle.run_scenario(b, sid)
        e = compare(st[sid], o, sid)
        if e:
            bad.append((sid, e))
        s = w.scenarios[sid].segment
        want_seg[s, :896] += o["hist_e2e"]
        want_seg[s, 896:1792] += o["hist_ttft"]
        want_seg[s, 1792:2304] += o["hist_r"]
        want_seg[s, 2304:2505] += o["hist_q_active"]
        want_seg[s, 2505:2706] += o["hist_q_inactive"]
    _assert_ok(bad)
    assert np.array_equal(seg.astype(np.int64), want_seg)
    assert sim.last_launches == 1


def test_debug_series_rows_and_controller_log():
    """NEXT-1 debug record mode: per-second rows (attribution S:382) and
    the controller log equal the oracle's element by element."""
    import torch

    from paper_2510_15330_b200 import Simulator

    ws = [W.config_c1(), W.config_c3(n_seeds=1), W.config_c2(n_seeds=1, rates=[0.5, 2.5, 6.0]), _preempt_workload()]
    for w in ws:
        sel = list(range(0, w.n_scenarios, max(1, w.n_scenarios // 12)))
        for sid in sel:
            w.scenarios[sid].record |= 2
        cols = w.columns()
        sim = Simulator(cols)
        sim.run()
        torch.cuda.synchronize()
        st = sim.stats()
        b = oracle.Bound(cols)
        for sid in sel:
            o = oracle.run_scenario(b, sid, rows_cap=100000, ctrl_log_cap=100000)
            assert not compare(st[sid], o, sid), (w.name, sid)
            rows, ctrl = sim.series(sid)
            orow = o["rows"]
            assert len(rows) == len(orow), (w.name, sid, len(rows), len(orow))
            for f in orow.dtype.names:
                assert np.array_equal(rows[f].astype(np.int64), orow[f].astype(np.int64)), (w.name, sid, f)
            oc = o["ctrl_log"]
            assert len(ctrl) == len(oc), (w.name, sid)
            for g, e in zip(ctrl, oc):
                assert (int(g["second"]), int(g["sample"]), int(g["k"]), int(g["r_bp"]), int(g["active"]),
                        int(g["A"])) == (e["second"], e["sample"], e["k"], e["r_bp"], e["active"], e["A"])


def test_next3_classes_bypass_and_ttft_signal():
    """NEXT-3: a request-class mix with per-class bypass and short-output bypass
     under MAP/STEP/CONST laws, and the TTFT signal."""
    import dataclasses

    w = W.config_c3(n_seeds=2)
    w.class_cum = W.MIXED_CLASSES
    w.ctrls = [dataclasses.replace(c, bypass_mask=(i % 3) * 2, min_words_bypass=(0, 420, 480)[i % 3])
               if c.law != W.LAW_OFF else c for i, c in enumerate(w.ctrls)]
    w.ctrls.append(W.map_ctrl(400_000, 900_000, signal=W.SIG_TTFT))
    w.ctrls.append(W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 1500, bypass_mask=0b0110, min_words_bypass=450))
    for k in (len(w.ctrls) - 2, len(w.ctrls) - 1):
        for s in range(3):
            w.scenarios.append(W.Scenario(s, wid=0, trace=0, profile=0, ctrl=k, segment=0, mode=W.MODE_DRAIN,
                                          horizon_us=1920 * W.US))
    w.scenarios = w.scenarios[::7] + w.scenarios[-6:]
    bad, st = check_all(w.columns())
    _assert_ok(bad)
    assert int(st["bypassed"].sum()) > 0


def test_next4_kv_capacity_admission():
    """NEXT-4 KV-capacity admission (FIFO, oversized requests alone) across
    capacities, controllers (rewrite changes the admitted context), bypass and
    drain/cutoff modes."""
    import dataclasses

    w = W.config_c3(n_seeds=1)
    w.class_cum = W.MIXED_CLASSES
    caps = [0, 40_000, 150_000, 300_000, 700_000]
    w.profiles = [dict(W.PROFILES["P24"], kv_cap_words=c) for c in caps] + [dict(W.PROFILES["L8B"], kv_cap_words=90_000)]
    w.ctrls[5] = dataclasses.replace(w.ctrls[5], bypass_mask=2, min_words_bypass=470)
    sc = []
    for i, s in enumerate(w.scenarios[::5]):
        sc.append(dataclasses.replace(s, profile=i % len(w.profiles), mode=i % 2,
                                      horizon_us=(1920 if i % 2 else 700) * W.US))
    w.scenarios = sc
    bad, st = check_all(w.columns())
    _assert_ok(bad)


def _preempt_workload():
    """NEXT-4 KV preemption (kv_policy 1): paper-trace scenarios under several
    capacities, with and without the KV cost term, every law (the rewrite
    decides R, kept across re-admissions), TBT / E2E / INPUT signals, class
    bypass, drain and cutoff, next to reserve-policy and uncapped profiles."""
    import dataclasses

    w = W.config_c3(n_seeds=1)
    w.class_cum = W.MIXED_CLASSES
    pre = dict(kv_policy=1)
    w.profiles = [dict(W.PROFILES["P24"], kv_cap_words=c, **pre) for c in (60_000, 150_000, 300_000)] + \
                 [dict(W.PROFILES["L8B"], kv_cap_words=120_000, **pre), dict(W.PROFILES["P24"], kv_cap_words=150_000),
                  W.PROFILES["P24"], dict(W.PROFILES["L8B"], kv_cap_words=9_000, **pre)]
    w.ctrls[5] = dataclasses.replace(w.ctrls[5], bypass_mask=2, min_words_bypass=470)
    w.ctrls[7] = dataclasses.replace(w.ctrls[7], signal=W.SIG_E2E, t1=8_000_000, t2=40_000_000)
    w.ctrls[9] = dataclasses.replace(w.ctrls[9], signal=W.SIG_INPUT, t1=20_000, t2=60_000)
    sc = []
    for i, s in enumerate(w.scenarios[::5]):
        sc.append(dataclasses.replace(s, profile=i % len(w.profiles), mode=i % 2,
                                      horizon_us=(1920 if i % 2 else 700) * W.US))
    w.scenarios = sc
    return w


def test_next4_kv_preemption():
    bad, st = check_all(_preempt_workload().columns())
    _assert_ok(bad)
    assert int(st["preemptions"].sum()) > 100 and int(st["recompute_words"].sum()) > 0


def test_next4_trace_replay():
    """NEXT-4 replay of explicit arrival lists: lists longer than one
    32-entry refill, arrival caps, simultaneous arrivals, classes, with KV
    capacity and the controller, next to Poisson traces in the same run."""
    rng = np.random.default_rng(77)
    reps = []
    for t in range(3):
        n = int(rng.integers(40, 900))
        gaps = rng.exponential(1e6 / (1.0 + 2 * t), n).astype(np.int64)
        gaps[rng.random(n) < 0.1] = 0  # simultaneous arrivals
        a = np.cumsum(gaps)
        reps.append([(int(a[k]), int(rng.integers(1, 1300)), int(rng.integers(1, 20000)), int(rng.integers(0, 4)))
                     for k in range(n)])
    traces = [{"replay": reps[0]}, {"replay": reps[1], "cap": 33}, {"replay": reps[2]}, W.paper_trace()]
    profs = [W.PROFILES["P24"], dict(W.PROFILES["L8B"], kv_cap_words=200_000)]
    ctrls = [W.OFF, W.map_ctrl(21_000, 26_000), W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 900, bypass_mask=2)]
    sc = [W.Scenario(s, wid=t, trace=t, profile=pi, ctrl=ci, segment=0, mode=s % 2, horizon_us=2000 * W.US)
          for t in range(4) for pi in range(2) for ci in range(3) for s in range(2)]
    w = W.custom(traces, profs, ctrls, sc)
    w.class_cum = W.MIXED_CLASSES
    bad, _ = check_all(w.columns())
    _assert_ok(bad)


def _long_workload():
    """The event loop keeps instants as 32-bit offsets from an epoch that moves
    every 2^30 µs: idle gaps longer than 2^32 µs, horizons far
    beyond the window, overload queues whose head arrived before the current
    epoch, seconds / windows / debug rows across rebase points."""
    US = W.US
    gap_trace = [(0, 5000), (60 * US, 5000), (60 * US, 0), (10_860 * US, 0), (10_860 * US, 3000),
                 (10_980 * US, 3000)]  # 3 h silence (> 2^32 µs) between two bursts
    sparse = W.const_trace(0.02, 18_000)  # ~360 arrivals over 5 h: idle rebases
    overload = W.const_trace(8.0, 1500)  # queue far deeper than one epoch can drain
    rep = [(0, 500, 9000, 0), (3 * US, 800, 4000, 1), (3 * US + (1 << 33), 600, 9000, 2),
           (4 * US + (1 << 33), 700, 12000, 0)]  # 2^33 µs between arrivals
    traces = [gap_trace, sparse, overload, {"replay": rep}]
    profs = [W.PROFILES["P24"], W.PROFILES["L8B"], dict(W.PROFILES["L8B"], kv_cap_words=300_000),
             dict(W.PROFILES["P24"], replicas=3, max_batch=8, route=1)]  # round 2: replica ends across rebases
    ctrls = [W.OFF, W.map_ctrl(30_000, 60_000), W.map_ctrl(5_000_000, 900_000_000, signal=W.SIG_E2E, window=3),
             W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 1500)]
    sc = []
    for t in range(4):
        for pi in range(4):
            for ci in range(4):
                for H, mode in ((11_000 * US, W.MODE_CUTOFF), (20_000 * US, W.MODE_DRAIN), (1 << 40, t % 2)):
                    rec = 2 if (H == 11_000 * US and ci == 1 and pi == 0) else 0
                    sc.append(W.Scenario(t * 7 + ci, wid=t, trace=t, profile=pi, ctrl=ci, segment=0, mode=mode,
                                         horizon_us=H, w0_us=1_000 * US, w1_us=9_000 * US, record=rec))
    return W.custom(traces, profs, ctrls, sc)


def test_long_horizons_far_gaps_and_epoch_rebases():
    bad, st = check_all(_long_workload().columns())
    _assert_ok(bad)
    assert int(st["end_us"].max()) > (1 << 32)


@pytest.mark.parametrize("poly", [(-(1 << 20), 70_000, 3),  # int64 path (|poly| bound < 2^43)
                                  (0, 32_768, 512),          # 128-bit path (bound >= 2^43)
                                  (5 << 16, -(1 << 14), 1 << 8)])
def test_rewrite_polynomial_paths(poly):
    """a7 rewrite (R11) through both device paths: the int64 one the
    host enables for small coefficients and the 128-bit general one."""
    ctrls = [W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 1300), W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 4900),
             W.map_ctrl(20_000, 30_000)]
    sc = [W.Scenario(s, wid=0, trace=0, profile=p, ctrl=c, segment=0, mode=W.MODE_DRAIN, horizon_us=200 * W.US)
          for s in range(4) for p in range(2) for c in range(3)]
    w = W.custom([W.const_trace(4.0, 150)], [W.PROFILES["P24"], W.PROFILES["L8B"]], ctrls, sc, poly_q16=poly)
    bad, st = check_all(w.columns())
    _assert_ok(bad)
    assert int(st["rewritten"].sum()) > 0


def test_next3_input_and_util_signals():
    """NEXT-3 signals P:211 names: input words admitted per second (INPUT) and
    decode-batch occupancy (UTIL), under MAP and STEP laws, with thresholds
    calibrated from an OFF run recording the same signal, and in debug record
    mode (controller log and rows compared element by element)."""
    US = W.US
    traces = [W.paper_trace(), W.const_trace(3.0, 400), W.const_trace(6.0, 300)]
    profs = [W.PROFILES["P24"], W.PROFILES["L8B"], dict(W.PROFILES["P24"], max_batch=13, knee=4)]
    ctrls = [W.OFF,
             W.map_ctrl(15_000, 30_000, signal=W.SIG_INPUT),
             W.map_ctrl(3_000, 7_000, signal=W.SIG_UTIL, window=3),
             W.step_ctrl(4_000, 9_000, (500, 1000, 1500, 2000), signal=W.SIG_UTIL),
             W.step_ctrl(20_000, 40_000, (300, 900, 2000), signal=W.SIG_INPUT),
             W.Ctrl(W.LAW_MAP, W.SIG_INPUT, 5, 500, 2000, 0, 0, 0, 0, 1, ()),   # calibrated
             W.Ctrl(W.LAW_MAP, W.SIG_UTIL, 5, 500, 2000, 0, 0, 0, 0, 1, ()),    # calibrated
             W.Ctrl(W.LAW_OFF, W.SIG_INPUT, 5, 500, 2000, 0, 0, 0, 0, 0, ()),   # OFF sources
             W.Ctrl(W.LAW_OFF, W.SIG_UTIL, 5, 500, 2000, 0, 0, 0, 0, 0, ())]
    sc = []
    for t in range(3):
        for pi in range(3):
            for ci in range(1, 5):
                for s in range(2):
                    rec = 2 if (s == 0 and pi == 0) else 0
                    sc.append(W.Scenario(s, wid=t, trace=t, profile=pi, ctrl=ci, segment=0, mode=s % 2,
                                         horizon_us=1400 * US, record=rec))
            for src_ctrl, cal_ctrl in ((7, 5), (8, 6)):
                src = len(sc)
                sc.append(W.Scenario(4, wid=t, trace=t, profile=pi, ctrl=src_ctrl, segment=0,
                                     mode=W.MODE_DRAIN, horizon_us=1400 * US, record=1))
                sc.append(W.Scenario(4, wid=t, trace=t, profile=pi, ctrl=cal_ctrl, segment=0,
                                     mode=W.MODE_DRAIN, horizon_us=1400 * US, calib_src=src))
    w = W.custom(traces, profs, ctrls, sc)
    bad, st = check_all(w.columns())
    _assert_ok(bad)
    assert int(st["activations"].sum()) > 0 and int(st["rewritten"].sum()) > 0
    # debug-recorded scenarios: rows and controller logs equal the oracle's
    import oracle
    from paper_2510_15330_b200 import Simulator

    cols = w.columns()
    sim = Simulator(cols, device=0)
    sim.run()
    b = oracle.Bound(cols)
    for sid in [i for i, x in enumerate(sc) if x.record & 2]:
        rows, ctrl = sim.series(sid)
        o = oracle.run_scenario(b, sid, rows_cap=len(rows) + 8, ctrl_log_cap=len(ctrl) + 8)
        assert [int(c["sample"]) for c in ctrl] == [e["sample"] for e in o["ctrl_log"]], sid
    sim.close()


def test_next4_contending_prefill():
    """NEXT-4 prefill/decode contention: profiles with prefill_mode = 1
    next to non-blocking ones, under every law and several signals, with KV
    capacity, replay and Poisson traces, ragged max_batch, 1 µs prefills,
    calibrated pairs and debug rows."""
    US = W.US
    rng = np.random.default_rng(3)
    rep = sorted((int(t), int(rng.integers(50, 900)), int(rng.integers(100, 15000)), int(rng.integers(0, 4)))
                 for t in rng.integers(0, 600 * US, 700))
    traces = [W.paper_trace(), W.const_trace(1.2, 500), W.const_trace(4.0, 300), {"replay": rep}]
    C = dict(prefill_mode=1)
    profs = [dict(W.PROFILES["P24"], **C), dict(W.PROFILES["L8B"], **C), dict(W.PROFILES["spec-literal"], **C),
             dict(W.PROFILES["P24"], max_batch=33, knee=5, **C), dict(W.PROFILES["P24"], max_batch=1, knee=0, **C),
             dict(W.PROFILES["L8B"], kv_cap_words=250_000, **C), dict(W.PROFILES["P24"], prefill_ns_per_word=0, **C),
             W.PROFILES["P24"]]
    ctrls = [W.OFF, W.map_ctrl(25_000, 60_000), W.step_ctrl(30_000, 70_000, (500, 1000, 1500, 2000)),
             W.Ctrl(W.LAW_CONST, W.SIG_TBT, 5, 500, 2000, 1200), W.map_ctrl(2_000_000, 9_000_000, signal=W.SIG_TTFT),
             W.map_ctrl(3_000, 8_000, signal=W.SIG_UTIL), W.Ctrl(W.LAW_MAP, W.SIG_TBT, 5, 500, 2000, 0, 0, 0, 0, 1, ())]
    sc = []
    for t in range(4):
        for pi in range(len(profs)):
            for ci in range(6):
                rec = 2 if (ci == 1 and pi in (0, 1) and t == 0) else 0
                sc.append(W.Scenario(ci, wid=t, trace=t, profile=pi, ctrl=ci, segment=0, mode=(t + ci) % 2,
                                     horizon_us=1400 * US, w0_us=130 * US, w1_us=500 * US, record=rec))
            src = len(sc)
            sc.append(W.Scenario(9, wid=t, trace=t, profile=pi, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                                 horizon_us=1400 * US, record=1))
            sc.append(W.Scenario(9, wid=t, trace=t, profile=pi, ctrl=6, segment=0, mode=W.MODE_DRAIN,
                                 horizon_us=1400 * US, calib_src=src))
    w = W.custom(traces, profs, ctrls, sc)
    w.class_cum = W.MIXED_CLASSES
    bad, st = check_all(w.columns())
    _assert_ok(bad)
    assert int(st["served"].sum()) > 0 and int(st["activations"].sum()) > 0


def _next3_laws_workload():
    """NEXT-3 MPC / BBR / PCC laws (readings R41-R43) across loads,
    profiles, windows, signals and both termination modes; every fourth
    scenario debug-recorded (the DBG instantiation and its controller log)."""
    traces = [W.paper_trace(), W.paper_trace(3.5, 180, 0.6), W.const_trace(3.0, 400), W.const_trace(1.6, 500),
              W.paper_trace(2.0, 90, 0.2)]
    profs = [W.PROFILES["P24"], W.PROFILES["L8B"], dict(W.PROFILES["P24"], max_batch=33, knee=7)]
    ctrls = [
        W.mpc_ctrl(24_000),
        W.mpc_ctrl(26_000, horizon_s=0, w_lat=1, w_q=2, w_osc=1, rungs=(500, 1000, 1500, 2000), window=1),
        W.mpc_ctrl(22_000, horizon_s=16, w_lat=65535, w_q=65535, w_osc=65535, window=8, r_min_bp=1, r_max_bp=5000),
        W.mpc_ctrl(8_000_000, horizon_s=5, w_lat=2, w_q=1, w_osc=0, signal=W.SIG_E2E, window=3),
        W.bbr_ctrl(3_000),
        W.bbr_ctrl(1_000, rungs=(300, 700, 1200, 1900), window=1),
        W.bbr_ctrl(6_000, step_bp=5000, r_min_bp=100, r_max_bp=5000, window=8),
        W.pcc_ctrl(24_000),
        W.pcc_ctrl(22_000, delta_bp=100, w_lat=3, w_q=1, window=1),
        W.pcc_ctrl(300, delta_bp=5000, w_lat=65535, w_q=65535, signal=W.SIG_SLO, slo_us=9_000_000, window=2,
                   r_min_bp=1, r_max_bp=5000),
    ]
    sc = []
    for ti in range(len(traces)):
        for pi in range(len(profs)):
            for ci in range(len(ctrls)):
                for seed in range(2):
                    mode = (ti + ci + seed) % 2
                    rec = 2 if (ti + pi + ci + seed) % 4 == 0 else 0
                    sc.append(W.Scenario(seed + 7 * ti, wid=ti, trace=ti, profile=pi, ctrl=ci, segment=0, mode=mode,
                                         horizon_us=(1400 if mode else 900) * W.US, record=rec))
    return W.custom(traces, profs, ctrls, sc)


def test_next3_mpc_bbr_pcc_laws():
    """GPU parity for the NEXT-3 laws: every summary field, per-scenario
    histograms, and for debug-recorded scenarios the per-second rows and the
    controller log element by element."""
    import torch

    from paper_2510_15330_b200 import Simulator

    w = _next3_laws_workload()
    cols = w.columns()
    bad, st = check_all(cols)
    _assert_ok(bad)
    laws = np.asarray(cols["ctrl_law"])[np.asarray(cols["sc_ctrl"])]
    for law in (W.LAW_MPC, W.LAW_BBR, W.LAW_PCC):
        assert int(st["rewritten"][laws == law].sum()) > 0, law  # every law acted
    sim = Simulator(cols)
    sim.run()
    torch.cuda.synchronize()
    b = oracle.Bound(cols)
    for sid in [i for i, s in enumerate(w.scenarios) if s.record & 2]:
        o = oracle.run_scenario(b, sid, rows_cap=100000, ctrl_log_cap=100000)
        rows, ctrl = sim.series(sid)
        for f in o["rows"].dtype.names:
            assert np.array_equal(rows[f].astype(np.int64), o["rows"][f].astype(np.int64)), (sid, f)
        assert len(ctrl) == len(o["ctrl_log"]), sid
        for g, e in zip(ctrl, o["ctrl_log"]):
            assert (int(g["second"]), int(g["sample"]), int(g["k"]), int(g["r_bp"]), int(g["active"]),
                    int(g["A"])) == (e["second"], e["sample"], e["k"], e["r_bp"], e["active"], e["A"]), sid


def test_next4_token_level_costs():
    """NEXT-4 token-level costs (R44): profiles at 0.25, 0.75, 1.3 and 3
    tokens per word with KV term, KV capacity (reserve and preempt),
    contending prefill and a replayed trace, under OFF / MAP / MPC laws:
    every summary field and histogram vs the oracle."""
    T13 = round(1.3 * 65536)
    traces = [W.paper_trace(), W.const_trace(2.0, 400),
              {"replay": [(0, 500, 9000, 0), (2 * W.US, 800, 4000, 1), (2 * W.US, 300, 15000, 0),
                          (9 * W.US, 700, 12000, 2)] + [(int(10 * W.US + k * 370_000), 400 + k, 2000 + 37 * k, 0)
                                                       for k in range(300)]}]
    profs = [dict(W.PROFILES["P24"], tpw_q16=T13), dict(W.PROFILES["L8B"], tpw_q16=49152),
             dict(W.PROFILES["P24"], tpw_q16=16384, kv_cap_words=60_000),
             dict(W.PROFILES["P24"], tpw_q16=196608, max_batch=16),
             dict(W.PROFILES["L8B"], tpw_q16=T13, kv_cap_words=200_000, kv_policy=1),
             dict(W.PROFILES["P24"], tpw_q16=T13, prefill_mode=1, max_batch=8)]
    ctrls = [W.OFF, W.map_ctrl(24_000, 40_000), W.mpc_ctrl(24_000)]
    sc = []
    for ti in range(len(traces)):
        for pi in range(len(profs)):
            for ci in range(len(ctrls)):
                mode = (ti + pi + ci) % 2
                sc.append(W.Scenario(3 + ti + ci, wid=ti, trace=ti, profile=pi, ctrl=ci, segment=0, mode=mode,
                                     horizon_us=(1500 if mode else 800) * W.US))
    bad, st = check_all(W.custom(traces, profs, ctrls, sc).columns())
    _assert_ok(bad)
    assert int(st["served"].sum()) > 1000


def _replicas_workload():
    """NEXT-4 multi-replica routing (reading R45): 2-8 replicas sharing
    the arrival queue under both routing policies, light to heavy load, with
    token costs, every controller family, the UTIL / E2E / TTFT signals and a
    replayed trace; every fifth scenario debug-recorded."""
    T13 = round(1.3 * 65536)
    traces = [W.paper_trace(), W.const_trace(4.0, 300), W.const_trace(9.0, 120), W.paper_trace(3.5, 180, 0.6),
              {"replay": [(int(k * 250_000), 300 + 7 * k % 500, 1000 + 37 * k % 9000, k % 3) for k in range(400)]}]
    profs = [dict(W.PROFILES["P24"], replicas=2, max_batch=32, route=0),
             dict(W.PROFILES["P24"], replicas=4, max_batch=16, route=1),
             dict(W.PROFILES["P24"], replicas=8, max_batch=8, knee=0, route=0),
             dict(W.PROFILES["L8B"], replicas=3, max_batch=21, route=1, tpw_q16=T13),
             dict(W.PROFILES["L8B"], replicas=2, max_batch=4, route=0),
             dict(W.PROFILES["P24"], replicas=5, max_batch=1, knee=1, route=1)]
    ctrls = [W.OFF, W.map_ctrl(24_000, 40_000), W.mpc_ctrl(24_000), W.bbr_ctrl(3_000), W.pcc_ctrl(24_000),
             W.map_ctrl(5000, 9000, signal=W.SIG_UTIL, window=3), W.map_ctrl(6_000_000, 20_000_000, signal=W.SIG_E2E),
             W.step_ctrl(500_000, 900_000, (500, 1000, 2000), signal=W.SIG_TTFT)]
    sc = []
    k = 0
    for ti in range(len(traces)):
        for pi in range(len(profs)):
            for ci in range(len(ctrls)):
                if (ti * 7 + pi * 3 + ci) % 2:
                    continue
                mode = (ti + pi + ci) % 2
                rec = 2 if k % 5 == 0 else 0
                sc.append(W.Scenario(k % 13, wid=ti, trace=ti, profile=pi, ctrl=ci, segment=0, mode=mode,
                                     horizon_us=(1500 if mode else 700) * W.US, record=rec))
                k += 1
    return W.custom(traces, profs, ctrls, sc)


def test_next4_multi_replica_routing():
    """GPU parity of the multi-replica path: every summary field and histogram,
    and for debug-recorded scenarios the per-second rows and controller log."""
    import torch

    from paper_2510_15330_b200 import Simulator

    w = _replicas_workload()
    cols = w.columns()
    bad, st = check_all(cols)
    _assert_ok(bad)
    assert int(st["ticks"].sum()) > 10**5 and int(st["rewritten"].sum()) > 0
    sim = Simulator(cols)
    sim.run()
    torch.cuda.synchronize()
    b = oracle.Bound(cols)
    for sid in [i for i, s in enumerate(w.scenarios) if s.record & 2]:
        o = oracle.run_scenario(b, sid, rows_cap=100000, ctrl_log_cap=100000)
        rows, ctrl = sim.series(sid)
        for f in o["rows"].dtype.names:
            assert np.array_equal(rows[f].astype(np.int64), o["rows"][f].astype(np.int64)), (sid, f)
        assert [tuple(int(g[k]) for k in ("second", "sample", "k", "r_bp", "active", "A")) for g in ctrl] == \
               [(e["second"], e["sample"], e["k"], e["r_bp"], e["active"], e["A"]) for e in o["ctrl_log"]], sid

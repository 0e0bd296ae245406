"""Queueing-theory and sample-path pins for the oracle (reading R26).

* max_batch = 1, kv = 0: the server is exactly a FIFO M/G/1 queue with service
  S = prefill + (R - 1) d(1) (no alignment wait: the loop starts at the prefill
  end and the next admission happens at the completion instant).  The mean
  queueing delay must match Pollaczek-Khinchine, Wq = lambda E[S^2] / (2 (1 - rho)),
  with E[S], E[S^2] computed exactly from the workload tables.
* Little's law on the sample path: for a drained run,
  sum_i (completion_i - arrival_i) = integral (queued + in_system) dt and
  sum_i queueing_i = integral queued dt, as exact integers.
* Uncongested regime (knee >= max_batch, slope = 0, kv = 0, slots never full):
  prefill + (R-1) t0 <= E2E < prefill + R t0 for every request.
* Determinism (A8) and the null controller.
"""
import numpy as np
import pytest

import workloads as W


def _mg1_workload(lam, D, tabs, seeds, prof):
    scs = [W.Scenario(s, wid=0, trace=0, profile=0, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                      horizon_us=(D + 10**5) * W.US) for s in seeds]
    return W.custom([W.const_trace(lam, D)], [prof], [W.OFF], scs, tables=tabs)


def test_md1_pollaczek_khinchine(orc):
    """M/D/1: R = 500, input = 9000, t0 = 20 ms -> S = 0.72 + 499*0.02 = 10.70 s.
    lambda = 0.05 -> rho = 0.535, Wq = 6.155 s; lambda = 0.08 -> Wq = 31.8 s."""
    prof = dict(W.PROFILES["P24"], max_batch=1)
    tabs = W.constant_tables(L=500, I=9000)
    S = 0.72 + 499 * 0.02
    for lam, D, tol in ((0.05, 200_000, 0.03), (0.08, 400_000, 0.08)):
        rs = orc.run_batch(_mg1_workload(lam, D, tabs, range(16), prof).columns())
        wq = np.mean([r["sum_queue_us"] / r["admitted"] / 1e6 for r in rs])
        want = lam * S * S / (2 * (1 - lam * S))
        assert abs(wq / want - 1) < tol, (lam, wq, want)
        for r in rs:  # sojourn = wait + S exactly for every request
            assert r["sum_e2e_us"] == r["sum_queue_us"] + r["served"] * int(S * 1e6 + 0.5)


def test_mg1_pollaczek_khinchine(orc):
    """M/G/1 with the default workload tables: E[S], E[S^2] enumerated exactly
    over the 4096-entry tables (input independent of (L, Fvar))."""
    prof = dict(W.PROFILES["P24"], max_batch=1)
    tabs = W.quantile_tables()
    pf = prof["prefill_ns_per_word"] * tabs["I"].astype(np.float64) // 1000
    L = tabs["L"].astype(np.int64)[:, None]
    F = tabs["fvar"].astype(np.int64)[None, :]
    U = np.maximum(1, (L * F + 32768) // 65536).astype(np.float64).ravel()
    dec = (U - 1) * prof["t0_us"]
    ES = (pf.mean() + dec.mean()) / 1e6
    ES2 = (np.mean(pf**2) + 2 * pf.mean() * dec.mean() + np.mean(dec**2)) / 1e12
    lam = 0.06
    rs = orc.run_batch(_mg1_workload(lam, 200_000, tabs, range(16), prof).columns())
    wq = np.mean([r["sum_queue_us"] / r["admitted"] / 1e6 for r in rs])
    want = lam * ES2 / (2 * (1 - lam * ES))
    assert abs(wq / want - 1) < 0.04, (wq, want)
    es = np.mean([(r["sum_e2e_us"] - r["sum_queue_us"]) / r["served"] / 1e6 for r in rs])
    assert abs(es / ES - 1) < 0.01


def test_littles_law_sample_path(orc):
    """Exact integer identities on drained runs under batching and the controller."""
    for cfg in (W.config_c3(n_seeds=2), W.config_c1()):
        cols = cfg.columns()
        for sid in range(0, cfg.n_scenarios, max(1, cfg.n_scenarios // 12)):
            r = orc.run_scenario(cols, sid)
            if r["flags"] & 1:
                continue
            assert r["sum_sojourn_us"] == r["int_system_us"]
            assert r["sum_queue_us"] == r["int_queue_us"]
            # conservation at the end
            assert r["arrivals"] == r["served"] + r["queued_end"] + r["inflight_end"]


def test_uncongested_bound(orc):
    """knee >= max_batch, slope 0, kv 0, max_batch never reached: the only waits are
    boundary alignments (admission at the next iteration end, then joining the
    next iteration after the prefill), each shorter than t0:
    prefill + (R-1) t0 <= E2E < prefill + (R+1) t0."""
    prof = dict(t0_us=20_000, knee=64, slope_us=0, kv_ns_per_word=0, max_batch=64,
                prefill_ns_per_word=80_000, e_in=0.05, e_out=0.5, p_idle=300.0)
    w = W.custom([W.const_trace(0.5, 2000)], [prof], [W.OFF],
                 [W.Scenario(4, wid=0, trace=0, profile=0, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                             horizon_us=4000 * W.US)])
    arr = orc.arrivals(w.columns(), 0)
    reqs = [dict(a_us=int(a["a_us"]), input=int(a["input"]), U=int(a["U"])) for a in arr]
    d = orc.simulate(reqs, prof, mode=W.MODE_DRAIN)
    assert d["served"] == len(reqs) > 500
    for q, r in zip(reqs, d["requests"]):
        pf = 80 * q["input"]
        e2e = r["done_us"] - q["a_us"]
        assert 0 <= r["admit_us"] - q["a_us"] < 20_000
        assert pf + (q["U"] - 1) * 20_000 <= e2e < pf + (q["U"] + 1) * 20_000


def test_determinism_and_null_controller(orc):
    """Re-runs are identical (A8); a constant-zero controller equals OFF;
    a constant 20% controller rewrites every admitted request."""
    w = W.config_c2(n_seeds=2, rates=[2.5], horizon_s=120)
    cols = w.columns()
    a = orc.run_scenario(cols, 0)
    b = orc.run_scenario(cols, 0)
    for k in a:
        assert np.array_equal(a[k], b[k]) if isinstance(a[k], np.ndarray) else a[k] == b[k]
    base = dict(W.PROFILES["L8B"])
    arr = orc.arrivals(cols, 0)
    reqs = [dict(a_us=int(x["a_us"]), input=int(x["input"]), U=int(x["U"]), P=int(x["P"]),
                 fcomp_q16=int(x["fcomp_q16"])) for x in arr]
    off = orc.simulate(reqs, base, mode=W.MODE_CUTOFF, horizon_us=120 * W.US)
    zero = orc.simulate(reqs, base, ctrl=orc.make_ctrl(law=W.LAW_CONST, r_const_bp=0),
                        mode=W.MODE_CUTOFF, horizon_us=120 * W.US)
    for k in ("ticks", "served", "words_out", "sum_e2e_us", "energy_j", "rewritten"):
        assert off[k] == zero[k]
    c20 = orc.simulate(reqs, base, ctrl=orc.make_ctrl(law=W.LAW_CONST, r_const_bp=2000),
                       mode=W.MODE_CUTOFF, horizon_us=120 * W.US)
    assert c20["rewritten"] == c20["admitted"] > 0
    assert all(r["r_bp"] == 2000 for r in c20["requests"] if r["admit_us"] != 2**64 - 1)


def test_fewer_words_when_bounded(orc):
    """compliance noise 0, a fixed r > 0 on every request, drained: total
    realized words <= unbounded total (here with the predictor = truth, fvar = 1)."""
    tabs = W.quantile_tables()
    tabs["fcomp"][:] = 65536
    tabs["noise"][:] = 0
    tabs["fvar"][:] = 65536
    w = W.custom([W.paper_trace()], ["P24"], [W.OFF],
                 [W.Scenario(1, wid=0, trace=0, profile=0, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                             horizon_us=3000 * W.US)], tables=tabs)
    arr = orc.arrivals(w.columns(), 0)
    reqs = [dict(a_us=int(x["a_us"]), input=int(x["input"]), U=int(x["U"]), P=int(x["P"])) for x in arr]
    un = orc.simulate(reqs, W.PROFILES["P24"], mode=W.MODE_DRAIN)
    bd = orc.simulate(reqs, W.PROFILES["P24"], ctrl=orc.make_ctrl(law=W.LAW_CONST, r_const_bp=1000),
                      mode=W.MODE_DRAIN)
    assert un["served"] == bd["served"] == len(reqs)
    assert bd["words_out"] <= un["words_out"]
    assert bd["words_out"] == sum(max(1, (q["U"] * 9000 + 5000) // 10000) for q in reqs)


@pytest.mark.parametrize("profile", ["P24", "L8B"])
def test_a3_saturation_brackets(profile):
    """A3 (readings R1 / R27): the recalibrated profiles saturate near
    the paper's onset (~2.4 RPS).  Fluid queue slope between 300 s and
    600 s of a constant-rate Poisson stream, averaged over 32 seeds (same seed =
    same arrivals at both horizons, R32): |slope| < 0.01 req/s at 2.2 RPS and
    > 0.05 req/s at 2.6 RPS.  This is the sweep DESIGN.md §3 R1 cites."""
    import oracle

    seeds = 32
    slopes = {}
    for rate in (2.2, 2.6):
        sc = []
        for s in range(seeds):
            for H in (300, 600):
                sc.append(W.Scenario(s, wid=0, trace=0, profile=0, ctrl=0, segment=0, mode=W.MODE_CUTOFF,
                                     horizon_us=H * W.US))
        w = W.custom([W.const_trace(rate, 600)], [W.PROFILES[profile]], [W.OFF], sc)
        rs = oracle.run_batch(oracle.Bound(w.columns()))
        q = np.array([r["queued_end"] for r in rs], dtype=np.float64).reshape(seeds, 2)
        slopes[rate] = float(np.mean(q[:, 1] - q[:, 0]) / 300.0)
    assert abs(slopes[2.2]) < 0.01, slopes
    assert slopes[2.6] > 0.05, slopes

"""Pins for the oracle's controller (a6) and the signals, percentiles and
transition log it reports — the parts VERDICT r1 listed as unpinned.

* hand-worked controller sequences for every law (tests/golden/controller_sequences.json:
  STEP ladder, MAP with a partial window and gap seconds, MPC, BBR, PCC),
  through the controller-only entry orc_ctrl_trace;
* the E2E and SLO per-second signals recomputed from the per-request log
  (R3: E2E by completion second; SLO per-mille with a strict > slo_us);
* the transition log recomputed from the controller log of whole runs;
* histogram percentiles (a9, R13): the exact nearest-rank value lies in the
  reported bin, and median r / median similarity recomputed from the request log;
* STEP / E2E / the NEXT-3 laws in the loop vs the brute-force simulator.
"""
import json
import os

import numpy as np
import pytest

import workloads as W
from tests import bruteforce

GOLD = os.path.join(os.path.dirname(__file__), "golden", "controller_sequences.json")
NONE = 0xFFFFFFFF


def _cases():
    with open(GOLD) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"][:40])
def test_hand_worked_controller_sequence(orc, case):
    c = dict(case["ctrl"])
    rungs = tuple(c.pop("rungs", ()))
    ctrl = orc.make_ctrl(rungs=rungs, **c)
    got = orc.ctrl_trace(ctrl, case["x"], words=case.get("w"), seconds=case.get("seconds"))
    assert got["r"] == case["r"]
    assert got["activations"] == case["activations"]
    assert got["first_act_s"] == (NONE if case["first_act_s"] is None else case["first_act_s"])
    assert got["last_deact_s"] == (NONE if case["last_deact_s"] is None else case["last_deact_s"])
    assert got["active_ingests"] == case["active_ingests"]


def _stream(rng, n=80, gap=250_000, inp=(100, 3000), U=(2, 40)):
    reqs, t = [], 0
    for _ in range(n):
        t += int(rng.integers(0, gap))
        reqs.append(dict(a_us=t, input=int(rng.integers(*inp)), U=int(rng.integers(*U)),
                         P=int(rng.integers(*U)) + 5))
    return reqs


LIT = W.PROFILES["spec-literal"]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_e2e_signal_is_mean_e2e_of_completions_per_second(orc, seed):
    """R3 E2E: the sample of second s is floor(sum E2E / n) over the requests
    completing in s (completion second, not admission second); seconds with no
    completion are gaps.  Recomputed from the per-request log."""
    reqs = _stream(np.random.default_rng(seed))
    c = orc.make_ctrl(law=W.LAW_MAP, signal=W.SIG_E2E, t1=10**10, t2=2 * 10**10)
    d = orc.simulate(reqs, LIT, ctrl=c, mode=W.MODE_DRAIN)
    per = {}
    for q, r in zip(reqs, d["requests"]):
        per.setdefault(r["done_us"] // 10**6, []).append(r["done_us"] - q["a_us"])
    got = {e["second"]: e["sample"] for e in d["ctrl_log"]}
    want = {s: sum(v) // len(v) for s, v in per.items() if (s + 1) * 10**6 <= d["end_us"]}
    assert got == want and len(got) > 5


@pytest.mark.parametrize("seed", [4, 5])
def test_slo_signal_is_strict_violation_per_mille(orc, seed):
    """R3 SLO: floor(1000 #(E2E > slo_us) / completions) per completion second;
    an E2E exactly equal to slo_us is not a violation (strict >).  The SLO is
    set to an E2E that occurs, so the boundary case is exercised."""
    reqs = _stream(np.random.default_rng(seed))
    probe = orc.simulate(reqs, LIT, mode=W.MODE_DRAIN)
    e2es = sorted(r["done_us"] - q["a_us"] for q, r in zip(reqs, probe["requests"]))
    slo = e2es[len(e2es) // 2]
    c = orc.make_ctrl(law=W.LAW_MAP, signal=W.SIG_SLO, slo_us=slo, t1=2000, t2=3000)  # never activates
    d = orc.simulate(reqs, LIT, ctrl=c, mode=W.MODE_DRAIN)
    per = {}
    for q, r in zip(reqs, d["requests"]):
        e = r["done_us"] - q["a_us"]
        per.setdefault(r["done_us"] // 10**6, []).append(e)
    got = {e["second"]: e["sample"] for e in d["ctrl_log"]}
    want = {s: 1000 * sum(1 for e in v if e > slo) // len(v) for s, v in per.items()
            if (s + 1) * 10**6 <= d["end_us"]}
    assert got == want
    assert d["slo_violations"] == sum(1 for e in e2es if e > slo)
    assert any(e == slo for e in e2es)


def _transitions(log):
    """S:332 transition log from the per-ingest controller log."""
    acts, first, last, active = 0, NONE, NONE, 0
    prev = 0
    for e in log:
        if e["active"] and not prev:
            acts += 1
            if first == NONE:
                first = e["second"]
        if not e["active"] and prev:
            last = e["second"]
        active += e["active"]
        prev = e["active"]
    return acts, first, last, active


@pytest.mark.parametrize("seed", range(4))
def test_transition_log_matches_controller_log(orc, seed):
    """activations, first activation second, last deactivation second and
    active ingests equal what the per-ingest controller log implies, on
    calibrated paper-trace pairs (MAP) and every other law."""
    w = W.config_paper_pair(seed)
    cols = w.columns()
    d = orc.run_scenario(cols, 1, ctrl_log_cap=5000)
    assert d["n_ctrl"] == len(d["ctrl_log"]) > 100
    assert _transitions(d["ctrl_log"]) == (d["activations"], d["first_act_s"], d["last_deact_s"],
                                           d["active_ingests"])
    assert d["activations"] >= 1


def test_transition_log_every_law(orc):
    rng = np.random.default_rng(17)
    reqs = _stream(rng, n=160, gap=150_000)
    P24 = W.PROFILES["P24"]
    ctrls = [orc.make_ctrl(law=W.LAW_STEP, t1=24_000, t2=40_000, rungs=(500, 1000, 1500, 2000)),
             orc.make_ctrl(law=W.LAW_MAP, t1=24_000, t2=40_000, window=3),
             orc.make_ctrl(law=W.LAW_MPC, t1=24_000, horizon_s=3, w_lat=4, w_q=1, w_osc=2),
             orc.make_ctrl(law=W.LAW_BBR, t1=3_000, step_bp=250),
             orc.make_ctrl(law=W.LAW_PCC, t1=24_000, w_lat=1, w_q=4, step_bp=250)]
    for c in ctrls:
        d = orc.simulate(reqs, dict(P24, max_batch=8), ctrl=c, mode=W.MODE_DRAIN)
        log = d["ctrl_log"]
        assert _transitions(log) == (d["activations"], d["first_act_s"], d["last_deact_s"], d["active_ingests"])
        # every r applied at admission is the one in force: the log's r of the last ingest before it
        for q, r in zip(reqs, d["requests"]):
            before = [e["r_bp"] for e in log if (e["second"] + 1) * 10**6 <= r["admit_us"]]
            assert r["r_bp"] == (before[-1] if before else 0)


def _nr(vals, p):
    v = sorted(vals)
    return v[max(1, -(-p * len(v) // 100)) - 1]


@pytest.mark.parametrize("sid", range(0, 64, 9))
def test_histogram_percentiles_bracket_exact_values(orc, sid):
    """a9 / R13: the histogram p50/p99 of E2E and TTFT is the lower edge of
    the bin holding the exact nearest-rank value: edge(b) <= exact < edge(b+1),
    exact recomputed from the per-request log (not the oracle's self-check)."""
    w = W.config_c2(n_seeds=4, rates=[1.5, 2.5, 4.0, 6.0], horizon_s=300)
    cols = w.columns()
    sid = sid % w.n_scenarios
    arr = orc.arrivals(cols, sid)
    reqs = [dict(a_us=int(a["a_us"]), j=int(a["j"]), L=int(a["L"]), input=int(a["input"]), U=int(a["U"]),
                 P=int(a["P"]), fcomp_q16=int(a["fcomp_q16"]), qnoise=int(a["qnoise"]), cls=int(a["cls"]))
            for a in arr]
    prof = W.PROFILES["L8B"]
    d = orc.simulate(reqs, prof, mode=W.MODE_CUTOFF, horizon_us=300 * 10**6)
    e2e = [(r["done_us"] - q["a_us"]) // 1000 for q, r in zip(reqs, d["requests"]) if r["done_us"] < 2**63]
    ttft = [(r["first_us"] - q["a_us"]) // 1000 for q, r in zip(reqs, d["requests"]) if r["first_us"] < 2**63]
    assert len(e2e) == d["served"] > 10
    for vals, keys in ((e2e, ("e2e_p50_ms", "e2e_p99_ms")), (ttft, ("ttft_p50_ms", "ttft_p99_ms"))):
        for p, k in zip((50, 99), keys):
            exact = _nr(vals, p)
            b = orc.lat_bin(d[k])
            assert orc.lat_edge(b) == d[k]
            assert orc.lat_edge(b) <= exact < orc.lat_edge(b + 1), (k, exact, d[k])


def test_median_r_and_similarity_from_request_log(orc):
    """median_r_bp (10 bp bins) and the active / inactive median similarity
    (0.5-point bins) recomputed from the per-request log: nearest-rank median of
    r over rewritten admissions floored to its bin; similarity of each admitted
    request from S:145-153 (orc.similarity, pinned by S:151-153) with its own
    U, R and noise."""
    rng = np.random.default_rng(23)
    reqs = []
    t = 0
    for i in range(300):
        t += int(rng.integers(0, 60_000))
        reqs.append(dict(a_us=t, input=int(rng.integers(100, 3000)), U=int(rng.integers(50, 700)),
                         P=int(rng.integers(50, 700)), qnoise=int(rng.integers(-400, 400)),
                         fcomp_q16=int(rng.integers(58000, 72000))))
    c = orc.make_ctrl(law=W.LAW_MAP, t1=22_000, t2=30_000, window=3)
    d = orc.simulate(reqs, dict(W.PROFILES["P24"], max_batch=16), ctrl=c, mode=W.MODE_DRAIN)
    rs = [r["r_bp"] for r in d["requests"] if r["r_bp"] > 0]
    assert len(rs) == d["rewritten"] > 20 and len(set(rs)) > 3
    assert d["median_r_bp"] == _nr(rs, 50) // 10 * 10
    act, inact = [], []
    for q, r in zip(reqs, d["requests"]):
        s = orc.similarity(q["U"], r["R"], r["r_bp"] > 0, q["qnoise"])
        (act if r["r_bp"] > 0 else inact).append(s)
    assert d["scored_active"] == len(act) and d["scored_inactive"] == len(inact)
    assert d["sim_active_p50"] == _nr(act, 50) // 50 * 50
    assert d["sim_inactive_p50"] == _nr(inact, 50) // 50 * 50


def _bf_reqs(rng, n=14, gap=250_000):
    reqs, t = [], 0
    for _ in range(n):
        t += int(rng.integers(0, gap))
        reqs.append(dict(a_us=t, input=int(rng.integers(1, 100)), U=int(rng.integers(2, 30)),
                         P=int(rng.integers(5, 40)), fcomp_q16=65536))
    return reqs


BF_PROF = dict(t0_us=20_000, knee=1, slope_us=9000, kv_ns_per_word=0, max_batch=4,
               prefill_ns_per_word=1000, e_in=0.05, e_out=0.5, p_idle=300.0)


@pytest.mark.parametrize("law", ["step", "mpc", "bbr", "pcc", "map_e2e", "map_slo"])
def test_bruteforce_controller_laws(orc, law):
    """Every law (and the E2E / SLO signals) in the loop vs the brute-force
    microsecond simulator, which computes its own per-second samples and its own
    law in exact rationals: same admissions, realized lengths and r per request."""
    rng = np.random.default_rng({"step": 31, "mpc": 32, "bbr": 33, "pcc": 34, "map_e2e": 35, "map_slo": 36}[law])
    acted = 0
    for case in range(6):
        reqs = _bf_reqs(rng)
        t1 = 25_000 + 2000 * case
        if law == "step":
            kw = dict(law="step", t1=t1, rungs=(500, 1000, 1500, 2000))
            c = orc.make_ctrl(law=W.LAW_STEP, t1=t1, t2=t1 + 1, rungs=(500, 1000, 1500, 2000))
        elif law == "mpc":
            kw = dict(law="mpc", t1=t1, horizon_s=2, w_lat=3, w_q=1, w_osc=1, window=3)
            c = orc.make_ctrl(law=W.LAW_MPC, t1=t1, window=3, horizon_s=2, w_lat=3, w_q=1, w_osc=1)
        elif law == "bbr":
            kw = dict(law="bbr", t1=2000 + 1000 * case, step_bp=300, window=3)
            c = orc.make_ctrl(law=W.LAW_BBR, t1=2000 + 1000 * case, window=3, step_bp=300)
        elif law == "pcc":
            kw = dict(law="pcc", t1=t1, w_lat=1, w_q=3, step_bp=300, window=2)
            c = orc.make_ctrl(law=W.LAW_PCC, t1=t1, window=2, w_lat=1, w_q=3, step_bp=300)
        elif law == "map_e2e":
            t1e = 400_000 + 50_000 * case
            kw = dict(law="map", t1=t1e, t2=t1e + 300_000, signal="e2e")
            c = orc.make_ctrl(law=W.LAW_MAP, signal=W.SIG_E2E, t1=t1e, t2=t1e + 300_000)
        else:
            kw = dict(law="map", t1=200, t2=800, signal="slo", slo_us=350_000 + 20_000 * case, window=2)
            c = orc.make_ctrl(law=W.LAW_MAP, signal=W.SIG_SLO, t1=200, t2=800, slo_us=350_000 + 20_000 * case,
                              window=2)
        bf = bruteforce.simulate(reqs, BF_PROF, 6_000_000, **kw)
        d = orc.simulate(reqs, BF_PROF, ctrl=c, mode=W.MODE_DRAIN, horizon_us=6_000_000)
        assert d["ticks"] == bf["ticks"], (law, case)
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["done_us"], r["R"], r["r_bp"]) == \
                   (bf["admit"][i], bf["done"][i], bf["R"][i], bf["r_bp"][i]), (law, case, i)
        acted += any(r["r_bp"] > 0 for r in d["requests"])
    assert acted >= 2, law  # the law acted in the loop, not only stayed at r = 0


def test_next3_law_invariants(orc):
    """Properties the NEXT-3 readings imply, over random sample streams:
    MPC (R41) — r in {0} U candidates; with no oscillation cost the chosen r is
    non-decreasing in the load (every sample scaled up); BBR (R42) — r in {0} U
    [r_min, r_max], one step per ingest at most, and it only rises at the
    bandwidth plateau while congested; PCC (R43) — r in {0} U [r_min, r_max]
    and, while active, consecutive experiments alternate above / below r_base."""
    rng = np.random.default_rng(77)
    for case in range(200):
        n = int(rng.integers(3, 40))
        x = [int(v) for v in rng.integers(10_000, 90_000, n)]
        w = [int(v) for v in rng.integers(1, 200, n)]
        # MPC
        c = orc.make_ctrl(law=W.LAW_MPC, t1=40_000, window=int(rng.integers(1, 9)), horizon_s=int(rng.integers(0, 5)),
                          w_lat=int(rng.integers(1, 20)), w_q=int(rng.integers(0, 5)), w_osc=0)
        cands = {0} | {500 + i * 1500 // 30 for i in range(31)}
        lo = orc.ctrl_trace(c, x)["r"]
        hi = orc.ctrl_trace(c, [v * 5 // 4 for v in x])["r"]
        assert set(lo) <= cands and set(hi) <= cands
        assert all(b >= a for a, b in zip(lo, hi)), case
        # BBR
        step = int(rng.integers(50, 800))
        c = orc.make_ctrl(law=W.LAW_BBR, t1=int(rng.integers(0, 20_000)), window=int(rng.integers(1, 9)), step_bp=step)
        r = orc.ctrl_trace(c, x, words=w)["r"]
        prev = 0
        for v in r:
            assert v == 0 or 500 <= v <= 2000
            assert abs(v - prev) <= max(step, 500), (case, prev, v)  # 0 <-> r_min jumps, else one step
            prev = v
        # PCC
        d = int(rng.integers(50, 800))
        c = orc.make_ctrl(law=W.LAW_PCC, t1=40_000, window=int(rng.integers(1, 9)), w_lat=1, w_q=4, step_bp=d)
        t = orc.ctrl_trace(c, x)
        for v in t["r"]:
            assert v == 0 or 500 <= v <= 2000
        run = []
        for v, a in zip(t["r"], t["active"]):
            if not a:
                run = []
                continue
            run.append(v)
            if len(run) >= 2 and run[-1] != run[-2]:
                assert (run[-1] > run[-2]) == (len(run) % 2 == 1) or min(run[-1], run[-2]) in (500, 2000)

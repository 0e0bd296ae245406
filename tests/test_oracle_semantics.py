"""Pins for the oracle's serving simulation and controller (a4-a10).

* hand-computed timelines (tests/golden/appendixA_fixtures.json: SPEC S:207,
  S:233 and SURVEY Appendix A F2-F5);
* SPEC.md's worked examples (S:124-144, S:215-226, S:233-235, S:289-327,
  S:376-378) — exact;
* a brute-force microsecond-stepping simulator (tests/bruteforce.py) on random
  tiny traces — exact, per request and per gap.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import workloads as W
from tests import bruteforce

GOLD = os.path.join(os.path.dirname(__file__), "golden", "appendixA_fixtures.json")


def _fixtures():
    with open(GOLD) as f:
        g = json.load(f)
    return [(g["profile"], fx) for fx in g["fixtures"]]


@pytest.mark.parametrize("prof,fx", _fixtures(), ids=lambda x: x.get("name", "") if isinstance(x, dict) else "")
def test_appendix_fixture(orc, prof, fx):
    prof = dict(prof, **fx.get("profile_override", {}))
    d = orc.simulate(fx["requests"], prof, mode=W.MODE_DRAIN)
    for i, er in enumerate(fx.get("expect_requests", [])):
        for k, v in er.items():
            assert d["requests"][i][k] == v, (fx["name"], i, k)
    for i, eg in enumerate(fx.get("expect_gaps", [])):
        assert d["gaps"][i] == eg, (fx["name"], i)
    for i, eg in enumerate(fx.get("expect_gap_first3", [])):
        assert d["gaps"][i][:3] == eg
    for k, v in fx["expect"].items():
        assert d[k] == v, (fx["name"], k, d[k], v)
    # latency ordering E2E >= TTFT >= queueing >= 0
    for i, q in enumerate(fx["requests"]):
        r = d["requests"][i]
        assert r["done_us"] - q["a_us"] >= r["first_us"] - q["a_us"] >= r["admit_us"] - q["a_us"] >= 0


LIT = W.PROFILES["spec-literal"]


def test_cost_law_examples(orc):
    """d(1) = 50 ms; d(16) = 50 + 6*8 = 98 ms (one iteration, drain)."""
    for B, d_us in ((1, 50_000), (16, 98_000), (8, 50_000), (9, 56_000)):
        reqs = [dict(a_us=0, input=1, U=2) for _ in range(B)]
        d = orc.simulate(reqs, LIT, mode=W.MODE_DRAIN)
        assert d["ticks"] == 1 and d["end_us"] == 80 + d_us
        assert d["tbt_sum_us"] == B * d_us


def test_prefill_examples(orc):
    """10,000 words at 80 ms/kword -> 800 ms; 1 word -> 0.08 ms."""
    for inp, pf in ((10_000, 800_000), (1, 80)):
        d = orc.simulate([dict(a_us=0, input=inp, U=1)], LIT, mode=W.MODE_DRAIN)
        assert d["requests"][0]["first_us"] == pf and d["ticks"] == 0


def test_kv_term(orc):
    """Reading R2: d = t0 + slope*max(0,B-knee) + floor(kv_ns*K/1000), K = sum of
    (input + words emitted) over the batch at iteration start."""
    prof = dict(LIT, kv_ns_per_word=70)
    d = orc.simulate([dict(a_us=0, input=1000, U=3), dict(a_us=0, input=3000, U=2)], prof, mode=W.MODE_DRAIN)
    # both first words at 80,000 / 240,000; A joins at 80,000 alone: K = 1001
    # -> d = 50,000 + 70 (floor(70*1001/1000) = 70)
    g = d["gaps"]
    assert g[0][0] == 50_070


def test_energy_examples(orc):
    """one request (10,000 in / 500 out) -> 750 J; 0 requests over
    10 s at 100 W -> 1,000 J; S:235 additivity over disjoint windows."""
    prof = dict(LIT, p_idle=100.0)
    d = orc.simulate([], prof, mode=W.MODE_CUTOFF, horizon_us=10 * W.US)
    assert d["energy_j"] == 1000.0
    d = orc.simulate([dict(a_us=0, input=10_000, U=500)], LIT, mode=W.MODE_DRAIN)
    assert d["energy_j"] == 750.0
    reqs = [dict(a_us=k * 400_000, input=1000 + k, U=20 + k) for k in range(12)]
    full = orc.simulate(reqs, LIT, mode=W.MODE_CUTOFF, horizon_us=8 * W.US)
    a = orc.simulate(reqs, LIT, mode=W.MODE_CUTOFF, horizon_us=8 * W.US, w0_us=0, w1_us=3 * W.US)
    b = orc.simulate(reqs, LIT, mode=W.MODE_CUTOFF, horizon_us=8 * W.US, w0_us=3 * W.US, w1_us=8 * W.US)
    assert a["win_energy_j"] + b["win_energy_j"] == pytest.approx(full["energy_j"], rel=1e-12)
    assert a["win_served"] + b["win_served"] == full["served"]
    assert a["win_words_out"] + b["win_words_out"] == full["words_out"]


def test_rewrite_examples(orc):
    """S:133-135 bounded_target: (500, 8%) -> 460, (350, 20%) -> 280; S:142 identity
    compliance 460 -> 460; S:144 poly (50, 0.8, 0) at N = 300 -> 290."""
    for P, r, want in ((500, 800, 460), (350, 2000, 280), (500, 0, None)):
        c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=r)
        d = orc.simulate([dict(a_us=0, input=1, U=777, P=P)], LIT, ctrl=c, mode=W.MODE_DRAIN)
        assert d["requests"][0]["R"] == (want if want else 777)
        assert d["rewritten"] == (1 if r else 0)
    poly = (50 * 65536, 52429, 0)  # Q16 of (50, 0.8, 0)
    c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=2000)
    d = orc.simulate([dict(a_us=0, input=1, U=777, P=375)], LIT, ctrl=c, mode=W.MODE_DRAIN, poly_q16=poly)
    assert d["requests"][0]["R"] == 290
    # compliance noise: realized = round(N * Fcomp)
    d = orc.simulate([dict(a_us=0, input=1, U=777, P=500, fcomp_q16=int(1.05 * 65536))], LIT, ctrl=orc.make_ctrl(
        law=W.LAW_CONST, r_const_bp=800), mode=W.MODE_DRAIN)
    assert d["requests"][0]["R"] == 483  # round(460 * 1.05 = 482.99...)


def test_controller_examples(orc):
    """S:289-301 with t1 = 50,000 µs, t2 = 100,000 µs."""
    c = orc.make_ctrl(law=W.LAW_MAP, t1=50_000, t2=100_000)
    assert orc.map_rate(10_000 * 3 + 50_000 * 2, 5, c) == 0      # MA 26 ms < t1
    assert orc.map_rate(5 * 50_000, 5, c) == 500                  # five samples = T1 -> 5%
    assert orc.map_rate(40_000, 1, c) == 0
    assert orc.map_rate(50_000, 1, c) == 500
    assert orc.map_rate(75_000, 1, c) == 1250
    assert orc.map_rate(180_000, 1, c) == 2000
    ladder = orc.make_ctrl(law=W.LAW_MAP, t1=50_000, t2=100_000, r_min_bp=500, r_max_bp=2000,
                           rungs=(500, 1000, 1500, 2000))
    assert orc.map_rate(75_000, 1, ladder) == 1000


def test_map_law_vs_fraction(orc):
    """The integer law equals floor(r_min + (r_max-r_min)(MA-t1)/(t2-t1)) in exact rationals."""
    rng = np.random.default_rng(5)
    for _ in range(3000):
        t1 = int(rng.integers(1, 100_000))
        t2 = t1 + int(rng.integers(1, 100_000))
        rmin = int(rng.integers(1, 3000))
        rmax = rmin + int(rng.integers(0, 2000))
        k = int(rng.integers(1, 9))
        A = int(rng.integers(0, 3 * t2 * k))
        c = orc.make_ctrl(law=W.LAW_MAP, t1=t1, t2=t2, r_min_bp=rmin, r_max_bp=rmax)
        ma = Fraction(A, k)
        want = 0 if ma < t1 else min(rmax, int(rmin + (rmax - rmin) * (ma - t1) / (t2 - t1)))
        got = orc.map_rate(A, k, c)
        assert got == want
        # range {0} U [r_min, r_max] and monotone in MA
        assert got == 0 or rmin <= got <= rmax
        assert orc.map_rate(A + k, k, c) >= got


def test_calibration_examples(orc):
    """S:308-310 and the percentile examples S:376-378."""
    assert orc.calibrate(list(range(10, 111, 10))) == (0, 60, 90)
    assert orc.calibrate([5, 5, 5, 5])[0] == 2
    assert orc.calibrate([1, 2, 3])[0] == 1
    assert orc.percentile(list(range(10, 111, 10)), 50) == 60
    v = [17, 3, 99, 42, 8]
    assert orc.percentile(v, 0) == 3 and orc.percentile(v, 100) == 99
    assert orc.percentile([7], 75) == 7


def test_latency_bins(orc):
    """a9 bins: exact below 32 ms, then 32 log-linear sub-buckets per octave."""
    assert [orc.lat_bin(x) for x in range(32)] == list(range(32))
    for b in range(895):
        lo, hi = orc.lat_edge(b), orc.lat_edge(b + 1)
        assert lo < hi
        assert orc.lat_bin(lo) == b and orc.lat_bin(hi - 1) == b
        if b >= 32:
            assert (hi - lo) * 32 <= lo  # relative width <= 1/32
    assert orc.lat_bin(2**32 - 1) == 895


def _random_tiny(rng):
    n = int(rng.integers(1, 7))
    reqs = []
    for i in range(n):
        reqs.append(dict(a_us=int(rng.integers(0, 4000)), input=int(rng.integers(1, 40)),
                         U=int(rng.integers(1, 9)), P=int(rng.integers(1, 12)),
                         fcomp_q16=int(rng.integers(50000, 80000))))
    reqs.sort(key=lambda q: q["a_us"])
    prof = dict(t0_us=int(rng.integers(1, 300)), knee=int(rng.integers(0, 4)), slope_us=int(rng.integers(0, 90)),
                kv_ns_per_word=int(rng.integers(0, 3000)), max_batch=int(rng.integers(1, 5)),
                prefill_ns_per_word=int(rng.integers(0, 40_000)), e_in=0.05, e_out=0.5, p_idle=300.0)
    prof["knee"] = min(prof["knee"], prof["max_batch"])
    return reqs, prof


def test_bruteforce_tiny_traces(orc):
    """Event-heap DES == microsecond-stepping brute force on 120 random tiny traces."""
    rng = np.random.default_rng(11)
    for case in range(120):
        reqs, prof = _random_tiny(rng)
        law = "const" if case % 3 == 0 else "off"
        rc = int(rng.integers(100, 3000)) if law == "const" else 0
        bf = bruteforce.simulate(reqs, prof, 10**6, law=law, r_const=rc)
        c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=rc) if law == "const" else None
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=10**6)
        assert d["ticks"] == bf["ticks"], case
        assert d["words_out"] == bf["words_out"], case
        assert d["end_us"] == bf["end_us"], case
        assert d["served"] == bf["served"], case
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["first_us"], r["done_us"], r["R"]) == \
                   (bf["admit"][i], bf["first"][i], bf["done"][i], bf["R"][i]), (case, i)
            assert d["gaps"][i] == bf["gaps"][i], (case, i)


def test_bruteforce_controller(orc):
    """Controller in the loop (MAP law, TBT signal) vs brute force on short traces
    spanning several seconds."""
    rng = np.random.default_rng(3)
    prof = dict(t0_us=20_000, knee=1, slope_us=9000, kv_ns_per_word=0, max_batch=4,
                prefill_ns_per_word=1000, e_in=0.05, e_out=0.5, p_idle=300.0)
    for case in range(6):
        reqs = []
        t = 0
        for i in range(14):
            t += int(rng.integers(0, 250_000))
            reqs.append(dict(a_us=t, input=int(rng.integers(1, 100)), U=int(rng.integers(2, 30)),
                             P=int(rng.integers(5, 40)), fcomp_q16=65536))
        t1, t2 = 25_000 + 2000 * case, 40_000 + 2000 * case
        bf = bruteforce.simulate(reqs, prof, 2_000_000 * 3, law="map", t1=t1, t2=t2)
        c = orc.make_ctrl(law=W.LAW_MAP, t1=t1, t2=t2)
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=6_000_000)
        assert d["ticks"] == bf["ticks"]
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["done_us"], r["R"], r["r_bp"]) == \
                   (bf["admit"][i], bf["done"][i], bf["R"][i], bf["r_bp"][i]), (case, i)


def test_similarity_model_examples(orc):
    """NEXT-2 quality model: inactive, reduction 0 -> 88;
    active, reduction 8 % -> 87; active, reduction 40 % (= decay_end) -> 65;
    S:158 non-increasing in the reduction beyond the safe window; S:159 clamps."""
    assert orc.similarity(500, 500, False) == 8800
    assert orc.similarity(500, 460, True) == 8700
    assert orc.similarity(500, 300, True) == 6500
    prev = None
    for R in range(400, 200, -1):  # reduction 20 % .. 60 %
        s = orc.similarity(500, R, True)
        assert prev is None or s <= prev
        prev = s
    assert orc.similarity(500, 450, True, noise=3000) == 10000
    assert orc.similarity(500, 100, True, noise=-9000) == 0
    # linear decay midpoint: reduction 30 % -> 87 - 22/2 = 76 points
    assert orc.similarity(1000, 700, True) == 7600


def test_class_and_short_output_bypass(orc):
    """NEXT-3: a class with the bypass policy is never rewritten; S:314 /
    S:267: a predicted length below min_words_bypass is never rewritten; S:333:
    within one admission point all non-bypassed requests carry the same r."""
    reqs = [dict(a_us=k * 1000, input=10, U=50 + k, P=40 + 5 * k, cls=k % 3) for k in range(30)]
    c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=1500, bypass_mask=0b010, min_words_bypass=70)
    d = orc.simulate(reqs, LIT, ctrl=c, mode=W.MODE_DRAIN)
    for q, r in zip(reqs, d["requests"]):
        bypass = q["cls"] == 1 or q["P"] < 70
        assert r["r_bp"] == (0 if bypass else 1500)
        assert r["R"] == (q["U"] if bypass else max(1, (q["P"] * 8500 + 5000) // 10000))
    assert d["bypassed"] == sum(1 for q in reqs if q["cls"] == 1 or q["P"] < 70)
    assert d["rewritten"] + d["bypassed"] == d["admitted"]
    # fairness: equal r per admission instant among non-bypassed requests
    by_t = {}
    for q, r in zip(reqs, d["requests"]):
        if not (q["cls"] == 1 or q["P"] < 70):
            by_t.setdefault(r["admit_us"], set()).add(r["r_bp"])
    assert all(len(v) == 1 for v in by_t.values())


def test_ttft_signal_is_per_second_mean(orc):
    """NEXT-3 signal ("TTFT could offer early insights"): the sample of
    second s is floor(mean TTFT of the first words emitted in s)."""
    rng = np.random.default_rng(9)
    reqs = []
    t = 0
    for i in range(60):
        t += int(rng.integers(0, 300_000))
        reqs.append(dict(a_us=t, input=int(rng.integers(100, 3000)), U=int(rng.integers(2, 40))))
    c = orc.make_ctrl(law=W.LAW_MAP, signal=W.SIG_TTFT, t1=10**9, t2=2 * 10**9)
    d = orc.simulate(reqs, LIT, ctrl=c, mode=W.MODE_DRAIN)
    want = {}
    for q, r in zip(reqs, d["requests"]):
        s = r["first_us"] // 10**6
        want.setdefault(s, []).append(r["first_us"] - q["a_us"])
    got = {e["second"]: e["sample"] for e in d["ctrl_log"]}
    closed = {s: sum(v) // len(v) for s, v in want.items() if (s + 1) * 10**6 <= d["end_us"]}
    assert got == closed


def _signal_run(orc, signal, seed, max_batch=None):
    rng = np.random.default_rng(seed)
    reqs = []
    t = 0
    for i in range(80):
        t += int(rng.integers(0, 250_000))
        reqs.append(dict(a_us=t, input=int(rng.integers(100, 3000)), U=int(rng.integers(2, 40))))
    prof = dict(LIT, max_batch=max_batch) if max_batch else LIT
    c = orc.make_ctrl(law=W.LAW_MAP, signal=signal, t1=10**9, t2=2 * 10**9)
    return reqs, prof, orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN)


def test_input_signal_is_admitted_words_per_second(orc):
    """NEXT-3 signal ("input tokens per unit time to the LLM serving
    system"): the sample of second s is the input words admitted in s; seconds
    without an admission are gaps.  Recomputed from the per-request log."""
    reqs, _, d = _signal_run(orc, W.SIG_INPUT, 10)
    want = {}
    for q, r in zip(reqs, d["requests"]):
        want[r["admit_us"] // 10**6] = want.get(r["admit_us"] // 10**6, 0) + q["input"]
    got = {e["second"]: e["sample"] for e in d["ctrl_log"]}
    assert got == {s: v for s, v in want.items() if (s + 1) * 10**6 <= d["end_us"]}
    assert len(got) > 5


@pytest.mark.parametrize("max_batch", [3, 7])
def test_util_signal_is_mean_batch_occupancy(orc, max_batch):
    """NEXT-3 signal ("GPU utilization metrics"): the sample of second s is
    the mean decode-batch occupancy over the iteration ends in s, in basis
    points: floor(10000 sum(B) / (max_batch n)), B the number of requests
    emitting a decode word at an end.  Iteration ends and B are rebuilt from
    each request's first word and its TBT gaps."""
    reqs, prof, d = _signal_run(orc, W.SIG_UTIL, 11, max_batch)
    ends = {}
    for r, gaps in zip(d["requests"], d["gaps"]):
        t = r["first_us"]
        for g in gaps:
            t += g
            ends[t] = ends.get(t, 0) + 1
    per_sec = {}
    for t, b in ends.items():
        per_sec.setdefault(t // 10**6, []).append(b)
    got = {e["second"]: e["sample"] for e in d["ctrl_log"]}
    assert got == {s: 10000 * sum(v) // (max_batch * len(v)) for s, v in per_sec.items()
                   if (s + 1) * 10**6 <= d["end_us"]}
    assert len(got) > 5 and max(got.values()) > 10000 // max_batch


def test_bruteforce_kv_capacity(orc):
    """NEXT-4 KV-capacity admission vs the brute-force simulator on random tiny
    traces, with and without a constant rewrite rate."""
    rng = np.random.default_rng(21)
    for case in range(80):
        reqs, prof = _random_tiny(rng)
        prof["max_batch"] = int(rng.integers(2, 6))
        prof["knee"] = min(prof["knee"], prof["max_batch"])
        prof["kv_cap_words"] = int(rng.integers(20, 120))
        law = "const" if case % 2 else "off"
        rc = int(rng.integers(100, 3000)) if law == "const" else 0
        bf = bruteforce.simulate(reqs, prof, 10**6, law=law, r_const=rc)
        c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=rc) if law == "const" else None
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=10**6)
        assert d["ticks"] == bf["ticks"], case
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["first_us"], r["done_us"], r["R"]) == \
                   (bf["admit"][i], bf["first"][i], bf["done"][i], bf["R"][i]), (case, i)


def test_kv_capacity_invariant_and_fifo(orc):
    """At every instant the admitted contexts fit the capacity unless a single
    oversized request runs alone; admission order stays FIFO."""
    w = W.config_paper_pair(2)
    w.profiles[0] = dict(w.profiles[0], kv_cap_words=120_000)
    arr = orc.arrivals(w.columns(), 0)
    reqs = [dict(a_us=int(x["a_us"]), input=int(x["input"]), U=int(x["U"])) for x in arr]
    d = orc.simulate(reqs, w.profiles[0], mode=W.MODE_DRAIN)
    R = [r["R"] for r in d["requests"]]
    adm = [r["admit_us"] for r in d["requests"]]
    done = [r["done_us"] for r in d["requests"]]
    assert all(a <= b for a, b in zip(adm, adm[1:]))
    for i, t in enumerate(adm):  # just after each admission
        live = [k for k in range(len(reqs)) if adm[k] <= t < done[k]]
        used = sum(reqs[k]["input"] + R[k] for k in live)
        assert used <= 120_000 or len(live) == 1
    free = orc.simulate(reqs, dict(w.profiles[0], kv_cap_words=0), mode=W.MODE_DRAIN)
    assert d["sum_queue_us"] > free["sum_queue_us"]


# ---------------------------------------------------------------------------
# NEXT-4 contending prefill (S:257 flags prefill/decode contention as unmodelled;
# profile prefill_mode = 1): the requests admitted at an iteration boundary
# prefill inside the next iteration, which lasts cost(B) + their prefill times.

CONT = dict(LIT, prefill_mode=1)


def test_bruteforce_contending_prefill(orc):
    """Contending prefill: event-heap DES == microsecond brute force on random tiny traces."""
    rng = np.random.default_rng(23)
    for case in range(120):
        reqs, prof = _random_tiny(rng)
        prof["prefill_mode"] = 1
        law = "const" if case % 3 == 0 else "off"
        rc = int(rng.integers(100, 3000)) if law == "const" else 0
        if case % 4 == 1:
            prof["kv_cap_words"] = int(rng.integers(20, 120))
        bf = bruteforce.simulate(reqs, prof, 10**6, law=law, r_const=rc)
        c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=rc) if law == "const" else None
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=10**6)
        assert (d["ticks"], d["words_out"], d["end_us"], d["served"]) == \
               (bf["ticks"], bf["words_out"], bf["end_us"], bf["served"]), case
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["first_us"], r["done_us"], r["R"]) == \
                   (bf["admit"][i], bf["first"][i], bf["done"][i], bf["R"][i]), (case, i)
            assert d["gaps"][i] == bf["gaps"][i], (case, i)


def test_bruteforce_controller_contending(orc):
    """MAP controller in the loop with contending prefill vs brute force."""
    rng = np.random.default_rng(31)
    prof = dict(t0_us=20_000, knee=1, slope_us=9000, kv_ns_per_word=0, max_batch=4,
                prefill_ns_per_word=100_000, e_in=0.05, e_out=0.5, p_idle=300.0, prefill_mode=1)
    for case in range(5):
        reqs = []
        t = 0
        for i in range(14):
            t += int(rng.integers(0, 250_000))
            reqs.append(dict(a_us=t, input=int(rng.integers(1, 200)), U=int(rng.integers(2, 30)),
                             P=int(rng.integers(5, 40)), fcomp_q16=65536))
        t1, t2 = 25_000 + 4000 * case, 45_000 + 4000 * case
        bf = bruteforce.simulate(reqs, prof, 6_000_000, law="map", t1=t1, t2=t2)
        d = orc.simulate(reqs, prof, ctrl=orc.make_ctrl(law=W.LAW_MAP, t1=t1, t2=t2), mode=W.MODE_DRAIN,
                         horizon_us=6_000_000)
        assert d["ticks"] == bf["ticks"]
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["first_us"], r["done_us"], r["R"], r["r_bp"]) == \
                   (bf["admit"][i], bf["first"][i], bf["done"][i], bf["R"][i], bf["r_bp"][i]), (case, i)


def test_contending_prefill_spec_example_and_hand_timeline(orc):
    """S:207 (single request on an idle server: TTFT 800 ms, E2E 25,750 ms) holds
    under contention; and a hand-worked two-request timeline (spec-literal
    profile, 80 µs per input word): A (0 s, 1000 words in, 3 out), B (0.1 s, 500
    in, 2 out).  Contending: A prefills alone [0, 80 ms); A decodes [80, 130);
    B admitted at 130 and prefilled inside A's next iteration, 50 + 40 = 90 ms,
    so A's second gap is 90 ms and both A's last word and B's first word land at
    220 ms; B's word 2 at 270 ms.  Non-blocking, for contrast: B's prefill ends
    at 170 ms mid-iteration, A completes at 180 ms, B at 230 ms."""
    d = orc.simulate([dict(a_us=0, input=10_000, U=500)], CONT, mode=W.MODE_DRAIN)
    r = d["requests"][0]
    assert (r["first_us"], r["done_us"]) == (800_000, 25_750_000)
    reqs = [dict(a_us=0, input=1000, U=3), dict(a_us=100_000, input=500, U=2)]
    c = orc.simulate(reqs, CONT, mode=W.MODE_DRAIN)
    a, b = c["requests"]
    assert (a["admit_us"], a["first_us"], a["done_us"]) == (0, 80_000, 220_000)
    assert c["gaps"][0] == [50_000, 90_000]
    assert (b["admit_us"], b["first_us"], b["done_us"]) == (130_000, 220_000, 270_000)
    assert c["gaps"][1] == [50_000]
    assert c["ticks"] == 4  # the prefill-only iteration at 0 counts
    n = orc.simulate(reqs, LIT, mode=W.MODE_DRAIN)
    a, b = n["requests"]
    assert (a["done_us"], b["first_us"], b["done_us"]) == (180_000, 170_000, 230_000)
    assert n["gaps"][1] == [60_000]


def test_contending_gap_is_cost_plus_admitted_prefills(orc):
    """Closed form from the request log: with no batch slowdown (knee =
    max_batch) and no KV term, every decode gap under contention equals t0 plus
    the prefill times of the requests whose first word lands at the gap's end;
    and the mean TBT rises with the arrival rate (the load signal the paper's
    controller relies on), while it stays near t0 without contention."""
    prof = dict(CONT, knee=CONT["max_batch"], kv_ns_per_word=0)
    rng = np.random.default_rng(5)
    means = []
    for rate in (0.5, 1.0, 2.0, 3.0):
        reqs, t = [], 0
        for i in range(150):
            t += int(rng.exponential(1e6 / rate))
            reqs.append(dict(a_us=t, input=int(rng.integers(500, 6000)), U=int(rng.integers(5, 60))))
        d = orc.simulate(reqs, prof, mode=W.MODE_DRAIN)
        pf = [max(1, prof["prefill_ns_per_word"] * q["input"] // 1000) for q in reqs]
        first_at = {}
        for i, r in enumerate(d["requests"]):
            first_at.setdefault(r["first_us"], []).append(i)
        gaps = []
        for i, r in enumerate(d["requests"]):
            t = r["first_us"]
            for g in d["gaps"][i]:
                t += g
                assert g == prof["t0_us"] + sum(pf[j] for j in first_at.get(t, [])), (rate, i)
                gaps.append(g)
        means.append(sum(gaps) / len(gaps))
        nb = orc.simulate(reqs, dict(prof, prefill_mode=0), mode=W.MODE_DRAIN)
        assert nb["tbt_sum_us"] / nb["tbt_samples"] < 1.5 * prof["t0_us"]
    assert means == sorted(means) and means[-1] > 2 * means[0]


# ---------------------------------------------------------------------------
# NEXT-4 KV preemption (profile kv_policy = 1; SURVEY 8(f) f4 "KV-capacity
# admission and preemption"; S:255 keeps KV out of SPEC): vLLM-style recompute
# preemption.  Admission needs the head's current context (input + words
# emitted) to fit; at an iteration end whose contexts exceed kv_cap_words the
# latest admitted requests go back to the queue front (while more than one is
# in the system) and later prefill input + emitted again, the end of that
# prefill emitting their next word.
PRE = dict(t0_us=100, knee=4, slope_us=0, kv_ns_per_word=0, max_batch=4, prefill_ns_per_word=1000,
           e_in=0.05, e_out=0.5, p_idle=300.0, kv_cap_words=25, kv_policy=1)


def test_kv_preemption_hand_timeline(orc):
    """Two requests (input 10, 5 words each, cap 25 words, 1 µs prefill per
    word, 100 µs iterations), worked by hand: both admitted at 0 (contexts 10 +
    10), first words at 10; after the ends at 110 (contexts 12 + 12 = 24) and
    210 (13 + 13 = 26 > 25) the later admitted B goes back to the queue; B (13
    context words) fits only when A completes at 410; its recompute prefill
    ends at 423 with B's 4th word (gap 423 - 210), the 5th at 523."""
    reqs = [dict(a_us=0, input=10, U=5), dict(a_us=0, input=10, U=5)]
    d = orc.simulate(reqs, PRE, mode=W.MODE_DRAIN)
    a, b = d["requests"]
    assert (a["admit_us"], a["first_us"], a["done_us"]) == (0, 10, 410)
    assert (b["admit_us"], b["first_us"], b["done_us"]) == (0, 10, 523)
    assert d["gaps"][0] == [100, 100, 100, 100]
    assert d["gaps"][1] == [100, 100, 213, 100]
    assert (d["preemptions"], d["recompute_words"], d["sum_queue_us"]) == (1, 13, 200)
    assert (d["ticks"], d["words_in"], d["words_out"], d["served"], d["admitted"]) == (5, 33, 10, 2, 2)
    assert d["energy_j"] == (0.05 * 33 + 0.5 * 10) + 300.0 * 0 / 1e6
    # no preemption when the capacity holds both contexts to the end (or is unlimited)
    for cap in (30, 0):
        n = orc.simulate(reqs, dict(PRE, kv_cap_words=cap), mode=W.MODE_DRAIN)
        assert n["preemptions"] == 0 and [r["done_us"] for r in n["requests"]] == [410, 410]


def test_bruteforce_kv_preemption(orc):
    """KV preemption vs the brute-force simulator on random tiny traces (exact
    per request and per gap, preemption and recompute counts, queue stays)."""
    rng = np.random.default_rng(23)
    total = 0
    for case in range(120):
        reqs, prof = _random_tiny(rng)
        n = int(rng.integers(3, 9))  # a denser mix than _random_tiny: several contexts that grow
        reqs = sorted([dict(a_us=int(rng.integers(0, 3000)), input=int(rng.integers(1, 20)),
                            U=int(rng.integers(2, 16)), P=int(rng.integers(2, 16)),
                            fcomp_q16=int(rng.integers(50000, 80000))) for _ in range(n)], key=lambda q: q["a_us"])
        prof["max_batch"] = int(rng.integers(2, 7))
        prof["knee"] = min(prof["knee"], prof["max_batch"])
        prof["kv_cap_words"] = int(rng.integers(15, 60))
        prof["kv_policy"] = 1
        law = "const" if case % 2 else "off"
        rc = int(rng.integers(100, 3000)) if law == "const" else 0
        bf = bruteforce.simulate(reqs, prof, 10**6, law=law, r_const=rc)
        c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=rc) if law == "const" else None
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=10**6)
        assert (d["ticks"], d["words_out"], d["served"], d["end_us"]) == \
               (bf["ticks"], bf["words_out"], bf["served"], bf["end_us"]), case
        assert (d["preemptions"], d["recompute_words"], d["sum_queue_us"]) == \
               (bf["preemptions"], bf["recompute_words"], bf["sum_queue_us"]), case
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["first_us"], r["done_us"], r["R"]) == \
                   (bf["admit"][i], bf["first"][i], bf["done"][i], bf["R"][i]), (case, i)
            assert d["gaps"][i] == bf["gaps"][i], (case, i)
        total += d["preemptions"]
    assert total > 50  # the cases do exercise preemption


def test_kv_preemption_identities(orc):
    """On a congested paper-trace run under a tight capacity: requests are
    preempted, yet every admitted request completes with all R words (one gap
    per word after the first), the sample-path identities hold with preempted
    requests counted as queued (Little's law: sum of sojourns = integral of
    queue + system; sum of every queue stay = integral of the queue), and a
    capacity that never binds gives the run without a capacity."""
    w = W.config_paper_pair(1)
    arr = orc.arrivals(w.columns(), 0)
    reqs = [dict(a_us=int(x["a_us"]), input=int(x["input"]), U=int(x["U"])) for x in arr]
    prof = dict(w.profiles[0], kv_cap_words=200_000, kv_policy=1)
    d = orc.simulate(reqs, prof, mode=W.MODE_DRAIN)
    assert d["preemptions"] > 10 and d["recompute_words"] > 0
    assert d["served"] == d["admitted"] == len(reqs) and d["inflight_end"] == 0
    assert d["words_out"] == sum(r["R"] for r in d["requests"])
    assert all(r["n_gaps"] == r["R"] - 1 for r in d["requests"])
    assert d["sum_sojourn_us"] == d["int_system_us"]
    assert d["sum_queue_us"] == d["int_queue_us"]
    assert d["words_in"] == sum(q["input"] for q in reqs) + d["recompute_words"]
    big = orc.simulate(reqs, dict(prof, kv_cap_words=2**30), mode=W.MODE_DRAIN)
    free = orc.simulate(reqs, dict(prof, kv_cap_words=0), mode=W.MODE_DRAIN)
    assert big["preemptions"] == 0
    assert [r["done_us"] for r in big["requests"]] == [r["done_us"] for r in free["requests"]]


TPW13 = round(1.3 * 65536)  # R31 / S:249: 1.3 tokens per word


def test_token_costs_spec_example_in_tokens(orc):
    """NEXT-4 token-level costs (R44): S:207's single request (input 10,000
    words, R = 500 words) with 1.3 tokens per word is 13,000 input tokens and 650
    output tokens: prefill 13,000 x 80 µs = 1.04 s, 649 decode iterations of
    50 ms, E2E = 1,040,000 + 649 x 50,000 µs; energy 0.05 x 13,000 + 0.5 x 650."""
    prof = dict(LIT, tpw_q16=TPW13)
    d = orc.simulate([dict(a_us=0, input=10_000, U=500)], prof, mode=W.MODE_DRAIN)
    r = d["requests"][0]
    assert r["first_us"] == 1_040_000 and r["R"] == 650
    assert r["done_us"] == 1_040_000 + 649 * 50_000
    assert d["ticks"] == 649 and d["words_in"] == 13_000 and d["words_out"] == 650
    assert d["energy_j"] == 0.05 * 13_000 + 0.5 * 650
    # rounding: 1 word -> round(1.3) = 1 token; 5 words -> round(6.5) = 7 (half up); tpw 0.25: 1 word -> 1
    d = orc.simulate([dict(a_us=0, input=5, U=1)], dict(LIT, tpw_q16=TPW13), mode=W.MODE_DRAIN)
    assert d["words_in"] == 7 and d["requests"][0]["R"] == 1
    d = orc.simulate([dict(a_us=0, input=1, U=1)], dict(LIT, tpw_q16=16384), mode=W.MODE_DRAIN)
    assert d["words_in"] == 1


def test_token_costs_identities(orc):
    """tpw = 1.0 (65536) is byte-identical to the word engine (tpw = 0); and a
    run at tpw = 2.0 equals the word run with every input and unbounded
    length doubled (no rewriting), field by field and gap by gap."""
    rng = np.random.default_rng(41)
    reqs = []
    t = 0
    for _ in range(200):
        t += int(rng.integers(0, 200_000))
        reqs.append(dict(a_us=t, input=int(rng.integers(100, 3000)), U=int(rng.integers(2, 60)),
                         P=int(rng.integers(2, 60))))
    P24 = dict(W.PROFILES["P24"], max_batch=8, kv_ns_per_word=30)
    c = orc.make_ctrl(law=W.LAW_MAP, t1=22_000, t2=30_000)
    a = orc.simulate(reqs, P24, ctrl=c, mode=W.MODE_DRAIN)
    b = orc.simulate(reqs, dict(P24, tpw_q16=65536), ctrl=c, mode=W.MODE_DRAIN)
    for k in orc.SUMMARY_FIELDS:
        assert a[k] == b[k], k
    assert a["gaps"] == b["gaps"] and a["rewritten"] > 0
    dbl = [dict(q, input=2 * q["input"], U=2 * q["U"]) for q in reqs]
    w = orc.simulate(dbl, P24, mode=W.MODE_DRAIN)
    x = orc.simulate(reqs, dict(P24, tpw_q16=131072), mode=W.MODE_DRAIN)
    for k in ("ticks", "served", "words_in", "words_out", "end_us", "idle_us", "sum_e2e_us", "sum_ttft_us",
              "sum_queue_us", "e2e_p50_ms", "e2e_p99_ms", "energy_j"):
        assert w[k] == x[k], k
    assert w["gaps"] == x["gaps"]


def test_bruteforce_token_costs(orc):
    """Token-level costs in the loop (rewrite in words, decode in tokens) vs the
    brute-force simulator, with KV capacity and a MAP controller."""
    rng = np.random.default_rng(43)
    for case in range(60):
        reqs, prof = _random_tiny(rng)
        prof["tpw_q16"] = int(rng.choice([16384, 50000, TPW13, 131072, 262144]))
        if case % 2:
            prof["kv_cap_words"] = int(rng.integers(20, 200))
        law = "const" if case % 3 == 0 else "off"
        rc = int(rng.integers(100, 3000)) if law == "const" else 0
        bf = bruteforce.simulate(reqs, prof, 10**6, law=law, r_const=rc)
        c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=rc) if law == "const" else None
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=10**6)
        assert (d["ticks"], d["words_out"], d["end_us"], d["served"]) == \
               (bf["ticks"], bf["words_out"], bf["end_us"], bf["served"]), case
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["first_us"], r["done_us"], r["R"]) == \
                   (bf["admit"][i], bf["first"][i], bf["done"][i], bf["R"][i]), (case, i)
            assert d["gaps"][i] == bf["gaps"][i], (case, i)

"""Pins for the multi-replica DES (NEXT-4, reading R45; "the request
scheduler picks requests from the arrival queue and assigns to GPU servers").

* one replica through orc_simulate_replicas is orc_simulate, field by field;
* a hand-worked two-replica timeline where least-loaded and round-robin
  routing differ (tests/golden is not needed: the timeline is in the test);
* the brute-force microsecond simulator (tests/bruteforce.simulate_replicas)
  on random tiny traces, both policies, with a controller in the loop.
"""
import numpy as np
import pytest

import workloads as W
from tests import bruteforce

LIT = W.PROFILES["spec-literal"]


def _stream(rng, n, gap, inp=(100, 3000), U=(2, 40)):
    reqs, t = [], 0
    for _ in range(n):
        t += int(rng.integers(0, gap))
        reqs.append(dict(a_us=t, input=int(rng.integers(*inp)), U=int(rng.integers(*U)),
                         P=int(rng.integers(*U)) + 3, fcomp_q16=int(rng.integers(60000, 70000)),
                         qnoise=int(rng.integers(-300, 300))))
    return reqs


@pytest.mark.parametrize("seed", range(4))
def test_one_replica_is_the_single_engine(orc, seed):
    rng = np.random.default_rng(100 + seed)
    reqs = _stream(rng, 200, 120_000)
    prof = dict(W.PROFILES["L8B"] if seed % 2 else W.PROFILES["P24"], max_batch=int(rng.integers(1, 12)))
    prof["knee"] = min(prof["knee"], prof["max_batch"])
    ctrls = [None, orc.make_ctrl(law=W.LAW_MAP, t1=24_000, t2=40_000),
             orc.make_ctrl(law=W.LAW_STEP, t1=24_000, t2=40_000, rungs=(500, 1000, 2000)),
             orc.make_ctrl(law=W.LAW_PCC, t1=24_000, w_lat=1, w_q=4, step_bp=250)]
    c = ctrls[seed]
    a = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, record=2)
    b = orc.simulate(reqs, dict(prof, replicas=1), ctrl=c, mode=W.MODE_DRAIN, record=2, multi=True)
    for k in orc.SUMMARY_FIELDS + orc.RESULT_EXTRA:
        assert a[k] == b[k], k
    assert a["requests"] == b["requests"] and a["gaps"] == b["gaps"] and a["ctrl_log"] == b["ctrl_log"]


@pytest.mark.parametrize("route,a_done", [(0, 130_000), (1, 178_000)])
def test_two_replica_hand_timeline(orc, route, a_done):
    """spec-literal cost (50 ms iterations), 2 replicas x 2 slots, prefill 80 µs/word.
    A (t=0, 1000 words in, R=2) -> replica 0 (tie -> lowest; RR pointer 0).
    B (t=10, 100 in, R=1) -> replica 1 (fewer in system; RR pointer 1); done at 8,010.
    C (t=20,000, 100 in, R=3): both replicas idle, A still prefilling, loads (1, 0):
      least loaded -> replica 1: C words at 28,000 / 78,000 / 128,000; A first word
        80,000 on its own replica, iteration [80,000, 130,000]: A done 130,000;
      round robin (pointer 0) -> replica 0: C iterates [28,000, 78,000, 128,000];
        A's first word at 80,000 lands mid-iteration and joins at 128,000:
        A done 178,000 (gap 98,000).  C done 128,000 either way."""
    prof = dict(LIT, max_batch=2, knee=2, replicas=2, route=route)
    reqs = [dict(a_us=0, input=1000, U=2), dict(a_us=10, input=100, U=1), dict(a_us=20_000, input=100, U=3)]
    d = orc.simulate(reqs, prof, mode=W.MODE_DRAIN)
    A, B, C = d["requests"]
    assert (A["first_us"], A["done_us"]) == (80_000, a_done)
    assert (B["first_us"], B["done_us"]) == (8_010, 8_010)
    assert (C["admit_us"], C["first_us"], C["done_us"]) == (20_000, 28_000, 128_000)
    assert d["gaps"][0] == [a_done - 80_000] and d["gaps"][2] == [50_000, 50_000]
    assert d["ticks"] == 3 and d["served"] == 3


@pytest.mark.parametrize("route", [0, 1])
def test_bruteforce_replicas(orc, route):
    rng = np.random.default_rng(200 + route)
    for case in range(40):
        n = int(rng.integers(1, 9))
        reqs = sorted([dict(a_us=int(rng.integers(0, 3000)), input=int(rng.integers(1, 40)),
                            U=int(rng.integers(1, 9)), P=int(rng.integers(1, 12)),
                            fcomp_q16=int(rng.integers(50000, 80000))) for _ in range(n)], key=lambda q: q["a_us"])
        NR = int(rng.integers(1, 5))
        prof = dict(t0_us=int(rng.integers(1, 300)), knee=0, slope_us=int(rng.integers(0, 90)),
                    kv_ns_per_word=int(rng.integers(0, 3000)), max_batch=int(rng.integers(1, 4)),
                    prefill_ns_per_word=int(rng.integers(0, 40_000)), e_in=0.05, e_out=0.5, p_idle=300.0,
                    replicas=NR, route=route, tpw_q16=int(rng.choice([0, 85197])))
        law = "const" if case % 3 == 0 else "off"
        rc = int(rng.integers(100, 3000)) if law == "const" else 0
        bf = bruteforce.simulate_replicas(reqs, prof, 10**6, law=law, r_const=rc)
        c = orc.make_ctrl(law=W.LAW_CONST, r_const_bp=rc) if law == "const" else None
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=10**6, multi=True)
        assert (d["ticks"], d["served"], d["end_us"]) == (bf["ticks"], bf["served"], bf["end_us"]), case
        for i in range(n):
            r = d["requests"][i]
            assert (r["admit_us"], r["first_us"], r["done_us"], r["R"]) == \
                   (bf["admit"][i], bf["first"][i], bf["done"][i], bf["R"][i]), (case, i)
            assert d["gaps"][i] == bf["gaps"][i], (case, i)


def test_bruteforce_replicas_controller(orc):
    """Controller in the loop (MAP and MPC on the TBT of all replicas) over
    several seconds: same admissions, lengths and r per request."""
    rng = np.random.default_rng(211)
    for case in range(6):
        reqs = []
        t = 0
        for _ in range(24):
            t += int(rng.integers(0, 150_000))
            reqs.append(dict(a_us=t, input=int(rng.integers(1, 100)), U=int(rng.integers(2, 30)),
                             P=int(rng.integers(5, 40)), fcomp_q16=65536))
        prof = dict(t0_us=20_000, knee=1, slope_us=9000, kv_ns_per_word=0, max_batch=2, prefill_ns_per_word=1000,
                    e_in=0.05, e_out=0.5, p_idle=300.0, replicas=2 + case % 3, route=case % 2)
        t1 = 22_000 + 1000 * case
        if case % 2:
            kw = dict(law="mpc", t1=t1, horizon_s=2, w_lat=3, w_q=1, w_osc=1, window=3)
            c = orc.make_ctrl(law=W.LAW_MPC, t1=t1, window=3, horizon_s=2, w_lat=3, w_q=1, w_osc=1)
        else:
            kw = dict(law="map", t1=t1, t2=t1 + 15_000)
            c = orc.make_ctrl(law=W.LAW_MAP, t1=t1, t2=t1 + 15_000)
        bf = bruteforce.simulate_replicas(reqs, prof, 8_000_000, **kw)
        d = orc.simulate(reqs, prof, ctrl=c, mode=W.MODE_DRAIN, horizon_us=8_000_000)
        assert d["ticks"] == bf["ticks"], case
        for i in range(len(reqs)):
            r = d["requests"][i]
            assert (r["admit_us"], r["done_us"], r["R"], r["r_bp"]) == \
                   (bf["admit"][i], bf["done"][i], bf["R"][i], bf["r_bp"][i]), (case, i)


def test_replicas_raise_capacity(orc):
    """Sanity of the routing model: at the same per-replica batch, 4 replicas
    serve a stream that saturates one replica with far lower queueing."""
    rng = np.random.default_rng(7)
    reqs = _stream(rng, 400, 200_000)
    prof = dict(W.PROFILES["P24"], max_batch=4)
    one = orc.simulate(reqs, prof, mode=W.MODE_DRAIN)
    four = orc.simulate(reqs, dict(prof, replicas=4), mode=W.MODE_DRAIN)
    assert one["served"] == four["served"] == 400
    assert four["sum_queue_us"] * 4 < one["sum_queue_us"]

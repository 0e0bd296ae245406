"""Pins for the oracle's random-number layer (a2, a3; readings R32, R33).

Each pin is external to the oracle: published known-answer vectors, libm,
a 50-digit Decimal evaluation, and distributional closed forms.
"""
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest
from scipy import stats

import workloads as W


# Random123 philox4x32-10 known-answer vectors (kat_vectors, Salmon et al. SC'11).
KATS = [
    ((0, 0), (0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF,) * 4, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0xA4093822, 0x299F31D0), (0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("key,ctr,out", KATS)
def test_philox_kat(orc, key, ctr, out):
    assert orc.philox(key[0], key[1], ctr) == out


def test_log2_table_vs_decimal(orc):
    """T[i] = round(2^32 log2(1 + i/4096)) checked against 50-digit Decimal arithmetic."""
    getcontext().prec = 50
    ln2 = Decimal(2).ln()
    two32 = Decimal(2) ** 32
    for i in list(range(0, 4097, 1)):
        exact = (Decimal(1) + Decimal(i) / Decimal(4096)).ln() / ln2 * two32
        want = int((exact + Decimal("0.5")).to_integral_value(rounding="ROUND_FLOOR"))
        assert orc.log2_table(i) == want, i


def test_neglog_vs_libm(orc):
    """-ln U within the interpolation bound of libm for U = (2u+1)/2^33 (R33).

    Linear interpolation of log2(1+x) on cells of width h = 2^-12 errs by at most
    h^2/(8 ln 2) = 1.07e-8 in log2 units = 46 Q32 LSB of log2, i.e. 32 LSB of ln;
    plus table rounding (0.35 LSB) and final truncation (1 LSB): <= 34 LSB absolute."""
    rng = np.random.default_rng(0)
    us = list(rng.integers(0, 2**32, 20000, dtype=np.uint64)) + [0, 1, 2**31 - 1, 2**31, 2**32 - 2, 2**32 - 1]
    for u in us:
        u = int(u)
        U = (2 * u + 1) / 2**33
        want = -math.log(U) * 2**32
        got = orc.neglog_q32(u)
        assert abs(got - want) <= 34.0 + 1e-12 * want, (u, got, want)


def test_neglog_special_points(orc):
    # U = (2^32 + 1)/2^33 = 0.5 + 2^-33: -ln U = ln 2 - 2^-32 + O(2^-66)
    assert abs(orc.neglog_q32(2**31) - 2977044471) <= 2
    # u = 0 is the smallest U = 2^-33: -ln U = 33 ln 2
    assert abs(orc.neglog_q32(0) - 33 * 2977044472) <= 40


def test_neglog_monotone(orc):
    """-ln U is non-increasing in u (sampled densely incl. every table boundary)."""
    prev = None
    for e in range(0, 32):
        base = 1 << e
        for k in range(0, 64):
            u = base + (k * base) // 64 if e > 6 else base + k
            if u >= 2**32:
                continue
            v = orc.neglog_q32(u)
            if prev is not None and u > prev[0]:
                assert v <= prev[1], (u, v, prev)
            prev = (u, v)


def test_exponential_interarrivals(orc):
    """Constant-rate trace: inter-arrival mean within 5% of 1/lambda over >=1000
    events and a KS test against Exp(lambda) (P:183 'inter-arrival times
    follow an exponential distribution')."""
    for rps in (0.5, 2.5, 8.0):
        n = 1
        w = W.custom([W.const_trace(rps, 4000)], ["P24"], [W.OFF],
                     [W.Scenario(7, wid=0, trace=0, profile=0, ctrl=0, segment=0, mode=0, horizon_us=10)])
        arr = orc.arrivals(w.columns(), 0)
        a = arr["a_us"].astype(np.float64) / 1e6
        assert len(a) >= 1000
        gaps = np.diff(np.concatenate([[0.0], a]))
        assert abs(gaps.mean() * rps - 1.0) < 0.05
        assert stats.kstest(gaps, "expon", args=(0, 1 / rps)).pvalue > 1e-3
        # constant rate: every candidate is accepted (lambda(tau) = lambda_max)
        assert list(arr["j"]) == list(range(len(arr)))
        n += 1


def _arrivals(orc, knots, seed=0, cap=0):
    w = W.custom([(knots, cap)], ["P24"], [W.OFF],
                 [W.Scenario(seed, wid=0, trace=0, profile=0, ctrl=0, segment=0, mode=0, horizon_us=10)])
    return orc.arrivals(w.columns(), 0)


def test_trace_examples(orc):
    # phase (90 s, 2.5 RPS) -> 165..285 events
    for seed in range(5):
        n = len(_arrivals(orc, W.const_trace(2.5, 90), seed))
        assert 165 <= n <= 285
    # zero rate -> 0 events
    assert len(_arrivals(orc, W.const_trace(0.0, 60))) == 0
    # two phases -> phase-2 events are >= the phase-1 duration; sorted, unique ids
    knots = [(0, 1000), (30 * W.US, 1000), (30 * W.US, 3000), (60 * W.US, 3000)]
    a = _arrivals(orc, knots, 3)
    assert np.all(np.diff(a["a_us"].astype(np.int64)) >= 0)
    assert len(set(a["j"])) == len(a)
    # arrival cap (R28)
    assert len(_arrivals(orc, W.const_trace(2.5, 600), 0, cap=100)) == 100


def test_paper_trace_plateaus(orc):
    """realized plateau rates within 15% of 2.5 and 1.5 RPS over 20 seeds
    (P:183 'two peaks of 2.5 RPS ... and 1.5 RPS'); duration 1,320 s."""
    knots = W.paper_trace()
    assert knots[-1][0] == 1_320_000_000
    c1, c2 = 0, 0
    for seed in range(20):
        a = _arrivals(orc, knots, seed)["a_us"]
        c1 += np.sum((a >= 60 * W.US) & (a < 150 * W.US))
        c2 += np.sum((a >= 900 * W.US) & (a < 960 * W.US))
    assert abs(c1 / (20 * 90) / 2.5 - 1) < 0.15
    assert abs(c2 / (20 * 60) / 1.5 - 1) < 0.15


def test_ramp_thinning_rate(orc):
    """A 0 -> 4 RPS linear ramp over 1000 s has Lambda = 2000 expected events;
    the first and second halves hold 1/4 and 3/4 of them (exact thinning)."""
    knots = [(0, 0), (1000 * W.US, 4000)]
    tot, first = 0, 0
    for seed in range(10):
        a = _arrivals(orc, knots, seed)["a_us"]
        tot += len(a)
        first += np.sum(a < 500 * W.US)
    assert abs(tot / 10 / 2000 - 1) < 0.03
    assert abs(first / tot - 0.25) < 0.02

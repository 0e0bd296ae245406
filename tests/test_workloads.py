"""Pins for the input module (workload distributions are model inputs)."""
import math

import numpy as np

import workloads as W


def test_tables_moments():
    t = W.quantile_tables()
    L = t["L"].astype(np.float64)
    assert abs(L.mean() - 500) < 1 and abs(L.std() - 80) < 2          # S:84 Normal(500, 80)
    assert L.min() >= 100 and L.max() <= 1200
    noise = t["noise"].astype(np.float64)
    assert abs(np.abs(noise).mean() - 36) < 2                          # P:110 MAE 36 (A7)
    assert abs(noise.mean()) <= 1.5                                    # S:156 unbiased
    f = t["fvar"] / 65536.0
    assert f.min() >= 0.75 - 1e-4 and f.max() <= 1.38 + 1e-4             # P:97 band (R14)
    assert abs(np.median(f) - 1.0) < 1e-3
    I = t["I"].astype(np.float64)
    assert 2000 <= I.min() and I.max() <= 20000 and abs(np.median(I) - 9000) < 30
    c = t["fcomp"] / 65536.0
    assert abs(c.mean() - 1) < 1e-3 and abs(c.std() - 0.05) < 2e-3     # S:163 rel_noise 0.05


def test_configs_shapes():
    assert W.config_c1().n_scenarios == 2
    w2 = W.config_c2()
    assert w2.n_scenarios == 2048 and w2.n_segments == 32
    w3 = W.config_c3()
    assert w3.n_scenarios == 32 * 321
    c = w2.columns()
    assert c["sc_seed"].dtype == np.uint32 and len(c["sc_seed"]) == 2048
    # ON and OFF of the same (rate, seed) share the workload id (common random numbers, R32)
    assert c["sc_wid"][0] == c["sc_wid"][64] and c["sc_seed"][0] == c["sc_seed"][64]


def test_paper_trace_knots():
    k = W.paper_trace()
    assert k[0] == (0, 0) and k[-1][0] == 1320 * W.US
    assert dict(k)[60 * W.US] == 2500 and dict(k)[900 * W.US] == 1500
    for v in range(3):
        d = W.diurnal_trace(v)
        ts = [t for t, _ in d]
        assert ts == sorted(ts) and len(set(ts)) == len(ts) and ts[-1] == 86400 * W.US
        assert max(l for _, l in d) <= 3500 and min(l for _, l in d) >= 400


def test_shard_partition():
    for world in (1, 2, 3, 8):
        ids = np.concatenate([W.shard(1000, r, world) for r in range(world)])
        assert sorted(ids.tolist()) == list(range(1000))

"""GPU parity of K2L, the lane-per-scenario kernel (bellman_lane.cu), vs the
CPU oracle on the small configurations and edge cases, by forcing K2L on
every run (BELLMAN_LANE=2; by default only runs of >= 65,536 scenarios take
it, so C1-C4 exercise the warp engine and C5 the lane engine).  Also: the
warp engine alone (BELLMAN_LANE=0) on a C5 subset, and the same records from
both engines.

Bar as in test_gpu_parity: bit-exact integers and histograms, fp64 energy
within 1e-9 relative."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests import test_gpu_parity as G
from tests.parity import check_all, compare, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture
def lane(monkeypatch):
    monkeypatch.setenv("BELLMAN_LANE", "2")


def _ok(bad):
    assert not bad, "\n".join(f"scenario {sid}: {e}" for sid, e in bad[:10])


def test_lane_c1(lane):
    bad, st = check_all(W.config_c1().columns())
    _ok(bad)
    assert st[1]["activations"] >= 1


def test_lane_c2_full_every_record(lane):
    """C2 (L8B: the KV-term instantiation), all 2,048 records and segment histograms."""
    bad, _ = check_all(W.config_c2().columns())
    _ok(bad)


def test_lane_c3_reduced(lane):
    bad, _ = check_all(W.config_c3(n_seeds=2).columns())
    _ok(bad)


def test_lane_c5_reduced(lane):
    bad, _ = check_all(W.config_c5(n_seeds=4).columns())
    _ok(bad)


def test_lane_edge_cases(lane):
    """K2L's scenarios of the edge workload (the rest run in the warp engines of
    the same launch set): ragged max_batch, empty traces, caps, 1-µs prefills
    and iterations, every law / signal, degenerate calibration."""
    bad, st = check_all(G._edge_workload().columns())
    _ok(bad)


def test_lane_short_outputs(lane):
    G.test_short_outputs_and_tiny_tables()


@pytest.mark.parametrize("poly", [(-(1 << 20), 70_000, 3), (0, 32_768, 512), (5 << 16, -(1 << 14), 1 << 8)])
def test_lane_rewrite_polynomial_paths(lane, poly):
    G.test_rewrite_polynomial_paths(poly)


def test_lane_sharded_runs_match_single_run(lane):
    G.test_sharded_runs_match_single_run()


def test_lane_and_warp_engines_agree(monkeypatch):
    """A C5 subset through each engine: identical record bytes."""
    cols = W.config_c5(n_seeds=2).columns()
    monkeypatch.setenv("BELLMAN_LANE", "0")
    a, ha, _ = run_gpu(cols, per_scenario_segments=True)
    monkeypatch.setenv("BELLMAN_LANE", "2")
    b, hb, _ = run_gpu(cols, per_scenario_segments=True)
    assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    assert np.array_equal(ha, hb)
    sids = np.arange(0, len(cols["sc_seed"]), 37, dtype=np.uint64)
    rs = oracle.run_batch(oracle.Bound(cols), sids)
    _ok([(int(s), e) for s, o in zip(sids, rs) for e in [compare(b[int(s)], o, int(s))] if e])

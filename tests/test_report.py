"""NEXT-1 reporting layer (paper_2510_15330_b200/report.py) on oracle-produced
per-second rows: SPEC's compare_runs examples and the partition
properties of aggregate_per_second."""
import numpy as np
import pytest

import oracle
import workloads as W
from paper_2510_15330_b200 import report


def _sec(completions, energy, e2e=None):
    return dict(second=0, rps_in=0, queue_depth=0, avg_queueing_ms=None, avg_ttft_ms=None, avg_tbt_ms=None,
                avg_e2e_ms=e2e, active_r=0.0, completions=completions, energy_j=energy)


def test_compare_runs_spec_examples():
    # S:394 window completions 100 vs 119 -> +19.0 %; S:395 energies 1000 vs 750 -> -25.0 %
    u = [_sec(100, 1000.0, 8000.0)]
    b = [_sec(119, 750.0, 1000.0)]
    c = report.compare_runs(u, b, (0, 1))
    assert c.completions_delta_pct == pytest.approx(19.0)
    assert c.energy_delta_pct == pytest.approx(-25.0)
    assert c.e2e_peak_ratio == pytest.approx(8.0)
    # S:396 self-comparison -> zero deltas, ratio 1
    s = report.compare_runs(u, u, (0, 1))
    assert s.completions_delta_pct == 0 and s.energy_delta_pct == 0 and s.e2e_peak_ratio == 1
    # S:463 window beyond the horizon -> validation error
    with pytest.raises(ValueError):
        report.compare_runs(u, b, (5, 9))


def _ctrl_arr(log):
    dt = [("second", "<u4"), ("sample", "<u4"), ("k", "<u4"), ("r_bp", "<u4"), ("active", "<u4"), ("_pad", "<u4"),
          ("A", "<u8")]
    return np.array([(c["second"], c["sample"], c["k"], c["r_bp"], c["active"], 0, c["A"]) for c in log], dtype=dt)


def test_aggregate_partitions_totals():
    """per-second completions and energy partition the run totals; S:238
    conservation: queue depth never negative and ends at queued_end."""
    w = W.config_paper_pair(1)
    cols = w.columns()
    for sid in range(2):
        o = oracle.run_scenario(cols, sid, rows_cap=3000, ctrl_log_cap=3000)
        agg = report.aggregate_per_second(o["rows"], _ctrl_arr(o["ctrl_log"]), W.PROFILES["P24"])
        assert sum(a["completions"] for a in agg) == o["served"]
        assert sum(a["rps_in"] for a in agg) == o["arrivals"]
        assert sum(a["energy_j"] for a in agg) == pytest.approx(o["energy_j"], rel=1e-9)
        assert min(a["queue_depth"] for a in agg) >= 0 and agg[-1]["queue_depth"] == o["queued_end"]
        assert int(o["rows"]["tbt_count"].sum()) == o["tbt_samples"]
        assert int(o["rows"]["sum_tbt_us"].sum()) == o["tbt_sum_us"]
        if sid == 1:  # r in force follows the controller log, in {0} U [5 %, 20 %]
            assert all(a["active_r"] == 0 or 0.05 <= a["active_r"] <= 0.20 for a in agg)


def test_headline_report_runs():
    """A4 evaluated on the paper pair; directional, parity unpinned
    (DESIGN.md §6): only the invariant parts are asserted here."""
    w = W.config_paper_pair(0)
    cols = w.columns()
    u = oracle.run_scenario(cols, 0, rows_cap=3000)
    b = oracle.run_scenario(cols, 1, rows_cap=3000, ctrl_log_cap=3000)
    h = report.headline(u["rows"], b["rows"], _ctrl_arr(b["ctrl_log"]), b, W.PROFILES["P24"])
    assert h["checks"]["b_median_r_in_5_20pct"]
    assert h["checks"]["e_window_energy_bounded_lt_unbounded"]
    assert h["activation_s"] is not None


def test_active_r_applies_from_the_next_second():
    """the controller row of second s is ingested when s closes (R21),
    so its r governs second s + 1: active_r is 0 through the first activation
    second and equals that row's r from first_act_s + 1."""
    w = W.config_paper_pair(1)
    cols = w.columns()
    o = oracle.run_scenario(cols, 1, rows_cap=3000, ctrl_log_cap=3000)
    log = o["ctrl_log"]
    agg = report.aggregate_per_second(o["rows"], _ctrl_arr(log), W.PROFILES["P24"])
    fa = o["first_act_s"]
    first = next(c for c in log if c["active"])
    assert first["second"] == fa
    assert all(a["active_r"] == 0 for a in agg[: fa + 1])
    assert agg[fa + 1]["active_r"] == pytest.approx(first["r_bp"] / 1e4)

"""NEXT-4 trace files and replay."""
import os

import numpy as np
import pytest

import workloads as W


def test_trace_file_examples(tmp_path):
    # S:71 empty trace -> header only, round-trips to empty
    p = tmp_path / "e.csv"
    W.write_trace(p, [])
    assert open(p).read().strip() == W.TRACE_HEADER and W.read_trace(p) == []
    # S:72 three events -> three data lines, round-trip equality
    ev = [(0, 0, 9000, 500, 0), (1, 1500, 120, 60, 2), (2, 1500, 20000, 1200, 1)]
    W.write_trace(p, ev, comments=["seed 7"])
    assert len(open(p).read().strip().splitlines()) == 5 and W.read_trace(p) == ev
    # S:73 arrival_ms decreasing between lines 4 and 5 -> error citing line 5
    with open(p, "w") as f:
        f.write(W.TRACE_HEADER + "\n0,0,1,1,summarization\n1,5,1,1,coding\n2,9,1,1,coding\n3,7,1,1,coding\n")
    with pytest.raises(W.TraceFormatError, match="line 5"):
        W.read_trace(p)
    # S:69 malformed line names the line
    with open(p, "w") as f:
        f.write(W.TRACE_HEADER + "\n0,0,1,1,summarization\n1,x,1\n")
    with pytest.raises(W.TraceFormatError, match="line 3"):
        W.read_trace(p)


def test_replay_of_generated_arrivals_reproduces_the_run(orc, tmp_path):
    """With draw-neutral tables (Fvar = 1, no predictor or compliance noise) a
    replay of the generator's own arrivals — through a CSV file at ms
    resolution with ms-aligned arrivals — is the same run."""
    tabs = W.constant_tables()
    tabs["L"] = W.quantile_tables()["L"]
    tabs["I"] = W.quantile_tables()["I"]
    w = W.custom([W.const_trace(2.2, 400)], ["P24"], [W.OFF],
                 [W.Scenario(5, wid=0, trace=0, profile=0, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                             horizon_us=1200 * W.US)], tables=tabs)
    arr = orc.arrivals(w.columns(), 0)
    ms = [int(a) // 1000 for a in arr["a_us"]]
    ev = [(k, ms[k], int(arr["input"][k]), int(arr["L"][k]), 0) for k in range(len(arr))]
    p = tmp_path / "gen.csv"
    W.write_trace(p, ev)
    back = W.read_trace(p)
    rep = [(a * 1000, out, inp, cls) for _, a, inp, out, cls in back]
    # the Poisson run on the same ms-floored arrival times, via a replay of the exact list
    exact = [(m * 1000, int(arr["L"][k]), int(arr["input"][k]), 0) for k, m in enumerate(ms)]
    w2 = W.custom([{"replay": rep}, {"replay": exact}], ["P24"], [W.OFF],
                  [W.Scenario(5, wid=0, trace=t, profile=0, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                              horizon_us=1200 * W.US) for t in (0, 1)], tables=tabs)
    a = orc.run_scenario(w2.columns(), 0)
    b = orc.run_scenario(w2.columns(), 1)
    for k in orc.SUMMARY_FIELDS:
        assert a[k] == b[k], k
    # and with µs-exact arrivals the replay equals the generated run itself
    w3 = W.custom([W.const_trace(2.2, 400), {"replay": [(int(x["a_us"]), int(x["L"]), int(x["input"]), 0)
                                                        for x in arr]}], ["P24"], [W.OFF],
                  [W.Scenario(5, wid=0, trace=t, profile=0, ctrl=0, segment=0, mode=W.MODE_DRAIN,
                              horizon_us=1200 * W.US) for t in (0, 1)], tables=tabs)
    g = orc.run_scenario(w3.columns(), 0)
    r = orc.run_scenario(w3.columns(), 1)
    for k in ("ticks", "served", "words_out", "sum_e2e_us", "sum_ttft_us", "energy_j", "end_us", "idle_us"):
        assert g[k] == r[k], k

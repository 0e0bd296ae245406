"""Compute the fixed C2 controller thresholds from the oracle.

t1 / t2 = nearest-rank p50 / p75 of the per-second average-TBT samples pooled
over the 64 controller-OFF scenarios at 2.5 RPS (the paper picks "the median
TBT (T1) during the unbounded run" and "the 75th percentile TBT (T2)").
Calls only oracle/ and workloads/; prints the two integers that are frozen
into workloads.C2_T1_US / C2_T2_US.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import workloads as W  # noqa: E402


def main():
    w = W.config_c2(n_seeds=64, rates=[2.5])
    for s in w.scenarios:
        s.record = 1
    cols = w.columns()
    b = oracle.Bound(cols)
    pooled = []
    for sid, s in enumerate(w.scenarios):
        if w.ctrls[s.ctrl].law != W.LAW_OFF:
            continue
        r = oracle.run_scenario(b, sid, hist=False, series_cap=1000)
        pooled.extend(r["series"].tolist())
    st, t1, t2 = oracle.calibrate(np.asarray(pooled, dtype=np.uint32))
    print(f"samples={len(pooled)} status={st} C2_T1_US = {t1:_}  C2_T2_US = {t2:_}")


if __name__ == "__main__":
    main()

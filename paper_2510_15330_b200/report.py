"""Paper-headline reproduction layer: host post-processing
of debug-recorded runs.  Integer per-second rows and controller logs come from
the simulator (bellman_sim_series); this module only derives SPEC's reporting
quantities from them:

* aggregate_per_second: SecondAggregate rows with the columns of
  S:253 — rps_in, queue depth at the end of the second, average queueing /
  TTFT / TBT / E2E in ms (None when the denominator is 0), the r in force,
  completions, energy;
* compare_runs: RunComparison of an unbounded and a bounded run of
  the same trace and seed over a window;
* headline (acceptance A4): the paper's directional claims
  (activation 131 s, median r 8 %, up to 8x lower E2E, -25 % energy,
  +19 % served) evaluated on a pair.  Directional only — the
  paper's absolute values come from H100 hardware.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

US = 1_000_000


def aggregate_per_second(rows: np.ndarray, ctrl: np.ndarray | None, profile: dict) -> list[dict]:
    """SecondAggregate per second."""
    arr = rows["arrivals"].astype(np.int64)
    adm = rows["admitted"].astype(np.int64)
    depth = np.cumsum(arr) - np.cumsum(adm)
    r_at = np.zeros(len(rows), dtype=np.int64)
    if ctrl is not None and len(ctrl):
        cur, k = 0, 0
        order = list(ctrl)
        # the controller row of second s is ingested once s has closed, so its r
        # governs admissions from second s + 1 on (R21): row s is in force from s + 1
        for s in range(len(rows)):
            while k < len(order) and int(order[k]["second"]) < s:
                cur = int(order[k]["r_bp"])
                k += 1
            r_at[s] = cur

    def avg(num, den):
        return None if den == 0 else num / den / 1000.0

    out = []
    for s in range(len(rows)):
        r = rows[s]
        energy = (profile["e_in"] * float(r["words_in"]) + profile["e_out"] * float(r["words_out"])) + \
            profile["p_idle"] * float(r["idle_us"]) / 1e6
        out.append(dict(second=s, rps_in=int(r["arrivals"]), queue_depth=int(depth[s]),
                        avg_queueing_ms=avg(int(r["sum_queue_us"]), int(r["admitted"])),
                        avg_ttft_ms=avg(int(r["sum_ttft_us"]), int(r["first_tokens"])),
                        avg_tbt_ms=avg(int(r["sum_tbt_us"]), int(r["tbt_count"])),
                        avg_e2e_ms=avg(int(r["sum_e2e_us"]), int(r["completions"])),
                        active_r=r_at[s] / 1e4, completions=int(r["completions"]), energy_j=energy))
    return out


@dataclass
class RunComparison:
    """S:363-367."""
    window: tuple
    e2e_peak_ratio: float | None
    completions_unbounded: int
    completions_bounded: int
    completions_delta_pct: float | None
    energy_unbounded_j: float
    energy_bounded_j: float
    energy_delta_pct: float | None
    median_r_active: float | None


def compare_runs(unbounded: list[dict], bounded: list[dict], window: tuple, median_r_bp=None) -> RunComparison:
    """deltas in the window [start_s, end_s); the E2E ratio is peak
    per-second avg E2E unbounded / bounded within the window."""
    a, b = int(window[0]), int(window[1])
    if b <= a or a >= min(len(unbounded), len(bounded)):
        raise ValueError("window outside both runs (S:463)")
    U = unbounded[a:b]
    Bd = bounded[a:b]
    cu, cb = sum(x["completions"] for x in U), sum(x["completions"] for x in Bd)
    eu, eb = sum(x["energy_j"] for x in U), sum(x["energy_j"] for x in Bd)
    pu = max((x["avg_e2e_ms"] for x in U if x["avg_e2e_ms"] is not None), default=None)
    pb = max((x["avg_e2e_ms"] for x in Bd if x["avg_e2e_ms"] is not None), default=None)
    ratio = None if not pu or not pb else pu / pb
    med = None if median_r_bp in (None, 0xFFFFFFFF) else median_r_bp / 1e4
    return RunComparison((a, b), ratio, cu, cb, None if cu == 0 else (cb - cu) / cu * 100.0, eu, eb,
                         None if eu == 0 else (eb - eu) / eu * 100.0, med)


def headline(unb_rows, bnd_rows, bnd_ctrl, bnd_summary: dict, profile: dict, window=(130, 500)) -> dict:
    """Acceptance A4 on an unbounded / bounded pair of the same trace and seed."""
    U = aggregate_per_second(unb_rows, None, profile)
    Bd = aggregate_per_second(bnd_rows, bnd_ctrl, profile)
    cmp = compare_runs(U, Bd, window, bnd_summary.get("median_r_bp"))
    act = bnd_summary.get("first_act_s", 0xFFFFFFFF)
    deact = bnd_summary.get("last_deact_s", 0xFFFFFFFF)
    congested = [x["second"] for x in U if x["queue_depth"] > 10]
    last_cong = congested[-1] if congested else None
    return dict(
        activation_s=None if act == 0xFFFFFFFF else int(act),
        deactivation_s=None if deact == 0xFFFFFFFF else int(deact),
        unbounded_last_congested_s=last_cong,
        median_r=cmp.median_r_active,
        e2e_peak_ratio=cmp.e2e_peak_ratio,
        window=window,
        completions_delta_pct=cmp.completions_delta_pct,
        energy_delta_pct=cmp.energy_delta_pct,
        checks={
            "a_activation_in_90_200s": act != 0xFFFFFFFF and 90 <= act <= 200,
            "a_deactivation_before_unbounded_congestion_ends":
                deact != 0xFFFFFFFF and last_cong is not None and deact < last_cong,
            "b_median_r_in_5_20pct": cmp.median_r_active is not None and 0.05 <= cmp.median_r_active <= 0.20,
            "c_e2e_peak_ratio_ge_2": cmp.e2e_peak_ratio is not None and cmp.e2e_peak_ratio >= 2.0,
            "d_window_served_bounded_ge_unbounded": cmp.completions_bounded >= cmp.completions_unbounded,
            "e_window_energy_bounded_lt_unbounded": cmp.energy_bounded_j < cmp.energy_unbounded_j,
        },
    )

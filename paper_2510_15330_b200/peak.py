"""ctypes binding of include/bellman_peak.h: the integer issue / lane
microbenchmark behind the tick kernel's roofline (SURVEY §8(d) R_issue,
R_lane).  Measurement only; argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbellman_peak.so")


def measure(device: int = 0) -> dict:
    """Per SM per clock: warp-instructions and integer lanes of the alu pipe,
    the fma pipe, and both (alternating: the issue-port bound)."""
    lib = C.CDLL(LIB_PATH)
    lib.bellman_peak_int.argtypes = [C.c_int, C.POINTER(C.c_double)]
    lib.bellman_peak_int.restype = C.c_int
    out = (C.c_double * 6)()
    rc = lib.bellman_peak_int(device, out)
    if rc != 0:
        raise RuntimeError(f"bellman_peak_int failed: {rc}")
    return {"alu_warp_inst_per_clk_sm": out[0], "alu_lanes_per_clk_sm": out[1],
            "fma_warp_inst_per_clk_sm": out[2], "fma_lanes_per_clk_sm": out[3],
            "mixed_warp_inst_per_clk_sm": out[4], "mixed_lanes_per_clk_sm": out[5]}

"""B200-native beLLMan scenario simulator (arXiv 2510.15330).

The hot path — arrivals, per-request draws, continuous-batching decode
iterations, the word-limit controller, accounting, histograms and percentiles
— runs in hand-written sm_100a CUDA behind the C ABI of include/bellman_sim.h
(libbellman_sim.so).  This package is the thin Python binding.
"""
from . import _abi
from ._abi import STATS, SEG_HIST_WORDS, HIST_LAT, HIST_R, BellmanError
from .sim import Simulator, pack, stats_to_dicts, workspace_bytes

__all__ = ["Simulator", "pack", "stats_to_dicts", "workspace_bytes", "STATS", "SEG_HIST_WORDS", "HIST_LAT",
           "HIST_R", "BellmanError", "_abi"]

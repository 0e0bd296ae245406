"""Build libbellman_sim.so in-tree with nvcc for sm_100a (no torch extension)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libbellman_sim.so")
PEAK_OUT = os.path.join(HERE, "libbellman_peak.so")  # roofline microbenchmark (measurement only)
SOURCES = ["bellman_kernels.cu", "bellman_lane.cu", "bellman_host.cu"]
DEPS = SOURCES + ["bellman_internal.cuh", "bellman_lane.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build_peak(force: bool = False) -> str:
    src = os.path.join(CSRC, "bellman_peak.cu")
    hdr = os.path.join(os.path.dirname(HERE), "include", "bellman_peak.h")
    if not force and os.path.exists(PEAK_OUT) and all(os.path.getmtime(PEAK_OUT) >= os.path.getmtime(s)
                                                      for s in (src, hdr)):
        return PEAK_OUT
    cmd = [nvcc()] + [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")] + ["-o", PEAK_OUT, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    return PEAK_OUT


def build(force: bool = False, verbose: bool = False) -> str:
    build_peak(force)
    hdr = os.path.join(os.path.dirname(HERE), "include", "bellman_sim.h")
    srcs = [os.path.join(CSRC, s) for s in DEPS] + [hdr]
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(s) for s in srcs):
        return OUT
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", OUT] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stderr)
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    return OUT


if __name__ == "__main__":
    build(force=True, verbose=True)

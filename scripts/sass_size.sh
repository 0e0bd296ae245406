#!/bin/bash
# Static SASS size (instructions) per function of the tick kernel cubin.
# usage: scripts/sass_size.sh [extra nvcc flags...]
set -e
cd "$(dirname "$0")/.."
out=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -cubin -Iinclude "$@" \
  -o "$out/k.cubin" paper_2510_15330_b200/csrc/bellman_kernels.cu
cuobjdump -sass "$out/k.cubin" | awk '/Function :/ {f=$3} /^ +\/\*[0-9a-f]+\*\// {n[f]++} END {for (k in n) printf "%6d %s\n", n[k], k}' | sort -k2
rm -rf "$out"

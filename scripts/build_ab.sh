#!/bin/bash
# Development: build the library variant build/ab/lib_<name>.so with extra nvcc flags.
# usage: scripts/build_ab.sh <name> [extra nvcc flags...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/ab
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -shared -Iinclude "$@" \
  -o build/ab/lib_$name.so paper_2510_15330_b200/csrc/bellman_kernels.cu paper_2510_15330_b200/csrc/bellman_lane.cu paper_2510_15330_b200/csrc/bellman_host.cu
echo build/ab/lib_$name.so

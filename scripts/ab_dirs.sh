#!/bin/bash
# Development A/B across source trees (ABI changes allowed): alternate bench.py
# runs of build/old (a git worktree) and the current tree on the same box.
# usage (on the box): scripts/ab_dirs.sh <tag> [workload] [rounds]
set -u
cd "$(dirname "$0")/.."
tag=${1:-ab}; wl=${2:-C5}; n=${3:-2}
o=$PWD/gpurun_out; mkdir -p $o
for i in $(seq $n); do
  for d in build/old .; do
    (cd $d && timeout 600 python bench.py --workload $wl --no-cpu-baseline --e2e-steps 0 --no-peak --steps 5 --warmup 3 \
       2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', '$wl', round(d['kernel_ms_per_step'],3), d['ticks_per_step'])") | tee -a $o/${tag}.txt
  done
done

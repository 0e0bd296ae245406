#!/bin/bash
# quick GPU pass: the GPU suite (or a -k selection) and the C5 / C2 bench lines
# usage (on the box): scripts/gpu_quick.sh <tag> [pytest -k expr]
set -u
cd "$(dirname "$0")/.."
tag=${1:-q}
o=gpurun_out
mkdir -p $o
if [ -n "${2:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -k "$2" > $o/${tag}_pytest_gpu.txt 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $o/${tag}_pytest_gpu.txt 2>&1
fi
tail -3 $o/${tag}_pytest_gpu.txt
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $o/${tag}_bench_C5.json 2> $o/${tag}_bench_C5.err
python -c "import json,sys; d=json.load(open('$o/${tag}_bench_C5.json')); print('C5', d['value'], d['kernel_ms_per_step'], d['roofline']['frac'])"
timeout 600 python bench.py --workload C2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > $o/${tag}_bench_C2.json 2> $o/${tag}_bench_C2.err
python -c "import json,sys; d=json.load(open('$o/${tag}_bench_C2.json')); print('C2', d['value'], d['kernel_ms_per_step'], d['roofline']['frac'])"

#!/bin/bash
# One GPU-box pass that produces the round's measured evidence under gpurun_out/:
# GPU parity suite, compute-sanitizer, bench lines (C2 default, C5, reference
# arm), the ncu launch list of the C2 bench command and one ncu --set full
# capture of the tick kernel.  usage (on the box): scripts/round_measure.sh <tag>
set -u
cd "$(dirname "$0")/.."
tag=${1:-rXX}
o=gpurun_out
mkdir -p $o
python -m pytest tests -m gpu -q > $o/${tag}_pytest_gpu.txt 2>&1; tail -2 $o/${tag}_pytest_gpu.txt
python bench.py > $o/${tag}_bench_C2.json 2> $o/${tag}_bench_C2.err; tail -1 $o/${tag}_bench_C2.json
python bench.py --workload C5 --steps 5 --warmup 3 > $o/${tag}_bench_C5.json 2> $o/${tag}_bench_C5.err; tail -1 $o/${tag}_bench_C5.json
python bench.py --impl reference --steps 3 --warmup 3 > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err; tail -1 $o/${tag}_bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $o/${tag}_launches_bench.log 2>&1
python scripts/launch_summary.py $o/${tag}_launches.csv > $o/${tag}_launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:tick_kernel --launch-skip 3 --launch-count 1 -f \
  -o $o/${tag}_C2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $o/${tag}_ncu_full.log 2>&1
bash scripts/sanitize.sh > $o/${tag}_sanitizer.txt 2>&1; grep -c "ERROR SUMMARY: 0" $o/${tag}_sanitizer.txt

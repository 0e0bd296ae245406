#!/bin/bash
# One GPU-box pass that produces the round's measured evidence under gpurun_out/:
# GPU parity suite, smoke, bench lines (C5 default, C2, reference arm), the ncu
# launch list of the default bench command and ncu --set full captures of the
# tick kernel (the full C5 bench launch, a 1/16 C5 subset, the C2 bench launch).
# usage (on the box): scripts/round_measure.sh <tag> [skip-tests]
set -u
cd "$(dirname "$0")/.."
tag=${1:-rXX}
o=gpurun_out
mkdir -p $o
nproc > $o/${tag}_nproc.txt
if [ "${2:-}" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $o/${tag}_pytest_gpu.txt 2>&1; tail -2 $o/${tag}_pytest_gpu.txt
  python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.txt 2>&1; tail -1 $o/${tag}_smoke.txt
fi
timeout 900 python bench.py > $o/${tag}_bench_C5.json 2> $o/${tag}_bench_C5.err; tail -1 $o/${tag}_bench_C5.json
timeout 600 python bench.py --workload C2 --steps 20 --warmup 5 > $o/${tag}_bench_C2.json 2> $o/${tag}_bench_C2.err; tail -1 $o/${tag}_bench_C2.json
timeout 600 python bench.py --impl reference > $o/${tag}_bench_ref.json 2> $o/${tag}_bench_ref.err; tail -1 $o/${tag}_bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $o/${tag}_launches_bench.log 2>&1
python scripts/launch_summary.py $o/${tag}_launches.csv > $o/${tag}_launches.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tick_kernel|lane_kernel" --launch-skip 0 --launch-count 1 -f \
  -o $o/${tag}_C5 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-peak > $o/${tag}_ncu_C5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tick_kernel|lane_kernel" --launch-skip 1 --launch-count 1 -f \
  -o $o/${tag}_C5sub python scripts/run_lib_once.py paper_2510_15330_b200/libbellman_sim.so "W.config_c5(n_seeds=256)" \
  > $o/${tag}_ncu_C5sub.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tick_kernel --launch-skip 3 --launch-count 1 -f \
  -o $o/${tag}_C2 python bench.py --workload C2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-peak > $o/${tag}_ncu_C2.log 2>&1

for r in C5 C5sub C2; do python scripts/ncu_summary.py $o/${tag}_$r.ncu-rep > $o/${tag}_ncu_full_$r.txt 2>&1; done
python scripts/ncu_funcs.py $o/${tag}_C5.ncu-rep > $o/${tag}_ncu_funcs_C5.txt 2>&1
# compute-sanitizer (scripts/sanitize.sh) is closed on the GPU pool since r02p: not run here
echo done

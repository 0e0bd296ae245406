set -u
o=gpurun_out; mkdir -p $o; t=${1:-l2}
timeout 900 python -m pytest tests/test_gpu_lane.py -q -x > $o/${t}_pytest_lane.txt 2>&1; tail -3 $o/${t}_pytest_lane.txt
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > $o/${t}_bench_C5.json 2> $o/${t}_bench_C5.err
python -c "import json; d=json.load(open('$o/${t}_bench_C5.json')); print('C5', d['value'], d['kernel_ms_per_step'])"
if ls build/ab/*.so >/dev/null 2>&1; then AB_REPS=7 AB_WL="W.config_c5(n_seeds=256)" timeout 900 python scripts/ab_bench.py build/ab/*.so > $o/${t}_ab.txt 2>&1; cat $o/${t}_ab.txt | tail -6; fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_kernel --launch-skip 1 --launch-count 1 -f \
  -o $o/${t}_C5sub python scripts/run_lib_once.py paper_2510_15330_b200/libbellman_sim.so "W.config_c5(n_seeds=256)" > $o/${t}_ncu_C5sub.log 2>&1
python scripts/ncu_summary.py $o/${t}_C5sub.ncu-rep > $o/${t}_C5sub.txt 2>&1; head -20 $o/${t}_C5sub.txt

set -u
o=gpurun_out; t=${1:-ab}
timeout 600 python -m pytest tests/test_gpu_lane.py -q -x 2>&1 | tail -2
AB_REPS=5 AB_WL="W.config_c5()" timeout 900 python scripts/ab_bench.py build/ab/*.so > $o/${t}_ab.txt 2>&1; tail -4 $o/${t}_ab.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lane_kernel --launch-skip 1 --launch-count 1 \
  python scripts/run_lib_once.py paper_2510_15330_b200/libbellman_sim.so "W.config_c5(n_seeds=256)" 2>&1 | grep -E "dram__|gpu__time" > $o/${t}_dram.txt; cat $o/${t}_dram.txt
for f in build/ab/*.so; do echo $f; timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:lane_kernel --launch-skip 1 --launch-count 1 \
  python scripts/run_lib_once.py $f "W.config_c5(n_seeds=256)" 2>&1 | grep -E "dram__"; done > $o/${t}_dram_ab.txt; cat $o/${t}_dram_ab.txt

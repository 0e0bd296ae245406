set -u
o=gpurun_out; mkdir -p $o
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_kernel --launch-skip 1 --launch-count 1 -f \
  -o $o/l1_C5sub python scripts/run_lib_once.py paper_2510_15330_b200/libbellman_sim.so "W.config_c5(n_seeds=256)" > $o/l1_ncu_C5sub.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_kernel --launch-skip 1 --launch-count 1 -f \
  -o $o/l1_C2 python scripts/run_lib_once.py paper_2510_15330_b200/libbellman_sim.so "W.config_c2()" > $o/l1_ncu_C2.log 2>&1
python scripts/ncu_summary.py $o/l1_C5sub.ncu-rep > $o/l1_C5sub.txt 2>&1
python scripts/ncu_summary.py $o/l1_C2.ncu-rep > $o/l1_C2.txt 2>&1
tail -3 $o/l1_ncu_C2.log

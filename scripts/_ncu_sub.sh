# quick source-level ncu capture of K2L on a 1/16 C5 subset (development)
set -u
o=gpurun_out; t=${1:-sub}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lane_kernel --launch-skip 1 --launch-count 1 -f \
  -o $o/${t}_C5sub python scripts/run_lib_once.py paper_2510_15330_b200/libbellman_sim.so "W.config_c5(n_seeds=256)" > $o/${t}_ncu.log 2>&1
tail -2 $o/${t}_ncu.log

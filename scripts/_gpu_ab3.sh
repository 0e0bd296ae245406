set -u
o=gpurun_out; t=${1:-ab}
timeout 900 python -m pytest tests/test_gpu_lane.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
AB_REPS=7 AB_WL="W.config_c5()" timeout 900 python scripts/ab_bench.py build/ab/*.so > $o/${t}_ab.txt 2>&1; tail -4 $o/${t}_ab.txt

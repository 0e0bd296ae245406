set -u
o=gpurun_out; t=${1:-x}
# C3 through each engine (BELLMAN_LANE=2 forces K2L on the 10,272-scenario set)
for m in 0 2; do BELLMAN_LANE=$m timeout 600 python bench.py --workload C3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-peak 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 lane=$m', d['kernel_ms_per_step'], d['value'], d['engines'])"; done > $o/${t}_c3_engines.txt 2>&1
cat $o/${t}_c3_engines.txt
# strong-scaling projection: each rank's C5 shard alone (N = 8, rank 0 and 7) vs the whole set
timeout 900 python scripts/shard_balance.py > $o/${t}_shard_balance.txt 2>&1; tail -12 $o/${t}_shard_balance.txt

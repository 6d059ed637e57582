# tools/div_split_gpu.sh TAG -- the division head with and without the group
# split (DIV_PIPE_SPLIT): head-only cycles per step (tools/head_bench_s{0,1},
# built here), the pipelined-division parity tests, and the cfg3 bench line
# with the head's stats.  Outputs under gpurun_out/TAG.
T=${1:-divsplit}
O=gpurun_out/$T
mkdir -p $O
for v in 0 1; do
  for S in 64 128 256; do
    timeout 60 tools/head_bench_s$v $S >> $O/head_bench.jsonl 2>&1
  done
done
cat $O/head_bench.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "division or cfg3 or frozen or suite or fallback" > $O/pytest_div.log 2>&1
tail -2 $O/pytest_div.log
MMM_DIV_STATS=1 timeout 120 python tools/prof_one.py div --reps 1 > $O/stats_div.log 2>&1
tail -3 $O/stats_div.log
timeout 300 python bench.py --workload div --steps 10 --warmup 3 > $O/bench_div.log 2>&1
tail -1 $O/bench_div.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("div ms", d["ms_per_step"], "e2e ms", d["e2e"]["ms_per_step"], d["clocks"])'
MMM_DIV_STATS=1 MMM_DIV_BULK_GLOBAL_B=1 timeout 120 python tools/prof_one.py div --reps 1 > $O/stats_div_globalb.log 2>&1
tail -2 $O/stats_div_globalb.log

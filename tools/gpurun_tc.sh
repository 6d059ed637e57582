cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-tc1}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q --timeout 300 > $O/pytest_tc.log 2>&1; echo tc=$? >> $O/status
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -k "cfg5 or batched or fanout" > $O/pytest_cfg5.log 2>&1; echo cfg5=$? >> $O/status
timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/bench_batch.jsonl 2> $O/bench_batch.err; echo bench=$? >> $O/status

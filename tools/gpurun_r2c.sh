cd $GRAFT_REPO_ROOT; O=gpurun_out/r2c; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > $O/pytest.log 2>&1; echo pytest=$? >> $O/status
timeout 600 python bench.py --no-cpu-baseline > $O/bench_batch.jsonl 2> $O/bench_batch.err; echo bench=$? >> $O/status
timeout 600 python bench.py --workload ntt_batch --no-cpu-baseline > $O/bench_nttb.jsonl 2> $O/bench_nttb.err; echo nttb=$? >> $O/status

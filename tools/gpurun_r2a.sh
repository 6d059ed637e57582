cd $GRAFT_REPO_ROOT; O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/status
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rf > $O/pytest.log 2>&1; echo pytest=$? >> $O/status
timeout 600 python bench.py > $O/bench_batch.jsonl 2> $O/bench_batch.err; echo bench=$? >> $O/status
timeout 600 python bench.py --impl reference --steps 3 > $O/ref_batch.jsonl 2> $O/ref_batch.err; echo ref=$? >> $O/status
timeout 300 python bench.py --workload gcd --no-cpu-baseline > $O/bench_gcd.jsonl 2> $O/bench_gcd.err; echo gcd=$? >> $O/status

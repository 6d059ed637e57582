mkdir -p gpurun_out/ntt
timeout 600 python -m pytest tests -m gpu -x -q -k "ntt or fast or cfg1_via or smoke" > gpurun_out/ntt/pytest.log 2>&1; echo "pytest_exit=$?" >> gpurun_out/ntt/pytest.log
timeout 300 python bench.py --workload ntt --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ntt/bench_ntt.log 2>&1
timeout 300 python bench.py --workload ntt_batch --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ntt/bench_ntt_batch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ntt/launches.csv python bench.py --workload ntt --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ntt/ncu.log 2>&1

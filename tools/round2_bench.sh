# tools/round2_bench.sh TAG -- GPU parity + smoke, a bench line for every
# workload (and the reference arm of the default and the GCD), the launch
# list of the default bench command.  Outputs under gpurun_out/TAG.
T=${1:-r2}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$T; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/status
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > $O/pytest.log 2>&1; echo pytest=$? >> $O/status
timeout 900 python bench.py > $O/bench_batch.log 2>&1; echo batch=$? >> $O/status
timeout 600 python bench.py --impl reference --steps 3 > $O/ref_batch.log 2>&1; echo ref_batch=$? >> $O/status
for w in gcd mul div div_fast ntt ntt_batch; do
  timeout 600 python bench.py --workload $w --steps 10 > $O/bench_$w.log 2>&1; echo $w=$? >> $O/status
done
timeout 600 python bench.py --impl reference --workload gcd --steps 3 > $O/ref_gcd.log 2>&1; echo ref_gcd=$? >> $O/status
MMM_MUL_TC=0 MMM_DIV_TC=0 timeout 900 python bench.py --no-cpu-baseline --steps 5 > $O/bench_batch_simt.log 2>&1; echo batch_simt=$? >> $O/status
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_batch.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo launches=$? >> $O/status

# Time every NTT variant in tools/varlib/ (plus the in-tree library) on the
# cfg4 workloads: python bench.py device times, one line per (variant, workload).
O=gpurun_out/ntt_sweep; mkdir -p $O
for lib in paper_1402_0264_b200/lib/libmmm_cu.so tools/varlib/*/libmmm_cu.so; do
  n=$(basename $(dirname $lib))
  for w in ntt ntt_batch; do
    MMM_CU_LIB=$PWD/$lib timeout 120 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/$n.$w.log 2>&1
    echo "$n $w $(tail -1 $O/$n.$w.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), "us")' 2>&1 | tail -1)"
  done
done | tee $O/summary.txt

# Time the in-tree library and every variant in tools/varlib/ on the given
# workloads (device time per step):  bash tools/var_sweep.sh "div gcd"
O=gpurun_out/var_sweep; mkdir -p $O; rm -f $O/summary.txt
for lib in paper_1402_0264_b200/lib/libmmm_cu.so tools/varlib/*/libmmm_cu.so; do
  n=$(basename $(dirname $lib))
  for w in $1; do
    MMM_CU_LIB=$PWD/$lib timeout 180 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline $2 > $O/$n.$w.log 2>&1
    echo "$n $w $(tail -1 $O/$n.$w.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), "us")' 2>&1 | tail -1)"
  done
done | tee $O/summary.txt

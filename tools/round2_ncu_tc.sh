# tools/round2_ncu_tc.sh TAG -- ncu --set full of the tensor-core kernels
# (after the same command exited 0 without ncu) and the launch list of the
# default bench command.
T=${1:-r2}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$T; mkdir -p $O
cap() {
  local n=$1 w=$2 k=$3 c=$4; shift 4
  timeout 300 python tools/prof_one.py $w --reps 1 "$@" > $O/plain_$n.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c $c -o $O/full_$n \
      python tools/prof_one.py $w --reps 1 "$@" > $O/ncu_$n.log 2>&1
  echo full_$n=$? >> $O/status
}
cap tcmul batch tcmul_kernel 1
cap tcdiv batch tcdiv 1
cap mul mul tcmul_split 1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_batch.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
echo launches=$? >> $O/status
python tools/ncu_summary.py $O $O/sum > /dev/null 2>&1
for r in $O/full_*.ncu-rep; do python tools/ncu_brief.py $r > ${r%.ncu-rep}_brief.txt 2>&1; done
for r in $(ls -S $O/full_*.ncu-rep); do
  [ $(du -sm gpurun_out | cut -f1) -lt 56 ] && break
  rm -f $r
done

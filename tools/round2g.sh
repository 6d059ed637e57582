# tools/round2g.sh TAG -- the round-end measurement set after the tensor-core
# division rewrite: GPU parity + smoke, a bench line for every workload and the
# reference arm (tools/round2_bench.sh), the e2e anatomy (tools/e2e_probe.py),
# and ncu --set full captures of the cfg5 kernels (after the same command ran
# clean without ncu), summarised on the box.
T=${1:-r2g}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$T; mkdir -p $O
bash tools/round2_bench.sh $T
timeout 300 python tools/e2e_probe.py 5 > $O/e2e_probe.log 2>&1; echo e2e_probe=$? >> $O/status
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
python tools/ncu_summary.py $O $O/sum > /dev/null 2>&1
for r in $O/full_*.ncu-rep; do python tools/ncu_brief.py $r > ${r%.ncu-rep}_brief.txt 2>&1; done
ncu -i $O/full_tcdiv.ncu-rep --page source --csv --print-source sass > $O/tcdiv_src.csv 2>/dev/null
for r in $(ls -S $O/full_*.ncu-rep); do
  [ $(du -sm gpurun_out | cut -f1) -lt 56 ] && break
  rm -f $r
done

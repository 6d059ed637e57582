# tools/round2_ncu.sh TAG -- one `ncu --set full` capture per workload's
# dominant kernel (each after the same command exited 0 without ncu), then the
# s sweep: CUDA-event times per s (tools/s_sweep.py) and, per s, one ncu
# metric pass over the blocked kernel (cfg3 division, cfg2 GCD).
T=${1:-r2}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$T; mkdir -p $O
cap() {  # name workload kernel-regex count [extra args]
  local n=$1 w=$2 k=$3 c=$4; shift 4
  timeout 300 python tools/prof_one.py $w --reps 1 "$@" > $O/plain_$n.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c $c -o $O/full_$n \
      python tools/prof_one.py $w --reps 1 "$@" > $O/ncu_$n.log 2>&1
  echo full_$n=$? >> $O/status
}
cap tcmul batch tcmul 1
cap tcdiv batch tcdiv 1
cap gcd gcd gcd_kernel 1
cap mul mul tcmul_split 1
cap div div div_pipe 1
cap ntt ntt ntt_ 3
cap ntt_batch ntt_batch ntt_ 3
timeout 900 python tools/s_sweep.py --out $O/s_sweep.csv > $O/s_sweep.log 2>&1; echo s_sweep=$? >> $O/status
M=gpu__time_duration.sum,sm__inst_issued.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,dram__bytes.sum.per_second,lts__t_bytes.sum,sm__cycles_elapsed.avg
for s in 1 2 4 8 16 32 64 128; do
  timeout 300 python tools/prof_one.py div --s $s --reps 1 > $O/plain_div_s$s.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none -k regex:div_ -c 1 --csv python tools/prof_one.py div --s $s --reps 1 > $O/sweep_div_s$s.csv 2>&1
done
for s in 2 4 8 16 32 64 128; do
  timeout 300 python tools/prof_one.py gcd --s $s --reps 1 > $O/plain_gcd_s$s.log 2>&1 && \
  timeout 600 ncu --metrics $M --clock-control none -k regex:gcd_ -c 1 --csv python tools/prof_one.py gcd --s $s --reps 1 > $O/sweep_gcd_s$s.csv 2>&1
done
echo sweep_ncu=done >> $O/status
# summaries on the box (the copy-back is limited): key metrics, briefs, source pages
python tools/ncu_summary.py $O $O/sum > /dev/null 2>&1
for r in $O/full_*.ncu-rep; do
  python tools/ncu_brief.py $r > ${r%.ncu-rep}_brief.txt 2>&1
done
for r in $(ls -S $O/full_*.ncu-rep); do
  [ $(du -sm gpurun_out | cut -f1) -lt 56 ] && break
  rm -f $r
done

# tools/ncu_round.sh TAG -- bench lines for every workload, the launch list of
# the default bench command (after that command exited 0 without ncu), and one
# `ncu --set full` capture per workload's dominant kernel (after the plain run
# exited 0).  Outputs under gpurun_out/TAG; summarise with
#   python tools/ncu_summary.py gpurun_out/TAG profiles/TAG
set -x
T=${1:-r1}
O=gpurun_out/$T
mkdir -p $O
for w in gcd mul div div_fast ntt ntt_batch batch; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 > $O/bench_$w.log 2>&1
done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_gcd.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
for w in gcd mul div ntt ntt_batch batch; do
  c=1
  case $w in gcd) k=gcd_kernel;; mul) k=mul_kernel;; div) k=div_pipe_kernel;; ntt|ntt_batch) k=ntt_; c=3;; batch) k=div_cta_kernel;; esac
  timeout 120 python tools/prof_one.py $w --reps 1 > $O/plain_$w.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c $c -o $O/full_$w python tools/prof_one.py $w --reps 1 > $O/ncu_$w.log 2>&1
  tail -1 $O/ncu_$w.log
done
# Summarise on the box (gpurun copies back at most 64 MiB): per-kernel metric
# CSVs, a brief with stall samples and the source page of each capture; then
# drop the largest reports until the directory fits.
python tools/ncu_summary.py $O $O/sum > /dev/null 2>&1
for r in $O/full_*.ncu-rep; do
  python tools/ncu_brief.py $r > ${r%.ncu-rep}_brief.txt 2>&1
  ncu -i $r --page source --csv --print-source cuda > ${r%.ncu-rep}_src.csv 2>/dev/null
done
gzip -f $O/*_src.csv
for r in $(ls -S $O/full_*.ncu-rep); do
  [ $(du -sm gpurun_out | cut -f1) -lt 56 ] && break
  rm -f $r
done

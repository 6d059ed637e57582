set -x
mkdir -p gpurun_out/r1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1/launches_gcd.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1/ncu_launch.log 2>&1
for w in gcd mul div ntt batch; do
  case $w in gcd) k=gcd_kernel;; mul) k=mul_kernel;; div) k=div_grid_kernel;; ntt) k=ntt_rows;; batch) k=div_cta_kernel;; esac
  python tools/prof_one.py $w --reps 1 > gpurun_out/r1/plain_$w.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/r1/full_$w python tools/prof_one.py $w --reps 1 > gpurun_out/r1/ncu_$w.log 2>&1
  tail -1 gpurun_out/r1/ncu_$w.log
done

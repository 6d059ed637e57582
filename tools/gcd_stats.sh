# GCD phase clocks (MMM_GCD_STATS) for cfg2 through tools/prof_one.py, outputs in gpurun_out/$1
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-gcdstats}; mkdir -p $O
MMM_GCD_STATS=1 timeout 300 python tools/prof_one.py gcd --s 128 --reps 3 > $O/stats.log 2>&1; echo rc=$? >> $O/stats.log
timeout 300 python bench.py --workload gcd --steps 10 --no-cpu-baseline > $O/bench_gcd.log 2>&1
MMM_GCD_STATS=1 MMM_GCD_DEBUG=4 timeout 300 python tools/prof_one.py gcd --s 128 --reps 2 > $O/stats_dbg4.log 2>&1

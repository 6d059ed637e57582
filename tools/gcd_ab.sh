# A/B of GCD library variants (tools/varlib/*) on cfg2, plus the phase clocks of each
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-gcdab}; mkdir -p $O; shift
L=paper_1402_0264_b200/lib/libmmm_cu.so
V=""; for n in "$@"; do V="$V tools/varlib/$n/libmmm_cu.so"; done
timeout 900 python tools/ab.py gcd $L $V > $O/ab.txt 2>&1
for n in "$@"; do
  MMM_CU_LIB=$PWD/tools/varlib/$n/libmmm_cu.so MMM_GCD_STATS=1 timeout 300 python tools/prof_one.py gcd --s 128 --reps 1 > $O/stats_$n.log 2>&1
done

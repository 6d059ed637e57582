# tools/ncu_ntt.sh TAG -- ncu --set full (with source) of the cfg4 2^21 product's three kernels
T=${1:-ntt}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$T; mkdir -p $O
timeout 300 python tools/prof_one.py ntt --reps 1 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ntt_ -c 3 -o $O/full \
    python tools/prof_one.py ntt --reps 1 > $O/ncu.log 2>&1
echo full=$? >> $O/status
python tools/ncu_brief.py $O/full.ncu-rep > $O/brief.txt 2>&1
for i in 0 1 2; do
  ncu -i $O/full.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > $O/src$i.csv 2>/dev/null
done

# tools/ncu_tcdiv.sh TAG -- ncu --set full (with source) of tcdiv_kernel on the cfg5 batch,
# after the same command exited 0 without ncu; source page exported as CSV.
T=${1:-tcdiv}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$T; mkdir -p $O
K=${K:-tcdiv}
W=${W:-batch}
timeout 300 python tools/prof_one.py $W --reps 1 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o $O/full \
    python tools/prof_one.py $W --reps 1 > $O/ncu.log 2>&1
echo full=$? >> $O/status
ncu -i $O/full.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
python tools/ncu_brief.py $O/full.ncu-rep > $O/brief.txt 2>&1

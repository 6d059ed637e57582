cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-ncu_div}; mkdir -p $O
python tools/prof_batch.py div 296 > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tcdiv -s 1 -c 1 -o $O/tcdiv python tools/prof_batch.py div 296 > $O/ncu.log 2>&1
echo rc=$? >> $O/ncu.log

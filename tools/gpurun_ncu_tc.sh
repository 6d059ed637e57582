cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-ncu_tc}; mkdir -p $O
python tools/prof_batch.py mul 592 > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tcmul -s 1 -c 1 -o $O/tcmul python tools/prof_batch.py mul 592 > $O/ncu.log 2>&1
echo rc=$? >> $O/ncu.log

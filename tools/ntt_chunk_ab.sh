cd $GRAFT_REPO_ROOT; O=gpurun_out/nttc; mkdir -p $O
for c in 1073741824 16777216 8388608 4194304 2097152 1048576; do
  echo "chunk $c" >> $O/ab.log
  MMM_NTT_CHUNK_WORDS=$c AB_ROUNDS=1 timeout 300 python tools/ab.py ntt_batch paper_1402_0264_b200/lib/libmmm_cu.so >> $O/ab.log 2>&1
done
AB_ROUNDS=2 timeout 300 python tools/ab.py ntt paper_1402_0264_b200/lib/libmmm_cu.so >> $O/ab.log 2>&1

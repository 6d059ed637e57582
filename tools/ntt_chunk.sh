cd $GRAFT_REPO_ROOT; O=gpurun_out/ntt_chunk; mkdir -p $O
for c in 1073741824 33554432 16777216 8388608 4194304 2097152; do
  MMM_NTT_CHUNK_WORDS=$c timeout 300 python bench.py --workload ntt_batch --steps 10 --no-cpu-baseline > $O/c$c.log 2>&1
done

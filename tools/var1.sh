# tools/var1.sh FILE name "flags" [name2 "flags2" ...] -- variants of the kernel
# library that differ in ONE source file (FILE.cu compiled with the extra
# flags, every other object taken from the in-tree build) into
# tools/varlib/<name>/libmmm_cu.so, for tools/ab.py (MMM_CU_LIB).
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
F=$1; shift
make -s -C $R/paper_1402_0264_b200/csrc >/dev/null
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
OBJ=$R/build/obj
OTHERS=$(ls $OBJ/*.o | grep -v "/$F.o")
pids=()
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2
  mkdir -p $R/tools/varlib/$n
  ( $NV $f -c $R/paper_1402_0264_b200/csrc/$F.cu -o $R/tools/varlib/$n/$F.o > $R/tools/varlib/$n/ptxas.log 2>&1 && \
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/varlib/$n/libmmm_cu.so \
      $OTHERS $R/tools/varlib/$n/$F.o && echo "built $n" || (echo "FAILED $n"; tail -5 $R/tools/varlib/$n/ptxas.log) ) &
  pids+=($!)
done
for p in ${pids[@]}; do wait $p; done

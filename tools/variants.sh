# Build tuning variants of one kernel source into tools/varlib/<name>/ (select
# with MMM_CU_LIB=tools/varlib/<name>/libmmm_cu.so).  Usage:
#   bash tools/variants.sh SRC name "flags" [name2 "flags2" ...]     (SRC: ntt, divmod, gcd, mul, ...)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
SRC=$1; shift
make -s -C $R/paper_1402_0264_b200/csrc >/dev/null
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
OBJ=$R/build/obj
pids=()
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2
  mkdir -p $R/tools/varlib/$n
  objs=""
  for o in capi mul divmod gcd ntt fastdiv; do [ $o = $SRC ] && objs="$objs $R/tools/varlib/$n/$SRC.o" || objs="$objs $OBJ/$o.o"; done
  ( $NV $f -c $R/paper_1402_0264_b200/csrc/$SRC.cu -o $R/tools/varlib/$n/$SRC.o > $R/tools/varlib/$n/ptxas.log 2>&1 && \
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/varlib/$n/libmmm_cu.so $objs && echo "built $n" ) &
  pids+=($!)
done
for p in ${pids[@]}; do wait $p; done

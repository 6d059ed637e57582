# Build NTT tuning variants of the library into tools/varlib/<name>/ (select
# one with MMM_CU_LIB=tools/varlib/<name>/libmmm_cu.so).  Usage:
#   bash tools/ntt_variants.sh name "-DNTT_KMAX=3 -DNTT_TMAX=1024" [name2 "flags2" ...]
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
make -s -C $R/paper_1402_0264_b200/csrc >/dev/null
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
OBJ=$R/build/obj
pids=()
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2
  mkdir -p $R/tools/varlib/$n
  ( $NV $f -c $R/paper_1402_0264_b200/csrc/ntt.cu -o $R/tools/varlib/$n/ntt.o > $R/tools/varlib/$n/ptxas.log 2>&1 && \
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/varlib/$n/libmmm_cu.so \
      $OBJ/capi.o $OBJ/mul.o $OBJ/divmod.o $OBJ/gcd.o $OBJ/fastdiv.o $R/tools/varlib/$n/ntt.o && echo "built $n" ) &
  pids+=($!)
done
for p in ${pids[@]}; do wait $p; done

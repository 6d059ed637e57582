# tools/varbuild.sh NAME [EXTRA nvcc flags...] -- a variant of the kernel library
# (e.g. -DTCD_STATS=1) into tools/varlib/NAME/libmmm_cu.so for tools/ab.py.
N=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C $R/paper_1402_0264_b200/csrc OBJ=$R/build/var_$N OUT=$R/tools/varlib/$N EXTRA="$*" $R/tools/varlib/$N/libmmm_cu.so

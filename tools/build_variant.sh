#!/bin/bash
# Build an A/B variant of libse_b200.so with extra nvcc flags for one source:
#   tools/build_variant.sh <tag> <source.cu> <nvcc flags...>
# -> build_ab/<tag>/libse_b200.so (load it with SE_B200_LIB=...)
# SE_VARIANT_FILE=<path>: compile that file in place of csrc/<source.cu>
# (e.g. the committed version: git show HEAD:.../se_realspace.cu > /tmp/x.cu)
set -e
TAG=$1; SRC=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1712_04732_b200/csrc
O=$ROOT/build_ab/$TAG; mkdir -p $O
(cd $C && make -s -j8 >/dev/null)
ARCH="-gencode arch=compute_100a,code=sm_100a"
IN=${SE_VARIANT_FILE:-$C/$SRC}
if [ "$IN" != "$C/$SRC" ]; then cp "$IN" $C/.variant_$SRC; IN=$C/.variant_$SRC; fi
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$ROOT/include "$@" -c $IN -o $O/${SRC%.cu}.o
rm -f $C/.variant_$SRC
OBJS=""
for f in $C/build/*.o; do b=$(basename $f); if [ "$b" = "${SRC%.cu}.o" ]; then OBJS="$OBJS $O/$b"; else OBJS="$OBJS $f"; fi; done
nvcc $ARCH -shared -cudart static -o $O/libse_b200.so $OBJS -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath,/usr/local/cuda/lib64
echo $O/libse_b200.so

#!/bin/bash
# A/B timing of the real-space kernel: one process per library build
# (build_ab/<variant>/libse_b200.so from tools/build_variant.sh; "base" =
# the in-tree library), interleaved twice, phi_R compared against base.
#   bash tools/gpu/ab.sh <tag> "<workloads>" <variant> ...
set -u
TAG=$1; W=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
for rep in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then L=; else L=build_ab/$v/libse_b200.so; fi
    SE_B200_LIB=$L timeout 300 python tools/gpu/ab_realspace.py $O/$v.$rep.json $W > $O/$v.$rep.log 2>&1
  done
done
for v in "$@"; do for rep in 1 2; do
  python tools/gpu/ab_realspace.py --compare $O/base.$rep.json $O/$v.$rep.json >> $O/compare.txt 2>&1
done; done
rm -f $O/*.npy
cat $O/compare.txt

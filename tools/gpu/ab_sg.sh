#!/bin/bash
# Spread/gather A/B: tools/gpu/ab_sg.py for the in-tree library and each
# build_ab/<variant>, interleaved twice; then the spread/gather parity tests.
#   bash tools/gpu/ab_sg.sh <tag> "<workloads>" <variant> ...
set -u
TAG=$1; W=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
for rep in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then L=; else L=build_ab/$v/libse_b200.so; fi
    SE_B200_LIB=$L timeout 300 python tools/gpu/ab_sg.py $W >> $O/ab_sg.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stage_api.py tests/test_gpu_reference_properties.py -m gpu -x -q > $O/pytest_sg.log 2>&1; echo "pytest rc=$?"
cat $O/ab_sg.txt; tail -2 $O/pytest_sg.log

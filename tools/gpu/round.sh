#!/bin/bash
# One GPU session: GPU tests, bench (N=1), peaks, ncu launch list and
# --set full captures of the hot kernels, all into gpurun_out/<tag>/.
#   tools/gpu/round.sh <tag> [tests|bench|ncu|peaks ...]   (default: all)
set -u
TAG=${1:-r02}; shift || true
WHAT=${*:-"tests bench peaks ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
           timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" ;;
    peaks) nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu && /tmp/peaks > $OUT/peaks.json; echo "peaks rc=$?" ;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
        --log-file $OUT/launches.csv python tools/gpu/profile_step.py cfg2 > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
      for st in realspace spread gather; do
        case $st in realspace) K=realspace_cell;; spread) K=spread_tile;; gather) K=gather_tile;; esac
        timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
          -k regex:$K -c 1 -o $OUT/${st} -f \
          python tools/gpu/profile_step.py cfg2 $st > $OUT/ncu_$st.log 2>&1; echo "ncu $st rc=$?"
      done ;;
  esac
done

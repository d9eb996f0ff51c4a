#!/bin/bash
# ncu --set full captures beyond final.sh: the hot kernels at cfg5 (D = 0,
# clustered) and every kernel of the k-space stage (cuFFT + multipliers) at
# cfg2 and cfg5.   bash tools/gpu/ncu_more.sh <tag>
set -u
TAG=${1:-ncu_more}
O=gpurun_out/$TAG; mkdir -p $O
for st in realspace spread gather; do
  case $st in realspace) K=realspace_cell;; spread) K="spread_(tile|ws)";; gather) K=gather_tile;; esac
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:$K -c 1 -o $O/cfg5_${st} -f python tools/gpu/profile_step.py cfg5 $st > $O/ncu_cfg5_$st.log 2>&1; echo "ncu cfg5 $st rc=$?"
done
for w in cfg2 cfg5; do
  timeout 900 ncu --set full --clock-control none --profile-from-start off -c 40 -o $O/${w}_kspace -f \
    python tools/gpu/profile_step.py $w kspace > $O/ncu_${w}_kspace.log 2>&1; echo "ncu $w kspace rc=$?"
done

#!/bin/bash
# Copy the evidence of one tools/gpu/final.sh run (gpurun_out/<tag>/) into
# the tracked profiles/ tree under this round's names:
#   bash tools/collect_evidence.sh <tag> [round]
set -eu
TAG=$1; R=${2:-r02}
S=gpurun_out/$TAG; P=profiles
mkdir -p $P/${R}_configs $P/ncu
cp $S/bench.json $P/bench_${R}_cfg2.json
cp $S/bench_ref.json $P/bench_${R}_reference_arm.json
cp $S/bench_tr1.json $P/bench_${R}_torchrun1.json
for f in $S/bench_cfg*.json; do cp $f $P/${R}_configs/; done
cp $S/first_call.json $P/first_call_${R}.json
cp $S/peaks.json $P/peaks_${R}.json
python tools/summarize_ncu.py launches $S/launches.csv > $P/launches_${R}.txt
cp $S/realspace.ncu-rep $P/ncu/realspace_cfg2_${R}.ncu-rep
python tools/profile_summary.py $TAG $R
{ echo "# The reference's own test suite (pkg/tests, 190 tests, unmodified) against paper_1712_04732_b200 via the pmewald alias (tools/ref_suite), SE_B200_DETERMINISTIC=1, B200 (tools/gpu/final.sh $TAG); then this repo's pytest -m gpu of the same run"
  tail -n 2 $S/ref_suite.log; tail -n 2 $S/pytest.log; } > $P/ref_suite_${R}.txt
head -12 $P/launches_${R}.txt

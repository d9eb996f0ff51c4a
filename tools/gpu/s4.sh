O=gpurun_out/s4; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_domain.py -x -q -s > $O/domain.log 2>&1; echo "domain rc=$?"
python tools/gpu/ab_realspace.py /tmp/ab_cs.json cfg2 cfg5 cfg4 > $O/ab_sort.log 2>&1; echo "ab rc=$?"
bash tools/gpu/round.sh r02b ncu
python tools/summarize_ncu.py launches gpurun_out/r02b/launches.csv > $O/launches.txt 2>&1
grep -E "passed|failed|one-rank" $O/domain.log | tail -6; cat $O/ab_sort.log; head -12 $O/launches.txt

O=gpurun_out/s5; mkdir -p $O
python tools/gpu/ab_realspace.py /tmp/ab_cs2.json cfg2 cfg5 cfg4 > $O/ab_sort.log 2>&1; echo "ab rc=$?"
python tools/gpu/first_call.py $O/first_call.json cfg2 cfg5 cfg3_tol cfg4 > $O/first_call.log 2>&1; echo "first rc=$?"
for w in cfg5 cfg1_tol cfg4_tol cfg3_tol; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?"; done
cat $O/ab_sort.log $O/first_call.log

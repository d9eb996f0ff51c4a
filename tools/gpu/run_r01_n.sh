# round-1 measurement snapshot: full bench (cfg2 + cpu baseline), reference arm,
# per-config bench lines, ncu launch list, ncu --set full of the real-space kernel
set -x
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
for w in cfg1 cfg3 cfg3_tol cfg4 cfg5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w=$?; done
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:realspace_cell -c 1 -o gpurun_out/prof_final4 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
nproc; lscpu | grep -E "Model name|^CPU\(s\)"

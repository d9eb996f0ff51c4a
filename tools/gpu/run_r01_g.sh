set -x
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1200 -k "baseline_config" > gpurun_out/gpu_cfg_tests.log 2>&1; tail -15 gpurun_out/gpu_cfg_tests.log
for w in cfg1 cfg3 cfg3_tol cfg4 cfg5; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo $w rc=$?; tail -2 gpurun_out/bench_$w.err; done

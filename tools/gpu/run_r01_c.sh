set -x
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 2500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/gpu/sanity_small.py > gpurun_out/memcheck.log 2>&1; echo memcheck=$?; tail -5 gpurun_out/memcheck.log

timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "geometry_sweep" --timeout 1200 > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log

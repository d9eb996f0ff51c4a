timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "graph" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log

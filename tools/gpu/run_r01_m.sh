timeout 1200 python -m pytest tests/test_gpu_direct.py -x -q -s --timeout 900 > gpurun_out/gpu_direct.log 2>&1; tail -15 gpurun_out/gpu_direct.log

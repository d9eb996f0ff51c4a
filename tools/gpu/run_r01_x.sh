timeout 1500 python -m pytest tests/test_gpu_direct.py -x -q -s --timeout 1200 > gpurun_out/gpu_direct.log 2>&1; grep -E "rel RMS|passed|failed|Error" gpurun_out/gpu_direct.log | head

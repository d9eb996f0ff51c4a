timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1200 -k "baseline_config" > gpurun_out/gpu_cfg_tests.log 2>&1; tail -5 gpurun_out/gpu_cfg_tests.log

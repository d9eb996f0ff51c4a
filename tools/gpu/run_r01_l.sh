# full GPU suite + bench + realspace ncu
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2>/dev/null && python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('step', d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})" && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:realspace_cell -c 1 -o gpurun_out/prof_v27 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu=$?

timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "realspace or geometry or baseline or golden or randomized or graph" > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for W in cfg2 cfg5; do
for v in a default a default; do
  if [ $v = a ]; then export SE_B200_LIB=$PWD/paper_1712_04732_b200/_lib/libse_b200_a.so; else unset SE_B200_LIB; fi
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$W $v', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items() if k in ('realspace','sort')})"
done; done

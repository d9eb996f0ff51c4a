# A/B of alternative builds (paper_1712_04732_b200/_lib/libse_b200_<v>.so) vs
# the in-tree library ("new") over the workloads: step time and kernel spans.
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests/test_gpu_stage_api.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
fi
for W in ${WORKLOADS:-cfg1 cfg2 cfg3_tol cfg4 cfg5}; do
for rep in 1 2; do
for v in ${VARIANTS:-a new}; do
  if [ $v = new ]; then unset SE_B200_LIB; else export SE_B200_LIB=$PWD/paper_1712_04732_b200/_lib/libse_b200_$v.so; fi
  timeout 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$W $v', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}, 'sg', round(d['spread_gather']['spread']['ms_per_launch'],3), round(d['spread_gather']['gather']['ms_per_launch'],3))"
done; done; done

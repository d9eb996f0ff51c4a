for v in 1 2 3 1 2 3; do
  SE_OVL=$v timeout 600 python bench.py --workload ${W:-cfg2} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ovl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ovl.json'));print('v$v', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done

for k in 1 2 4 8 1 2 4 8; do
  SE_RSCHUNKS=$k timeout 600 python bench.py --workload ${W:-cfg2} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ch.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ch.json'));print('K$k', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
done

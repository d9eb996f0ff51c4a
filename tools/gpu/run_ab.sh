# A/B: alternative library build (SE_B200_LIB) vs the default, alternating
for i in 1 2; do
  for v in a default; do
    if [ $v = a ]; then export SE_B200_LIB=$PWD/paper_1712_04732_b200/_lib/libse_b200_a.so; else unset SE_B200_LIB; fi
    timeout 600 python bench.py --workload ${W:-cfg2} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
  done
done

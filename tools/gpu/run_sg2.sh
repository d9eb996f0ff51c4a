true
for w in cfg2 cfg3 cfg2; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bsg.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bsg.json'));sg=d['spread_gather'];print('$w', round(d['ms_per_step'],3), 'spread', round(sg['spread']['ms_per_launch'],3), 'gather', round(sg['gather']['ms_per_launch'],3))"; done

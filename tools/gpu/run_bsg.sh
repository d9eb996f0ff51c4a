timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bsg.json 2> gpurun_out/bsg.err; echo rc=$?; tail -3 gpurun_out/bsg.err
python -c "import json;d=json.load(open('gpurun_out/bsg.json'));print(d['ms_per_step']);print(json.dumps(d['spread_gather'], indent=1))"

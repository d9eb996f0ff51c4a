# Bench lines for every BASELINE config (profiles/r01_configs).
mkdir -p gpurun_out/configs
for W in ${WORKLOADS:-cfg1 cfg3 cfg3_tol cfg4 cfg5}; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline > gpurun_out/configs/bench_$W.json 2> gpurun_out/configs/bench_$W.err
  echo "$W rc=$?"; cut -c1-200 gpurun_out/configs/bench_$W.json
done

set -e
mkdir -p gpurun_out
for c in cfg4 cfg5 cfg3_tol; do timeout 600 python tools/gpu/crit_path.py $c 2>&1 | tail -1; done
for c in cfg4 cfg5 cfg3_tol; do
  timeout 300 python tools/gpu/ks_only.py $c 2 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ks_$c.csv python tools/gpu/ks_only.py $c 2 > /dev/null 2>&1
done

# Full round check: GPU tests, smoke, default bench, reference arm, ncu launch
# list, one ncu --set full capture of the real-space kernel.
set -o pipefail
TAG=${TAG:-check}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench_$TAG.json
if [ -z "$NOREF" ]; then
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_ref_$TAG.json
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:realspace_cell_kernel -c 1 \
  -o gpurun_out/rs_$TAG -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_rs.log 2>&1; echo "ncu full rc=$?"

#!/bin/bash
# Round-end evidence on one B200: GPU tests, the reference suite, the bench
# (default line + reference arm + torchrun world 1), per-config lines with
# enough steps for clock sampling, peaks, and the ncu launch list + --set
# full captures of the hot kernels of THIS build (profiles/ summaries are
# made from these by tools/profile_summary.py).
#   bash tools/gpu/final.sh <tag>
set -u
TAG=${1:-r02final}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"
bash baseline/_ref_suite/run.sh > $O/ref_suite.log 2>&1; echo "ref suite rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_tr1.json 2> $O/bench_tr1.err; echo "torchrun rc=$?"
for w in cfg1 cfg1_tol cfg3 cfg3_tol cfg4 cfg4_tol cfg5 cfg2_tol; do
  steps=40; case $w in cfg1*) steps=3000;; cfg3*) steps=300;; cfg4*) steps=150;; esac
  timeout 900 python bench.py --workload $w --steps $steps --warmup 5 --no-cpu-baseline --no-tol > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?"
done
python tools/gpu/first_call.py $O/first_call.json cfg2 cfg5 cfg3_tol cfg4 > $O/first_call.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu && /tmp/peaks > $O/peaks.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches.csv python tools/gpu/profile_step.py cfg2 > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for st in realspace spread gather; do
  case $st in realspace) K=realspace_cell;; spread) K="spread_(tile|ws)";; gather) K=gather_tile;; esac
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:$K -c 1 -o $O/${st} -f python tools/gpu/profile_step.py cfg2 $st > $O/ncu_$st.log 2>&1; echo "ncu $st rc=$?"
done
tail -n 2 $O/pytest.log $O/ref_suite.log

# session 2: new GPU tests, full suite, bench (plain + torchrun world 1)
O=gpurun_out/s2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_domain.py -x -q -s > $O/domain.log 2>&1; echo "domain rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_tr1.json 2> $O/bench_tr1.err; echo "bench torchrun rc=$?"
tail -3 $O/domain.log $O/pytest.log

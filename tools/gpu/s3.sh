O=gpurun_out/s3; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_deterministic.py tests/test_gpu_domain.py -x -q -s > $O/det.log 2>&1; echo "det rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"
bash baseline/_ref_suite/run.sh > $O/ref_suite.log 2>&1; echo "ref suite rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -2 $O/det.log $O/pytest.log $O/ref_suite.log

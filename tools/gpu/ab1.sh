# dense-batch threshold sweep of the real-space kernel + parity
O=gpurun_out/ab1; mkdir -p $O
for d in 513 460 410 360 300; do SE_B200_DENSE_MIN=$d python tools/gpu/ab_realspace.py $O/d$d.json cfg2 cfg5 cfg4 2>&1 | tail -3; done
for d in 460 410 360 300; do python tools/gpu/ab_realspace.py --compare $O/d$d.json $O/d513.json; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_reference.py -x -q 2>&1 | tail -3

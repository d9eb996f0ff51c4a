# dense threshold sweep on the current build
for d in 330 370 410 450; do SE_B200_DENSE_MIN=$d python tools/gpu/ab_realspace.py /tmp/d$d.json cfg2 cfg5 cfg4 > /dev/null 2>&1; done
for d in 330 370 450; do python tools/gpu/ab_realspace.py --compare /tmp/d$d.json /tmp/d410.json; done

# A/B of the real-space kernel: build_ab/libse_old.so (HEAD) vs the working tree build
for i in 1 2; do
SE_B200_LIB=$PWD/build_ab/libse_old.so python tools/gpu/ab_realspace.py /tmp/old.json cfg2 cfg5 cfg4 cfg3_tol 2>&1 | grep -v "^$"
python tools/gpu/ab_realspace.py /tmp/new.json cfg2 cfg5 cfg4 cfg3_tol 2>&1 | grep -v "^$"
python tools/gpu/ab_realspace.py --compare /tmp/new.json /tmp/old.json
done

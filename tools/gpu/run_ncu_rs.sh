# One ncu --set full capture of the cfg2 real-space kernel (source-level stalls).
W=${W:-cfg2}
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:realspace_cell_kernel -c 1 \
  -o gpurun_out/rs_${W} -f python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_rs.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_rs.log

set -x
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"realspace_cell_kernel|spread_tile_kernel|gather_tile_kernel" -s 3 -c 3 -o gpurun_out/prof_v10 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo ncu2=$?

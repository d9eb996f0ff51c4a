# ncu --set full of the field-mode real-space kernel at cfg2.
timeout 1500 ncu --set full --clock-control none -k regex:realspace_cell_kernel -c 1 -o gpurun_out/field_rs -f \
  python tools/gpu/field_time.py > gpurun_out/ncu_field.log 2>&1; echo "ncu rc=$?"

# ncu source view of the grid kernel (592 sources = two per resident CTA)
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:slices_lowdeg_sm_kernel" -c 1 \
  -o gpurun_out/ncu_r2_grid -f python tools/prof_batch.py --grid 512 --sources 592 --consecutive --no-profile > gpurun_out/ncu_r2_grid.log 2>&1
echo "ncu rc=$?"

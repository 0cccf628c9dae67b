# ncu --set full (+ sector efficiency, red instructions) of one 256-source S20 batch's level and push kernels, source view
timeout 300 python tools/prof_batch.py --sources 256 --streams 1 | tail -1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:lanes_(push|level)_kernel" -c 14 \
  --metrics smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__inst_executed_op_global_red.sum \
  -o gpurun_out/ncu_r2_s20 -f python tools/prof_batch.py --sources 256 --streams 1 > gpurun_out/ncu_r2_s20.log 2>&1
echo "ncu rc=$?"

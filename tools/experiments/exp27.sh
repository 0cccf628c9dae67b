timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3
timeout 120 python tools/prof_batch.py --grid 512 --sources 4096 --repeat 2 | tail -1
timeout 300 python bench.py --config grid --steps 8 --warmup 3 > gpurun_out/bench_grid.json 2> gpurun_out/bench_grid.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_grid.json
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:slices_lowdeg" -c 1 \
  -o gpurun_out/ncu_grid_v2 -f python tools/prof_batch.py --grid 512 --sources 1184 > gpurun_out/ncu_grid_v2.log 2>&1; echo "ncu rc=$?"

timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
timeout 300 python bench.py --config grid --steps 8 --warmup 3 > gpurun_out/bench_grid.json 2> gpurun_out/bench_grid.err; echo "bench grid rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_grid.csv python bench.py --config grid --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_grid.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:slices_lowdeg" -c 1 \
  -o gpurun_out/ncu_grid_r1 -f python tools/prof_batch.py --grid 512 --sources 8192 > gpurun_out/ncu_grid_r1.log 2>&1; echo "ncu rc=$?"

# round-2 final pass on one B200: GPU suite, smoke, bench lines of every config, launch list of the headline bench
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/pytest_gpu_r2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke_r2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r2.log
for c in rmat20 rmat12 rmat16 rmat16p grid rmat23; do
  st=10; [ $c = rmat23 ] && st=4
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/bench_r2_$c.json 2> gpurun_out/bench_r2_$c.err
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_r2_reference.json 2> gpurun_out/bench_r2_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2_s20.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1

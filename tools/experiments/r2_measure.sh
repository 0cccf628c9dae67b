# round-2 measurement pass: bench lines for every config, launch list + ncu --set full of one S20 batch, long-diameter ablation
set -x
for c in rmat20 rmat12 rmat16 rmat16p grid rmat23; do
  st=5; [ $c = rmat23 ] && st=3
  timeout 900 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/bench_r2_$c.json 2> gpurun_out/bench_r2_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2_s20.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
bash tools/ncu_cap.sh ncu_r2_s20_batch "regex:lanes_" 40 --sources 256 --streams 1 > gpurun_out/ncu_cap.log 2>&1
timeout 1500 python tools/ablation_long.py > gpurun_out/ablation_long.jsonl 2> gpurun_out/ablation_long.err

for c in rmat12 rmat16 rmat16p grid rmat23; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-400
done

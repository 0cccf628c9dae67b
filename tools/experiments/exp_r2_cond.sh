# device-driven batches: sigma tiers as conditional (IF) graph nodes (cond1) vs gated launches (cond0)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -x -p no:cacheprovider -k "device_loop or sigma or tiers or narrow or stream or small_suite_all" 2>&1 | tail -2
for v in cond0 cond1 cond0 cond1; do
  echo -n "$v S12: "; BC_SO=build_exp/lib_$v.so timeout 100 python tools/prof_batch.py --scale 12 --all --lane-words 0 --repeat 4 --no-profile | tail -1 | cut -c1-80
  echo -n "$v S16: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --all --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-80
  echo -n "$v S20: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done

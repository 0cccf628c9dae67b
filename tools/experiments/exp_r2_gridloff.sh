# grid kernel: level offsets in shared memory (BC_SM_LOFF), with the two-deep backward prefetch / forward queue buffer
for v in gb gl gl1k glp glr gb gl gl1k glp glr; do
  echo -n "$v grid consecutive: "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --consecutive --repeat 2 --no-profile | tail -1 | cut -c1-100
done
for v in gl glp; do
echo -n "$v parity: "; BC_SO=build_exp/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "slices or capture_small or grid" 2>&1 | tail -1
done

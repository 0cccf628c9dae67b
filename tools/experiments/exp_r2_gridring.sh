# grid kernel: forward shared queue double buffer (BC_SM_RING) and backward two-deep first-slot prefetch (BC_SM_BPF2)
for v in gb gr gp grp gb gr gp grp; do
  echo -n "$v grid consecutive: "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --consecutive --repeat 2 --no-profile | tail -1 | cut -c1-100
done
for v in gr gp grp; do
echo -n "$v parity: "; BC_SO=build_exp/lib_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "slices or capture_small or grid" 2>&1 | tail -1
done

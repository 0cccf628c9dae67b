# push parent-mask loads with an L2 policy (reds evict_last in all): none / evict_first / evict_last
for v in mh0 mh1 mh2 mh0 mh1 mh2; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
echo -n "mh0 parity: "; BC_SO=build_exp/lib_mh0.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "backward or small_suite or config4" 2>&1 | tail -1

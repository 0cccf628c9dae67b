# backward push: coef row in shared memory (CFSMEM=1) vs registers (0); 4 vs 5 CTAs per SM
for v in cf0 cf1 cf1m5 cf0m5 cf0 cf1; do
  echo -n "$v S20: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
echo -n "cf1 parity: "; BC_SO=build_exp/lib_cf1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "backward or small_suite or config4 or sigma or two_degree" 2>&1 | tail -1

# push: own sigma row evict_first too (ow2) vs accumulator only (ow1); forward item masks evict_last (fm2, with ow1)
for v in ow1 ow2 fm2 ow1 ow2 fm2; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in ow1 ow2 fm2; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
echo -n "ow1 parity: "; BC_SO=build_exp/lib_ow1.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "backward or small_suite or config4 or widens" 2>&1 | tail -1

# backward commit: BC[x] += contribution by red.global.add (br1) vs load + add + store (br0)
for v in br0 br1 br0 br1; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in br0 br1; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
echo -n "br1 parity: "; BC_SO=build_exp/lib_br1.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1

# 16-bit forward: hits per iteration with loads in flight (2 / 3 / 4; 4 at 3 CTAs/SM)
for v in n2 n3 n4 n4b n2 n3 n4; do
  echo -n "$v S20: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in n2 n3 n4; do
  echo -n "$v S16: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --sources 16384 --streams 1 --lane-words 8 --repeat 2 | tail -1 | cut -c1-120
done
echo -n "n3 parity: "; BC_SO=build_exp/lib_n3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1

# 16-bit forward: two hits per iteration (BC_FWD_HIT2=1) vs one (0)
for v in h0 h1 h0 h1; do
  echo -n "$v S20: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in h0 h1; do
  echo -n "$v S16: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --sources 16384 --streams 1 --lane-words 8 --repeat 2 | tail -1 | cut -c1-120
  echo -n "$v S12 all: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 12 --all --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
echo -n "h1 parity: "; BC_SO=build_exp/lib_h1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1

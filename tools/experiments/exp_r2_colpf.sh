# forward step loop: next step's columns fetched one step ahead (cp1; cp1m4 at 4 CTAs / 64 registers) vs cp0
for v in cp0 cp1 cp1m4 cp0 cp1 cp1m4; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in cp0 cp1; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
  echo -n "$v S16 all: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --all --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-80
done
echo -n "cp1 parity: "; BC_SO=build_exp/lib_cp1.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1

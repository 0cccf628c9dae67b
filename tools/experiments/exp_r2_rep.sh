# backward: replicated accumulator rows for the hub parents (BC_REP_H lowest ids x BC_REP_R copies)
for v in r0 r64 r16 r256 r0 r64 r16 r256; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in r0 r64; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
  echo -n "$v S16 16k: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --sources 16384 --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-80
done
echo -n "r64 suite: "; BC_SO=build_exp/lib_r64.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1

# 16-bit forward: whole hit rows (BC_FWD_UNCOND=1) vs per-pair c-tested loads (0)
for v in u0 u1 u0 u1; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-200
done
for v in u0 u1; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
  echo -n "$v S16 all: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --sources 65536 --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-80
done
echo -n "u1 parity: "; BC_SO=build_exp/lib_u1.so timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1

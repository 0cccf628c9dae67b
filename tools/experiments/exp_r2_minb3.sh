# level kernel occupancy at W = 2 (S23, auto lane width) and W = 8 (S16)
for v in b0 w2m4 w2m5; do
  echo -n "$v S23 2048: "; BC_SO=build_exp/lib_$v.so timeout 600 python tools/prof_batch.py --scale 23 --sources 2048 --lane-words 0 --repeat 2 | tail -1 | cut -c1-120
done
for v in b0 w8m4 b0 w8m4; do
  echo -n "$v S16 16k: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --sources 16384 --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-80
done

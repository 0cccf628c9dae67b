# push reds with an L2 eviction policy: none / evict_first / evict_last (S20 8192 sources, 1 pipeline and auto)
for v in rh0 rh1 rh2 rh0 rh1 rh2; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in rh0 rh1 rh2; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done

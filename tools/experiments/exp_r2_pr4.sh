# push kernel at W = 4: item steps in flight per warp (BC_PR4) and CTAs per SM
for v in pr1 pr2 pr2m3 pr1 pr2 pr2m3; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done

# 16-bit forward sigma-row gathers with an L2 policy: none / evict_first / evict_last
for v in fr0 fr1 fr2 fr0 fr1 fr2; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done

# whole-row forward: L2 policy of the row gathers (0 none, 1 evict_first, 2 evict_last = default)
for v in rh0 rh1 rh2 rh0 rh1 rh2; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done

# L2 policies re-checked after the round-2 kernels: forward mask loads evict_last (fmh1), push own-row hint off / 2 (poh0/poh2), push parent-mask evict_first (pmh1), push reds without policy (prh0)
for v in base fmh1 poh0 poh2 pmh1 prh0 base fmh1 poh0 poh2 pmh1 prh0; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done

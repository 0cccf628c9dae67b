# grid kernel: shared queue double buffer sized to stay inside the 164 KB shared carve-out (L1 unchanged)
for v in gb gr512 gr1k gr15 gb gr512 gr1k gr15; do
  echo -n "$v grid consecutive: "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --consecutive --repeat 2 --no-profile | tail -1 | cut -c1-100
done

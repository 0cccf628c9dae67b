# backward accumulator row padding (BC_A_PAD doubles after each K-double row): L2 slice balance of the push reds
for v in p0 p4 p16 p32 p0 p4 p16 p32; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done

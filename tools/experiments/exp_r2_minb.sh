# forward level kernel at W = 4: resident CTAs per SM (launch bounds 4 / 5 / 6 -> 63 / 48 / 40 registers)
for v in m4 m5 m6 m4 m5 m6; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done

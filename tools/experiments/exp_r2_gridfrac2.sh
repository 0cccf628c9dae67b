# concurrent pipelines: level / push kernel grid fractions re-measured after the 5-CTA forward
for v in g34 f11 f12 p11 p12 g34 f11 f12 p11 p12; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done

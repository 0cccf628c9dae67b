# forward / push grid fractions (x resident CTAs): S20 8192 sources (auto pipelines, device loop), S16 all
for v in f34p34 f12p1 f1p12 f34p1 f1p34 f23p23 f34p34 f34p1 f1p34; do
  echo -n "$v S20: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
for v in f34p34 f34p1 f1p34; do
  echo -n "$v S16: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --all --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-80
  echo -n "$v S12: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 12 --all --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done

# level / push kernel grid fraction (room for concurrent pipelines): S20 8192 sources, auto pipelines, device loop
for v in g11 g12 g34 g11 g12 g34; do
  echo -n "$v S20: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-100
done
for v in g11 g12; do
  echo -n "$v S16: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --all --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-100
done

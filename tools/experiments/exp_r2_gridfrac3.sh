# forward grid fraction 1/1 with push fractions 5/8, 3/4, 7/8; S16 / S12 all sources for the same builds
for v in g34 f11 f11p58 f11p78 g34 f11 f11p58 f11p78; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
for v in g34 f11 g34 f11; do
  echo -n "$v S16 all: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --all --lane-words 0 --repeat 2 --no-profile | tail -1 | cut -c1-80
  echo -n "$v S12 all: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 12 --all --lane-words 0 --repeat 5 --no-profile | tail -1 | cut -c1-80
done

# adaptive tile size (BC_TILE_MIN 256) vs fixed 8192-item tiles, device loop on (and off: BC_DEVLOOP=0 via --devloop)
for v in t8k t256; do
  for cfg in "--scale 12 --all --lane-words 0 --repeat 3" "--scale 16 --all --lane-words 0 --repeat 2" "--scale 20 --sources 8192 --lane-words 0 --repeat 2"; do
    echo -n "$v $cfg: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py $cfg --no-profile | tail -1 | cut -c1-90
  done
done

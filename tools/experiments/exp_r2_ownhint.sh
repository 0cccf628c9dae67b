# push: the slot's own accumulator row read / re-zeroed with L2 evict_first (1) or default (0)
for v in oh0 oh1 oh0 oh1; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in oh0 oh1; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
# S23 (bench step: 2048 sources): lane width / pipelines when memory-bound
for cfg in "--lane-words 4 --streams 1" "--lane-words 2 --streams 2" "--lane-words 2 --streams 3" "--lane-words 4 --streams 1"; do
  echo -n "S23 [$cfg]: "; timeout 600 python tools/prof_batch.py --scale 23 --sources 2048 --repeat 2 --no-profile $cfg | tail -1 | cut -c1-100
done

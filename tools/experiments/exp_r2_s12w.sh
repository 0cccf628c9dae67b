# S12 all sources: lane width x pipelines
for w in 8 4 2; do
  for s in 0 4 8; do
    echo -n "S12 W=$w streams=$s: "; timeout 120 python tools/prof_batch.py --scale 12 --all --lane-words $w --streams $s --repeat 5 --no-profile | tail -1 | cut -c1-90
  done
done

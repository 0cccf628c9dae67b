# lane width at S20 after the round-2 forward: W = 4 (K = 256, auto) vs W = 8 (K = 512)
for w in 4 8 4 8; do
  echo -n "W=$w S20 1pipe: "; timeout 300 python tools/prof_batch.py --sources 8192 --lane-words $w --streams 1 --repeat 2 | tail -1 | cut -c1-200
done
for w in 4 8; do
  for s in 2 3; do
  echo -n "W=$w S20 ${s}pipe: "; timeout 300 python tools/prof_batch.py --sources 8192 --lane-words $w --streams $s --repeat 3 --no-profile | tail -1 | cut -c1-80
  done
done

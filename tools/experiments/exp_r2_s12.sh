# S12 all sources: lane width and pipelines (device-driven batches, adaptive tiles)
for lw in 8 4 2; do for ns in 8 4; do
  echo -n "W=$lw NS=$ns: "; timeout 100 python tools/prof_batch.py --scale 12 --all --lane-words $lw --streams $ns --repeat 4 --no-profile | tail -1 | cut -c1-80
done; done

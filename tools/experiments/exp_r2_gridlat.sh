# grid kernel: time per source vs sources in flight (1 .. 8192 consecutive sources; 296 resident CTAs)
for s in 1 2 16 148 296 592 1184 8192; do
  echo -n "grid sources=$s: "; timeout 120 python tools/prof_batch.py --grid 512 --sources $s --consecutive --repeat 3 --no-profile | tail -1 | cut -c1-100
done

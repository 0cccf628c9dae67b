# hub degree threshold (adjacency cut into segments above it; default 4096) after the round-2 kernels
for h in 1024 2048 4096 8192 16384 1024 2048 4096 8192 16384; do echo -n "S20 hub=$h: "; timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --hub $h --repeat 3 --no-profile | tail -1 | cut -c1-80; done

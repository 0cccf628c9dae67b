# pipelines per call after the round-2 kernels (auto: 3 at S20, 8 at S16)
for s in 2 3 4 5; do echo -n "S20 streams=$s: "; timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --streams $s --repeat 3 --no-profile | tail -1 | cut -c1-80; done
for s in 2 3 4 5; do echo -n "S20 streams=$s: "; timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --streams $s --repeat 3 --no-profile | tail -1 | cut -c1-80; done
for s in 3 4 6 8; do echo -n "S16 streams=$s: "; timeout 200 python tools/prof_batch.py --scale 16 --all --lane-words 0 --streams $s --repeat 2 --no-profile | tail -1 | cut -c1-80; done

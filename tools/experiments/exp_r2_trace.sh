# host-side phase times of bc_compute (BC_TRACE=1) on the small and headline configs
export BC_TRACE=1
echo "== S12 all"; timeout 120 python tools/prof_batch.py --scale 12 --all --lane-words 0 --repeat 4 --no-profile 2>&1 | tail -4
echo "== S16 all"; timeout 120 python tools/prof_batch.py --scale 16 --all --lane-words 0 --repeat 3 --no-profile 2>&1 | tail -3
echo "== S20 8192"; timeout 120 python tools/prof_batch.py --scale 20 --sources 8192 --lane-words 0 --repeat 2 --no-profile 2>&1 | tail -2
echo "== grid 8192"; timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --lane-words 0 --repeat 2 --no-profile 2>&1 | tail -2

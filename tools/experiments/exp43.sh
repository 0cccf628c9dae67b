# breadth-first (Cuthill-McKee) relabel (BC_OPT_RELABEL = 2) vs degree relabel on the grid (slices mode)
for r in 1 2 0; do echo -n "relabel=$r "; BC_SO=build_exp/lib_bfsrl.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 --relabel $r | tail -1 | cut -c1-120; done
for r in 1 2; do echo -n "S20 relabel=$r "; BC_SO=build_exp/lib_bfsrl.so timeout 200 python tools/prof_batch.py --sources 4096 --repeat 2 --relabel $r | tail -1 | cut -c1-120; done

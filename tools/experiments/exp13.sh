for v in full0 full1; do echo $v; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 --lane-words 4 | tail -1 | cut -c1-150; done
BC_SO=build_exp/lib_full1.so timeout 120 python tools/prof_batch.py --scale 12 --sources 4096 --repeat 1 --lane-words 4 | tail -1 | cut -c1-150

for v in u2_r2 u4_r1 u4_r2 u3_r1; do echo $v; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --sources 4096 --repeat 2 --lane-words 4 | tail -1; done

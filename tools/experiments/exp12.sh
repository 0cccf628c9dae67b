for v in u2_r2 u1_r1_m3 u1_r2_m3 u2_r1_m3 u1_r1_m4; do echo $v; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 --lane-words 4 | tail -1 | cut -c1-150; done

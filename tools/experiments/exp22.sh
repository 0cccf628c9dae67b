for v in m4r2u1 m4r1u1 m3r4u1 m3r3u1; do echo $v; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 | tail -1 | cut -c1-110; done

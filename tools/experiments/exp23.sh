for v in ${VARIANTS:-head}; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 | tail -1 | cut -c1-110; done

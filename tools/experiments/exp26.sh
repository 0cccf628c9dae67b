timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for v in fr2 fr1 fr1m3 fr2m3; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 | tail -1 | cut -c1-110; done

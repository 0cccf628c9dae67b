timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "slices or grid" 2>&1 | tail -2
for v in p640 p512 p768 p384x3; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done

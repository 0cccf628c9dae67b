timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "slices or grid" 2>&1 | tail -3
for v in c256x4 e256x2 e256x4 e256x5 e256x6 e512x2 e512x3 e384x4; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done

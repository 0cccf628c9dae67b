timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 -k "slices or grid" 2>&1 | tail -3
echo -n "main "; timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100
for v in g256x4 s256x3 s384x3 s512x2 s512x3 s1024x2; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done

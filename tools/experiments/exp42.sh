# 3 CTAs per SM for the shared-memory-state slices kernel (grid 512x512, 8192 sources)
for v in b512m2 b256m3 b384m3 b320m3; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-120; done
for v in b256m3 b384m3; do echo -n "$v parity: "; BC_SO=build_exp/lib_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slices or grid" 2>&1 | tail -1; done

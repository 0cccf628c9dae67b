timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 600 -k "slices or grid" 2>&1 | grep -E "^(FAILED|E )|passed|failed" | head -8
for v in o640 o512 o768 o1024x1; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done

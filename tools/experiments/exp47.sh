# grid kernel discovery: one tail atomic per warp per neighbour group (BC_SM_AGG) vs one per neighbour slot
for v in a0 a1 a0 a1; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done
echo -n "a1 parity: "; BC_SO=build_exp/lib_a1.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slices or grid" 2>&1 | tail -1

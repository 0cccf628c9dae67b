# L2 cache hints in the grid kernel (BC_SM_L2HINT): ELL rows evict-last, queue slot stores evict-first
for v in h0 h1 h0 h1; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done
echo -n "h1 parity: "; BC_SO=build_exp/lib_h1.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slices or grid" 2>&1 | tail -1

# carried ELL rows in queue order (BC_SM_QROW): the level's first load is one 16-byte row per slot
# instead of Q[i] -> ell4[Q[i]] (grid 512x512, 8192 sources, BFS relabel)
for v in qrow0 qrow1 qrow0 qrow1; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-110; done
echo -n "qrow1 parity: "; BC_SO=build_exp/lib_qrow1.so timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "slices or grid" 2>&1 | tail -1

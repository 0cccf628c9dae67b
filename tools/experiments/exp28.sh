python -c "import torch;print('cuda', torch.cuda.is_available(), torch.cuda.device_count())"
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rs --timeout 300 -k "slices or grid" 2>&1 | tail -8
for v in a256x2 a256x4 a128x8 a128x12 a64x16 a64x24 a32x32; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done

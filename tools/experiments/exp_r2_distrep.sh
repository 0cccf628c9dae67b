# the whole NCCL dist test file, repeated (the prune test failed once on a 4-GPU box after the BC test)
nvidia-smi -L
for i in 1 2 3 4 5 6; do echo -n "full $i: "; timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done

# NEXT-4 NCCL test: repeat, then bisect the round's last kernel changes
for i in 1 2 3; do echo -n "cur $i: "; timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k prune 2>&1 | tail -1; done
for v in nobcred noseen m4; do for i in 1 2; do echo -n "$v $i: "; BC_SO=build_exp/lib_$v.so timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k prune 2>&1 | tail -1; done; done
for i in 1 2; do echo -n "cur bc-dist $i: "; timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "not prune" 2>&1 | tail -1; done

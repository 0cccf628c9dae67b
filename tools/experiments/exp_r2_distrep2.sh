# after the fix (share / apply / compute order after the legacy default stream when no stream is given)
for i in 1 2 3 4 5 6 7 8; do echo -n "full $i: "; timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29777 tools/dist_debug.py dist 10 2>&1 | grep -c "bad 0, host-vs-host bad 0"
timeout 600 python -m pytest tests/test_gpu_prune_shares.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1

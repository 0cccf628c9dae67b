for m in dist single; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 100)) tools/dist_debug.py $m 6 2>&1 | grep rank
done

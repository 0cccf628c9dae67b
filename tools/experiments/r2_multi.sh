# multi-GPU on one box: weak-scaling bench lines at N = 2 and 4 (torchrun, NCCL), NCCL dist test
nvidia-smi -L > gpurun_out/multi_gpus.txt
timeout 600 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_dist_nccl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist_nccl.log
port=29511
for N in 2 4; do
  for c in rmat20 grid rmat23; do
    st=10; [ $c = rmat23 ] && st=4
    port=$((port+1))
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus $N --config $c --steps $st --warmup 3 > gpurun_out/bench_r2_${c}_n$N.json 2> gpurun_out/bench_r2_${c}_n$N.err
  done
done

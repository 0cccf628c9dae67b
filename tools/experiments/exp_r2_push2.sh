# per-level push launches of one 256-source S20 batch: group form (c0), compacted rounds (c1), compacted + unpredicated full rounds (c2)
for v in c0 c1 c2; do
  BC_SO=build_exp/lib_$v.so timeout 300 ncu --kernel-name regex:lanes_push_kernel --launch-count 12 \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_op_global_red.sum,lts__t_sectors_op_red.sum \
    python tools/prof_batch.py --sources 256 --streams 1 > gpurun_out/ncu_push2_$v.txt 2>&1
done
for v in c2 c0 c2; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120; done

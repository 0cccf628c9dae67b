# backward push: compacted-lane rounds (BC_PUSH_COMPACT=1) vs 2W lane groups per hit (0), S20 8192 sources, one pipeline
for v in c0 c1 c0 c1; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-260; done
for v in c0 c1; do
  BC_SO=build_exp/lib_$v.so timeout 300 ncu --kernel-name regex:lanes_push_kernel --launch-skip 3 --launch-count 1 \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_op_global_red.sum,lts__t_sectors_op_red.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
    python tools/prof_batch.py --sources 256 > gpurun_out/ncu_push_$v.txt 2>&1
done
echo -n "c1 parity: "; BC_SO=build_exp/lib_c1.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -p no:cacheprovider -k "backward or small_suite or config4 or capture or two_degree or sigma" 2>&1 | tail -1

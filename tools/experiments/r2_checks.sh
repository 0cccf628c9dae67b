# (1) the -m gpu suite against the bounds-checked build; (2) grid kernel next-slot prefetch A/B
BC_SO=build_exp/lib_chk.so timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2_checks.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_r2_checks.log
bash tools/experiments/exp_r2_pf.sh > gpurun_out/exp_r2_pf.txt 2>&1

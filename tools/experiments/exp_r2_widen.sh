# per-level sigma widening (host-driven loop): parity + S23 step timing
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "widens or narrow or sigma or device_loop or two_degree" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "rmat23" 2>&1 | tail -2
timeout 900 python bench.py --config rmat23 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_widen_s23.json 2> gpurun_out/bench_widen_s23.err; tail -c 600 gpurun_out/bench_widen_s23.json

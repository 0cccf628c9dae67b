timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "widens or narrow or sigma or device_loop or two_degree" 2>&1 | grep -E "Error|error|assert|^E |FAILED|passed|failed" | head -40
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -p no:cacheprovider -k "rmat23" 2>&1 | grep -E "Error|error|assert|^E |FAILED|passed|failed" | head -30

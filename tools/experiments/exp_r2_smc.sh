# grid 512x512: shared-state kernel (4) vs + shared frontier ring and sigma/coef cache (5)
for sk in 4 5 4 5; do
  echo -n "sk=$sk consecutive: "; timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --consecutive --slices-kernel $sk --repeat 2 --no-profile | tail -1 | cut -c1-100
done
for sk in 4 5; do
  echo -n "sk=$sk sampled: "; timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --slices-kernel $sk --repeat 2 --no-profile | tail -1 | cut -c1-100
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -x -p no:cacheprovider -k "slices or capture_small" 2>&1 | tail -2

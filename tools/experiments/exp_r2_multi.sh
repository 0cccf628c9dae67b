# grid 512x512: one source per CTA (slices kernel 4, default) vs 4 / 8 sources per CTA in lockstep (5 / 6)
for sk in 4 5 6 4 5 6; do
  echo -n "sk=$sk consecutive: "; timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --consecutive --slices-kernel $sk --repeat 2 --no-profile | tail -1 | cut -c1-100
done
for sk in 4 5 6; do
  echo -n "sk=$sk sampled: "; timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --slices-kernel $sk --repeat 2 --no-profile | tail -1 | cut -c1-100
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -x -p no:cacheprovider -k "slices or capture or device_loop or stream" 2>&1 | tail -2

# forward commit: mask words by OR-reductions (gr1) vs ballots + interleave (gr0)
for v in gr0 gr1 gr0 gr1; do
  echo -n "$v S20 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-120
done
for v in gr0 gr1; do
  echo -n "$v S16 1pipe: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --sources 16384 --streams 1 --lane-words 8 --repeat 2 | tail -1 | cut -c1-120
done
echo -n "gr1 parity: "; BC_SO=build_exp/lib_gr1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1

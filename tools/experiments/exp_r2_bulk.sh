# forward gathers: bulk copies into a per-warp ring (BC_FWD_BULK=1) vs per-thread loads (0); tile sizing factor
for v in bulk0 bulk1 bulk0 bulk1; do
  echo -n "$v S20: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --streams 1 --repeat 2 | tail -1 | cut -c1-140
done
for v in bulk0 bulk1; do
  echo -n "$v S16: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --scale 16 --sources 16384 --streams 1 --lane-words 8 --repeat 2 | tail -1 | cut -c1-140
done
for v in tf1 bulk0 tf4 tf8; do
  for cfg in "--scale 12 --all --lane-words 0 --repeat 3" "--scale 16 --all --lane-words 0 --repeat 2"; do
    echo -n "$v $cfg: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py $cfg --no-profile | tail -1 | cut -c1-90
  done
done
echo -n "bulk1 parity: "; BC_SO=build_exp/lib_bulk1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1

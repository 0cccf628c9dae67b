# W = 4 level kernel at 5 CTAs per SM: whole step (3 pipelines) and parity
for v in m4 m5 m4 m5; do
  echo -n "$v S20 auto: "; BC_SO=build_exp/lib_$v.so timeout 200 python tools/prof_batch.py --sources 8192 --lane-words 0 --repeat 3 --no-profile | tail -1 | cut -c1-80
done
echo -n "m5 suite: "; BC_SO=build_exp/lib_m5.so timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1

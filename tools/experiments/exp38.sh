for v in q640 q512; do echo -n "$v "; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100; done
echo -n "main "; timeout 120 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-100

for v in sl256 sl512 sl1024; do echo $v; BC_SO=build_exp/lib_$v.so timeout 300 python tools/prof_batch.py --grid 512 --sources 8192 --repeat 2 | tail -1 | cut -c1-120; done

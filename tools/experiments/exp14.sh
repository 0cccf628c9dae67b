for v in hot0 hot16384 hot32768 hot65536; do echo $v; BC_SO=build_exp/lib_$v.so timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 --lane-words 4 | tail -1 | cut -c1-150; done

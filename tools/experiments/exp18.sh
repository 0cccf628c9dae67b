for o in 2 3; do echo order=$o; timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 --order $o | tail -1 | cut -c1-250; done

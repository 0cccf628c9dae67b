timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -3
for w in 4 2; do timeout 120 python tools/prof_batch.py --sources 4096 --repeat 2 --lane-words $w | tail -1; done

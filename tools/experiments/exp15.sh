timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2
timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 --lane-words 4 | tail -1 | cut -c1-150

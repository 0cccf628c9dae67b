timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 | tail -1 | cut -c1-150

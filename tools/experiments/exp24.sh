timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3
for b in 1 2; do timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 --bwd $b | tail -1 | cut -c1-150; done

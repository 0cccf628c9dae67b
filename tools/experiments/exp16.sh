timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 -k "slices or grid or stats" 2>&1 | tail -2
timeout 300 python tools/prof_batch.py --grid 512 --sources 4096 --repeat 2 | tail -1 | cut -c1-160
timeout 300 python tools/prof_batch.py --scale 16 --sources 4096 --repeat 2 --lane-words 4 | tail -1 | cut -c1-160

timeout 300 python -m pytest tests -m gpu -q -x --timeout 120 2>&1 | tail -2
for fp in 0 1 2; do echo fwdpush=$fp; timeout 120 python tools/prof_batch.py --sources 8192 --repeat 2 --fwd-push $fp | tail -1 | cut -c1-170; done

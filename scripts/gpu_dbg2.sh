export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_dist.py -m gpu -q --timeout 300 -x 2>&1 | tail -15

timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | grep -v "^  " | head -60

#!/bin/bash
# E5 native: word-wise ragged-edge stores. Tests + DiT sweep.
timeout 900 python -m pytest tests/test_e5m2.py -q -x -m gpu 2>&1 | tail -n 1
timeout 900 python bench.py --workload dit-e5m2 2>&1 >/dev/null | grep "dit-e5m2"

#!/bin/bash
# Variant 7 by load-ahead (main) vs at tile start (la0): parity + bench A/B.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_hooks.py -q -x -m gpu 2>&1 | tail -n 2
for v in main la0 main2 la0b; do
  unset ECF8_LIB; case $v in la0*) export ECF8_LIB=build/var/la0/libecf8_b200.so;; esac
  echo "== $v"; timeout 600 python bench.py --steps 20 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['verified_bit_exact'], d['clocks'])"
done

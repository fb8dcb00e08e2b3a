#!/bin/bash
# A/B on variant 7: section prefetch per tile vs windows only vs grouped.
for v in main pfw pg2 pg4 pg8a48 main2; do
  unset ECF8_LIB; case $v in main|main2) ;; *) export ECF8_LIB=build/var/$v/libecf8_b200.so;; esac
  echo "== $v"; timeout 600 python bench.py --steps 20 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['verified_bit_exact'], d['clocks'])"
done

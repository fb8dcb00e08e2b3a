#!/bin/bash
# A/B: L2 prefetch of the tile sections in groups (G tiles, AHEAD tiles ahead) vs per tile; direct-only kernel.
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -n 1
for v in main pf1 pf16 pf8a64 d28 d26 main2 pf1b; do
  unset ECF8_LIB ECF8_DIRECT_KERNEL
  case $v in pf1|pf16|pf8a64) export ECF8_LIB=build/var/$v/libecf8_b200.so;; pf1b) export ECF8_LIB=build/var/pf1/libecf8_b200.so;;
    d28) export ECF8_DIRECT_KERNEL=1;; d26) export ECF8_DIRECT_KERNEL=1 ECF8_LIB=build/var/d26/libecf8_b200.so;; esac
  echo "== $v"; timeout 600 python bench.py --steps 20 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['verified_bit_exact'], d['clocks'])"
done

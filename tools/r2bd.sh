#!/bin/bash
# A/B: direct-only decode kernel (per-tile prefetch) at 24/26/28/30 warps vs the default.
for v in main d28 d26 d24 d30 main2 d28b; do
  unset ECF8_LIB ECF8_DIRECT_KERNEL
  case $v in d28|d28b) export ECF8_DIRECT_KERNEL=1;; d26|d24|d30) export ECF8_DIRECT_KERNEL=1 ECF8_LIB=build/var/$v/libecf8_b200.so;; esac
  echo "== $v"; timeout 600 python bench.py --steps 20 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['verified_bit_exact'], d['clocks'])"
done

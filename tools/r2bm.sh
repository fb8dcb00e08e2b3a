#!/bin/bash
# A/B: lazy endgap words + no direct-bit load in variant 7 (main) vs before (prev); parity subset.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fused_large.py -q -x -m gpu 2>&1 | tail -n 1
for v in main prev main2 prev2; do
  unset ECF8_LIB; case $v in prev*) export ECF8_LIB=build/var/prev/libecf8_b200.so;; esac
  echo "== $v"; timeout 600 python bench.py --steps 20 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['verified_bit_exact'], d['clocks'])"
done
unset ECF8_LIB
export ECF8_BENCH_FUSED_MS=1,256
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="

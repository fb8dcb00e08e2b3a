#!/bin/bash
# Fused A/B after the lazy endgap load: main vs prev (before), twice.
export ECF8_BENCH_FUSED_MS=1,64,256
for v in main prev main2 prev2; do
  unset ECF8_LIB; case $v in prev*) export ECF8_LIB=build/var/prev/libecf8_b200.so;; esac
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done

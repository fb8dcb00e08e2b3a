#!/bin/bash
# A/B: fused ring-writer poll interval.
export ECF8_BENCH_FUSED_MS=1,64,256
for v in main ss256 ss1000 main2; do
  unset ECF8_LIB; case $v in ss*) export ECF8_LIB=build/var/$v/libecf8_b200.so;; esac
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done

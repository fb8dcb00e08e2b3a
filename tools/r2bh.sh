#!/bin/bash
# Timing probes of the L2-ring fused kernel: without MMAs, without ring stores.
export ECF8_BENCH_FUSED_MS=1,256
for v in main probe1 probe2; do
  unset ECF8_LIB; case $v in probe*) export ECF8_LIB=build/var/$v/libecf8_b200.so;; esac
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done

#!/bin/bash
# A/B: fused rings as an L2 persisting window.
export ECF8_BENCH_FUSED_MS=1,64,256
for v in 0 40 64 0b; do
  unset ECF8_FUSED_L2_PERSIST_MB; case $v in 40|64) export ECF8_FUSED_L2_PERSIST_MB=$v;; esac
  echo "== persist $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
done

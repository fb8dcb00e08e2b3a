#!/bin/bash
# A/B: mid-run flushes by 8 decode warps (main) vs 4 (fw4); fused tests.
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py -q -x -m gpu 2>&1 | tail -n 1
export ECF8_BENCH_FUSED_MS=1,64,256
for v in main fw4 main2 fw4b; do
  unset ECF8_LIB; case $v in fw4*) export ECF8_LIB=build/var/fw4/libecf8_b200.so;; esac
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done

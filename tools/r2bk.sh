#!/bin/bash
# Fused: final flush by all decode warps vs warps 0-3; decompress phase times.
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py -q -x -m gpu 2>&1 | tail -n 1
export ECF8_BENCH_FUSED_MS=1,64,256
for v in main fin0 main2; do
  unset ECF8_LIB; case $v in fin0) export ECF8_LIB=build/var/$v/libecf8_b200.so;; esac
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done
unset ECF8_LIB
ECF8_DIAG_DECOMPRESS=1 timeout 600 python tools/decompress_probe.py 8 2>&1 | tail -n 12

#!/bin/bash
# Fused slowdown hunt: m in {1, 16, 64} (no accumulator reuse), variants of the flush polling.
export ECF8_BENCH_FUSED_MS=1,16,64
for v in main old nopoll nomid neither; do
  if [ $v = main ]; then unset ECF8_LIB; else export ECF8_LIB=build/var/$v/libecf8_b200.so; fi
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
done

#!/bin/bash
export ECF8_BENCH_FUSED_MS=1,256
for v in main r32 r8 r64; do
  if [ $v = main ]; then unset ECF8_LIB; else export ECF8_LIB=build/var/$v/libecf8_b200.so; fi
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done

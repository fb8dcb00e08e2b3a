#!/bin/bash
export ECF8_BENCH_FUSED_MS=1,64,256
for v in noepi nox nomma noxmma; do
  export ECF8_LIB=build/var/$v/libecf8_b200.so
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
done

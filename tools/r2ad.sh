#!/bin/bash
for v in s12 s14 s16 g12; do
  export ECF8_LIB=build/var/$v/libecf8_b200.so
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
done

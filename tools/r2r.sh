#!/bin/bash
# Fused GEMM A/B: staged vs L2 packed bytes (GPK), watcher warp + 2 X stages (WATCH), decode warps.
mkdir -p gpurun_out
for v in main g1w1 g0w1 g1w0 g1w1w16; do
  if [ $v = main ]; then unset ECF8_LIB; else export ECF8_LIB=build/var/$v/libecf8_b200.so; fi
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
done

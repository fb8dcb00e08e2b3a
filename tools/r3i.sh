#!/bin/bash
# A/B: fused GEMM write-back unroll 4 (main) vs 2 vs 3.
mkdir -p gpurun_out
TAG=r3i
for lib in main build/var/fwb2/libecf8_b200.so build/var/fwb3/libecf8_b200.so main build/var/fwb2/libecf8_b200.so build/var/fwb3/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib" | tee -a gpurun_out/${TAG}_ab.txt
  timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m=" | tee -a gpurun_out/${TAG}_ab.txt
done

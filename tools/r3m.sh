#!/bin/bash
# A/B: fused decode warps 23 (main) vs 21 vs 25, with the FMA-pipe sink.
mkdir -p gpurun_out
TAG=r3m
for lib in main build/var/fw21/libecf8_b200.so build/var/fw25/libecf8_b200.so main build/var/fw21/libecf8_b200.so build/var/fw25/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib" | tee -a gpurun_out/${TAG}_ab.txt
  timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m=" | tee -a gpurun_out/${TAG}_ab.txt
done

#!/bin/bash
# A/B: native E5M2 write-back loop unrolled 1 (main) / 2 / 4 / 8 (raw-plane loads in flight together); DiT sweep.
mkdir -p gpurun_out
TAG=r3h
for lib in main build/var/e5u2/libecf8_b200.so build/var/e5u4/libecf8_b200.so build/var/e5u8/libecf8_b200.so main build/var/e5u4/libecf8_b200.so build/var/e5u8/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib" | tee -a gpurun_out/${TAG}_ab.txt
  timeout 600 python bench.py --workload dit-e5m2 2>&1 >/dev/null | grep "native" | tee -a gpurun_out/${TAG}_ab.txt
done

#!/bin/bash
# A/B: fused decode warps' L2 prefetch addresses from the section table (fpftab) vs main; fused parity under fpftab.
mkdir -p gpurun_out
TAG=r3p
for lib in main build/var/fpftab/libecf8_b200.so main build/var/fpftab/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib" | tee -a gpurun_out/${TAG}_ab.txt
  timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m=" | tee -a gpurun_out/${TAG}_ab.txt
done
ECF8_LIB=build/var/fpftab/libecf8_b200.so timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py -m gpu -q -x 2>&1 | tail -n 2 | tee -a gpurun_out/${TAG}_ab.txt

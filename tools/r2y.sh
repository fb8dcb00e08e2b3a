#!/bin/bash
export ECF8_BENCH_FUSED_MS=64,256
for v in main noepi; do
  if [ $v = main ]; then unset ECF8_LIB; else export ECF8_LIB=build/var/$v/libecf8_b200.so; fi
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
done
unset ECF8_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_gemm -s 2 -c 1 -o gpurun_out/r2y_fused_m256 python tools/fused_one.py 28672 8192 256 3 > /dev/null 2>&1

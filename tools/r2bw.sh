#!/bin/bash
# A/B: mid-run flush warps at m > 64: 8 (main) / 12 / 16; at m <= 64: 4 (main) / 8 (fs8). Fused tests first.
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py -q -x -m gpu 2>&1 | tail -n 1
export ECF8_BENCH_FUSED_MS=1,64,256
for v in main fw12 fw16 fs8 main2; do
  unset ECF8_LIB; case $v in fw*|fs*) export ECF8_LIB=build/var/$v/libecf8_b200.so;; esac
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done

#!/bin/bash
# Fused GEMM at m=256: epilogue cost (no y updates) and the cost of a second wave (m <= 128 forced to 2 waves).
echo "== main"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
echo "== noepi"; ECF8_LIB=build/var/noepi/libecf8_b200.so timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
echo "== 2 waves"; ECF8_FUSED_MIN_WAVES=2 timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2p}
for v in g0w0 g0w1 g1w0 g1w1w12; do echo "variant $v"; ECF8_LIB=build/var/$v/libecf8_b200.so timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="; done

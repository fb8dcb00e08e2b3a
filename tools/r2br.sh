#!/bin/bash
# Variant 7 on the other decode workloads; fused ncu at M=16 / 64 (tensor pipe, DRAM per M).
mkdir -p gpurun_out
TAG=r2br
timeout 900 python bench.py --workload llama3.1-8b > gpurun_out/${TAG}_8b.json 2> gpurun_out/${TAG}_8b.err; head -c 400 gpurun_out/${TAG}_8b.json; echo
timeout 900 python bench.py --workload deepseek-v3-experts > gpurun_out/${TAG}_dsv3.json 2> gpurun_out/${TAG}_dsv3.err; head -c 400 gpurun_out/${TAG}_dsv3.json; echo
for m in 16 64; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 2 -c 1 -o gpurun_out/${TAG}_fused_m$m python tools/fused_one.py 28672 8192 $m 3 > /dev/null 2>&1
done
ls gpurun_out/${TAG}_*

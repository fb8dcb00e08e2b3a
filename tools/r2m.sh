#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2m}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_pytest.log | head -20
for m in 1 256; do
ncu --set full --clock-control none --import-source on -k regex:fused_gemm -s 2 -c 1 -o gpurun_out/${TAG}_fused_m$m \
    python tools/fused_one.py 28672 8192 $m 3 > gpurun_out/${TAG}_ncu_m$m.log 2>&1; tail -1 gpurun_out/${TAG}_ncu_m$m.log
done

#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2n}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_pytest.log | head -20
python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/${TAG}_fused.json 2> gpurun_out/${TAG}_fused.err; grep "fused m=" gpurun_out/${TAG}_fused.err
for v in fw12 fw20; do echo "variant $v"; ECF8_LIB=build/var/$v/libecf8_b200.so python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="; done
ncu --set full --clock-control none --import-source on -k regex:fused_gemm -s 2 -c 1 -o gpurun_out/${TAG}_fused_m1 python tools/fused_one.py 28672 8192 1 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_gemm -s 2 -c 1 -o gpurun_out/${TAG}_fused_m256 python tools/fused_one.py 28672 8192 256 3 > /dev/null 2>&1
ls gpurun_out/${TAG}_*

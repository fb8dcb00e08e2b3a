#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2l}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_pytest.log | head -20
python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/${TAG}_fused.json 2> gpurun_out/${TAG}_fused.err; grep "fused m=" gpurun_out/${TAG}_fused.err
ECF8_FUSED_NO_FSM=1 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2f}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_pytest.log | head -20
python bench.py --steps 20 --warmup 5 --cpu-seconds 0 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cut -c1-300 gpurun_out/${TAG}_bench.json; grep -o '"e2e": {[^}]*}' gpurun_out/${TAG}_bench.json

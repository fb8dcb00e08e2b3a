#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-r2h}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/${TAG}_pytest.log | head -20
for nw in 24; do
ECF8_WARPS=$nw python bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/${TAG}_bench_w$nw.json 2> gpurun_out/${TAG}_bench.err; echo "warps $nw"; cut -c1-200 gpurun_out/${TAG}_bench_w$nw.json
ECF8_WARPS=$nw python bench.py --workload llama3.1-8b --steps 20 --warmup 5 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | cut -c1-160
done
ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 5 -c 1 -o gpurun_out/${TAG}_full \
    python bench.py --workload llama3.1-8b --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log

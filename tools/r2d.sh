#!/bin/bash
# FSM decoder: parity + bench + ncu
mkdir -p gpurun_out
TAG=${1:-r2d}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${TAG}_pytest.log
python bench.py --steps 20 --warmup 5 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json | cut -c1-400
python bench.py --workload llama3.1-8b --steps 20 --warmup 5 --e2e-steps 0 --cpu-seconds 0 > gpurun_out/${TAG}_bench8b.json 2>&1; tail -1 gpurun_out/${TAG}_bench8b.json | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 5 -c 1 -o gpurun_out/${TAG}_full \
    python bench.py --workload llama3.1-8b --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log

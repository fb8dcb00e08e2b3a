#!/bin/bash
mkdir -p gpurun_out
TAG=r2c
timeout 900 compute-sanitizer --tool racecheck --num-cuda-barriers 32 --target-processes all --print-limit 20 python tools/sanitize_cases.py fused > gpurun_out/${TAG}_san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/${TAG}_san_racecheck.log
s=$(date +%s); python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench wall $(( $(date +%s) - s ))s"; cat gpurun_out/${TAG}_bench.json
s=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref wall $(( $(date +%s) - s ))s"; cat gpurun_out/${TAG}_ref.json; tail -3 gpurun_out/${TAG}_ref.err

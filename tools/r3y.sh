#!/bin/bash
# Full ncu capture of the decode kernel on the final build (source lines match the tree).
mkdir -p gpurun_out
TAG=r3y
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 5 -c 1 -o gpurun_out/${TAG}_full \
    python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 0 --e2e-steps 0 2>/dev/null | tail -c 300

#!/bin/bash
# 8 mid-run flush warps (constant): fused tests + verified sweep + racecheck/memcheck on the fused cases.
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py tests/test_hooks.py tests/test_tp.py -q -m gpu 2>&1 | tail -n 2
timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/r2bx_fused.json 2> gpurun_out/r2bx_fused.err; grep "fused m=" gpurun_out/r2bx_fused.err
for tool in memcheck racecheck; do
  extra=""; [ $tool = racecheck ] && extra="--num-cuda-barriers 32"
  timeout 1200 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 python tools/sanitize_cases.py fused > gpurun_out/r2bx_san_${tool}_fused.log 2>&1
  echo "$tool fused rc=$?"; tail -n 1 gpurun_out/r2bx_san_${tool}_fused.log
done

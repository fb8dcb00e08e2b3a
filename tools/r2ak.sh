#!/bin/bash
# Sanitizers on the current kernels + the production caller's throughput.
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r2ak_san_${tool}.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -n 2 gpurun_out/r2ak_san_${tool}.log
done
for part in decode encode e5; do
  timeout 1200 compute-sanitizer --tool racecheck --target-processes all --print-limit 50 python tools/sanitize_cases.py $part > gpurun_out/r2ak_san_racecheck_${part}.log 2>&1
  echo "racecheck $part rc=$?"; tail -n 2 gpurun_out/r2ak_san_racecheck_${part}.log
done
timeout 1200 compute-sanitizer --tool racecheck --num-cuda-barriers 32 --target-processes all --print-limit 20 python tools/sanitize_cases.py fused > gpurun_out/r2ak_san_racecheck_fused.log 2>&1
echo "racecheck fused rc=$?"; tail -n 2 gpurun_out/r2ak_san_racecheck_fused.log
timeout 900 python tools/decompress_probe.py 8 > gpurun_out/r2ak_decompress.json 2> gpurun_out/r2ak_decompress.err; cat gpurun_out/r2ak_decompress.json; tail -n 2 gpurun_out/r2ak_decompress.err

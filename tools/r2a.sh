#!/bin/bash
# round-2 GPU call A: full GPU suite (incl. large fused parity), sanitizers, bench
mkdir -p gpurun_out
TAG=r2a
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/${TAG}_pytest.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python tools/sanitize_cases.py > gpurun_out/${TAG}_san_${tool}.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -4 gpurun_out/${TAG}_san_${tool}.log
done
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 600 gpurun_out/${TAG}_bench.json

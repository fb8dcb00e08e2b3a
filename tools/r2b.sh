#!/bin/bash
# round-2 GPU call B: racecheck of the fused GEMM after the free-barrier change, 70B default bench + reference arm
mkdir -p gpurun_out
TAG=r2b
timeout 600 python -m pytest tests/test_fused.py tests/test_fused_large.py -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 compute-sanitizer --tool racecheck --target-processes all --print-limit 50 python tools/sanitize_cases.py fused > gpurun_out/${TAG}_san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/${TAG}_san_racecheck.log
/usr/bin/time -v python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json; grep -E "Elapsed|Maximum resident" gpurun_out/${TAG}_bench.err
/usr/bin/time -v python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; cat gpurun_out/${TAG}_ref.json; grep -E "Elapsed|Maximum resident" gpurun_out/${TAG}_ref.err

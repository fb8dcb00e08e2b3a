#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ae_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ae_pytest.log
timeout 600 python bench.py > gpurun_out/r2ae_bench.json 2> gpurun_out/r2ae_bench.err; cat gpurun_out/r2ae_bench.json
timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/r2ae_fused.json 2> gpurun_out/r2ae_fused.err; grep "fused m=" gpurun_out/r2ae_fused.err

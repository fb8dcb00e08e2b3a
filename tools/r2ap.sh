#!/bin/bash
timeout 1200 python -m pytest tests/test_fused.py tests/test_fused_large.py tests/test_fused_container.py tests/test_tp.py tests/test_hooks.py -m gpu -q -x > gpurun_out/r2ap_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 15 gpurun_out/r2ap_pytest.log
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/r2ap_fused.json 2> gpurun_out/r2ap_fused.err; grep "fused m=" gpurun_out/r2ap_fused.err
ECF8_BENCH_FUSED_MS=64,128,129,256 ECF8_FUSED_LARGE_M=64 timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

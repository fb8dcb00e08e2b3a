#!/bin/bash
# Fused GEMM with accumulator reuse (one-wave plans): tests + bench.
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py tests/test_fused_container.py tests/test_tp.py -m gpu -q -x > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2u_pytest.log
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
echo "== seg cap 2 (old plans)"; ECF8_FUSED_SEG_CAP=2 timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

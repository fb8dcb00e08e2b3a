#!/bin/bash
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py tests/test_fused_container.py tests/test_tp.py tests/test_hooks.py -m gpu -q -x > gpurun_out/r2aw_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 15 gpurun_out/r2aw_pytest.log
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
echo "== smem ring"; ECF8_FUSED_L2=0 timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

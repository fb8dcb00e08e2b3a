#!/bin/bash
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py tests/test_fused_container.py tests/test_tp.py tests/test_hooks.py -m gpu -q -x > gpurun_out/r2ac_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ac_pytest.log
for v in main w20 w16 w24x2; do
  if [ $v = main ]; then unset ECF8_LIB; else export ECF8_LIB=build/var/$v/libecf8_b200.so; fi
  echo "== $v"; timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
done

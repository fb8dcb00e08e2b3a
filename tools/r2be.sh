#!/bin/bash
# Variant 7 (direct-only decode kernel) default: GPU suite + bench A/B against variant 4.
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2be_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2be_pytest.log
for v in v7 v4 v7b v4b; do
  unset ECF8_NO_DIRECT_KERNEL; case $v in v4|v4b) export ECF8_NO_DIRECT_KERNEL=1;; esac
  echo "== $v"; timeout 600 python bench.py --steps 20 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['verified_bit_exact'], d['clocks'], d['roofline']['kernel'])"
done

#!/bin/bash
timeout 900 python -m pytest tests/test_e5m2.py tests/test_capi.py -m gpu -q -x > gpurun_out/r2ar_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 15 gpurun_out/r2ar_pytest.log
timeout 900 python bench.py --workload dit-e5m2 --steps 10 --warmup 3 > gpurun_out/r2ar_dit.json 2> gpurun_out/r2ar_dit.err; grep "native" gpurun_out/r2ar_dit.err

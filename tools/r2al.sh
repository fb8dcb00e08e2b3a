#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_encode_device.py -m gpu -q -x > gpurun_out/r2al_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 15 gpurun_out/r2al_pytest.log
timeout 900 python bench.py --workload dit-e5m2 --steps 10 --warmup 3 > gpurun_out/r2al_dit.json 2> gpurun_out/r2al_dit.err; grep "dit-e5m2" gpurun_out/r2al_dit.err

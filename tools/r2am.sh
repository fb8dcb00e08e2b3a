#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2am_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2am_pytest.log
timeout 900 python tools/decompress_probe.py 8 > gpurun_out/r2am_decompress.json 2> gpurun_out/r2am_decompress.err; cat gpurun_out/r2am_decompress.json
timeout 600 python bench.py --steps 10 > gpurun_out/r2am_bench.json 2> /dev/null; python -c "import json; d=json.load(open('gpurun_out/r2am_bench.json')); print(d['value'], d['e2e'])"

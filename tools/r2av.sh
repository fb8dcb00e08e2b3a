#!/bin/bash
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2av_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r2av_pytest.log
timeout 900 python tools/decompress_probe.py 8 > gpurun_out/r2av_decompress.json 2> gpurun_out/r2av_decompress.err; cat gpurun_out/r2av_decompress.json; tail -n 2 gpurun_out/r2av_decompress.err

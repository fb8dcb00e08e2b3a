#!/bin/bash
# Deferred ring arrivals (fence after the next decode phase): fused tests + sweep.
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py -q -x -m gpu 2>&1 | tail -n 2
export ECF8_BENCH_FUSED_MS=1,16,64,256
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

#!/bin/bash
# Shared per-stream fused workspace + ring-write wait: fused tests, sanitizer (memcheck) on fused, fused sweep.
timeout 900 python -m pytest tests/test_fused.py tests/test_fused_large.py tests/test_hooks.py tests/test_tp.py -q -x -m gpu 2>&1 | tail -n 2
timeout 900 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 python tools/sanitize_cases.py fused 2>&1 | tail -n 2
timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

#!/bin/bash
# Pinned-arena decompress_streaming + fused final flush: GPU suite, decompress probe.
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -n 2
ECF8_DIAG_DECOMPRESS=1 timeout 600 python tools/decompress_probe.py 8 2>&1 | tail -n 5

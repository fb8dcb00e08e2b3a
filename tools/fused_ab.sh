#!/bin/bash
# A/B of library variants on the fused GEMM probe (gate/up and down at m=1, 256).
for lib in "$@"; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib"
  python tools/fused_probe.py 1 256 2>&1 | grep "gate/up\|down" | sed 's/(.*split_k [0-9])//'
done

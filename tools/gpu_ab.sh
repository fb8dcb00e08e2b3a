#!/bin/bash
# A/B of library variants on the probe workload (8 x 14336x4096, T 256).
# usage: bash tools/gpu_ab.sh TAG "main build/var/x/libecf8_b200.so ..." [probe args]
TAG=$1; LIBS=$2; shift 2
mkdir -p gpurun_out
for lib in $LIBS; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib $ECF8_AB_ENV" >> gpurun_out/${TAG}_ab.txt
  env $ECF8_AB_ENV python tools/probe.py "$@" 2>&1 | grep -v synth >> gpurun_out/${TAG}_ab.txt
done
cat gpurun_out/${TAG}_ab.txt

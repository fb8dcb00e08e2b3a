#!/bin/bash
mkdir -p gpurun_out
TAG=r3f
for lib in main build/var/wbu8/libecf8_b200.so build/var/wbs8/libecf8_b200.so build/var/wbs12/libecf8_b200.so build/var/wbu12/libecf8_b200.so main build/var/wbu8/libecf8_b200.so build/var/wbs8/libecf8_b200.so build/var/wbs12/libecf8_b200.so build/var/wbu12/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  b=$(timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 0 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['verified_bit_exact'], d['clocks'])")
  p=$(timeout 300 python tools/probe.py --n 28672000 --count 16 2>&1 | grep bit-exact | sed 's/.*T=256: //')
  echo "$lib | bench $b | probe $p" | tee -a gpurun_out/${TAG}_ab.txt
done
unset ECF8_LIB

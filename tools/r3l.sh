#!/bin/bash
# A/B: the pair join's second high multiply by a constant-bank 2^16 (IMAD.HI instead of LEA.HI) vs main.
mkdir -p gpurun_out
TAG=r3l
for lib in main build/var/jconst/libecf8_b200.so main build/var/jconst/libecf8_b200.so main build/var/jconst/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  b=$(timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 0 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['verified_bit_exact'], d['clocks'])")
  p=$(timeout 300 python tools/probe.py --n 28672000 --count 16 2>&1 | grep bit-exact | sed 's/.*T=256: //')
  echo "$lib | bench $b | probe $p" | tee -a gpurun_out/${TAG}_ab.txt
done
for lib in main build/var/jconst/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib" | tee -a gpurun_out/${TAG}_ab.txt
  timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m=" | tee -a gpurun_out/${TAG}_ab.txt
done

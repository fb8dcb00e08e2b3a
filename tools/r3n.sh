#!/bin/bash
# A/B: L2 prefetch addresses from a per-segment section table (pftab) vs main; parity under pftab.
mkdir -p gpurun_out
TAG=r3n
for lib in main build/var/pftab/libecf8_b200.so main build/var/pftab/libecf8_b200.so main build/var/pftab/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  b=$(timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 0 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['verified_bit_exact'], d['clocks'])")
  p=$(timeout 300 python tools/probe.py --n 28672000 --count 16 2>&1 | grep bit-exact | sed 's/.*T=256: //')
  echo "$lib | bench $b | probe $p" | tee -a gpurun_out/${TAG}_ab.txt
done
for lib in main build/var/pftab/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  echo "== $lib" | tee -a gpurun_out/${TAG}_ab.txt
  timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m=" | tee -a gpurun_out/${TAG}_ab.txt
done
ECF8_LIB=build/var/pftab/libecf8_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x 2>&1 | tail -n 2 | tee -a gpurun_out/${TAG}_ab.txt

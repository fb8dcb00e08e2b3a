#!/bin/bash
# PCIe chunking probe; A/B of the IMAD.HI pair join (main) vs the plain shifts (ECF8_JOIN_ALU=1).
mkdir -p gpurun_out
TAG=r3b
timeout 300 python tools/pcie_probe3.py 2>&1 | grep -v Warn | tee gpurun_out/${TAG}_pcie3.log
for lib in main build/var/joinalu/libecf8_b200.so main build/var/joinalu/libecf8_b200.so; do
  if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
  b=$(timeout 600 python bench.py --steps 5 --warmup 3 --cpu-seconds 0 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['verified_bit_exact'], d['clocks'])")
  echo "$lib | bench $b" | tee -a gpurun_out/${TAG}_ab.txt
  p=$(timeout 300 python tools/probe.py --n 28672000 --count 16 2>&1 | grep bit-exact)
  echo "$lib | probe $p" | tee -a gpurun_out/${TAG}_ab.txt
done

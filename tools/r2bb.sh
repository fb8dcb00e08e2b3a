#!/bin/bash
# A/B: direct-only decode kernel (slot-less warp state) at 26/28/32 warps vs the default 24; fused ring-mask sink.
for v in main d28 d26 d32; do
  unset ECF8_LIB ECF8_DIRECT_KERNEL
  case $v in d28) export ECF8_DIRECT_KERNEL=1;; d26|d32) export ECF8_DIRECT_KERNEL=1 ECF8_LIB=build/var/$v/libecf8_b200.so;; esac
  echo "== $v"; timeout 600 python bench.py --steps 20 --e2e-steps 0 --cpu-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['verified_bit_exact'], d['clocks'])"
done
unset ECF8_LIB ECF8_DIRECT_KERNEL
export ECF8_BENCH_FUSED_MS=1,256
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="

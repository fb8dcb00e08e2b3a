#!/bin/bash
# A/B: bench value + probe for each library variant and warp count.
# usage: bash tools/ab.sh "main build/var/wb4/libecf8_b200.so ..." "20 16"
for lib in $1; do
  for nw in $2; do
    if [ "$lib" = main ]; then unset ECF8_LIB; else export ECF8_LIB=$lib; fi
    export ECF8_WARPS=$nw
    p=$(python tools/probe.py 2>&1 | grep bit-exact | sed 's/.*T=256: //')
    b=$(python bench.py --steps 10 --cpu-seconds 0 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['config']['verified_bit_exact'])")
    echo "$lib warps=$nw | probe $p | bench $b"
  done
done

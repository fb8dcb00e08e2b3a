#!/bin/bash
for rep in 1 2; do
for v in main wbloop p6 p12; do
  if [ $v = main ]; then unset ECF8_LIB; else export ECF8_LIB=build/var/$v/libecf8_b200.so; fi
  echo -n "$v: "; timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --cpu-seconds 0 --no-verify 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done

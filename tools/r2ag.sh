#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2ag_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ag_pytest.log
for rep in 1 2; do
for v in main clip; do
  if [ $v = main ]; then unset ECF8_LIB; else export ECF8_LIB=build/var/$v/libecf8_b200.so; fi
  echo -n "$v: "; timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --cpu-seconds 0 --no-verify 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
unset ECF8_LIB
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 2>&1 >/dev/null | grep "fused m="
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 5 -c 1 -o gpurun_out/r2ag_full \
    python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > /dev/null 2>&1

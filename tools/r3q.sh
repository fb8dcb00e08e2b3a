#!/bin/bash
# Final check with the fused prefetch table default: GPU suite, smoke, fused sweep, bench.
mkdir -p gpurun_out
TAG=r3q
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/${TAG}_fused.json 2> gpurun_out/${TAG}_fused.err; grep "fused m=" gpurun_out/${TAG}_fused.err
for m in 1 256; do timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 2 -c 1 -o gpurun_out/${TAG}_fused_m$m python tools/fused_one.py 28672 8192 $m 3 > /dev/null 2>&1; done
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 400 gpurun_out/${TAG}_bench.json
ls gpurun_out/${TAG}_*

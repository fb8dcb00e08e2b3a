#!/bin/bash
# Final run of the session (prefetch table, FMA-pipe sink, write-back unroll 8): GPU suite, smoke, bench + reference arm, sweeps, decompress, ncu.
mkdir -p gpurun_out
TAG=r3o
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; tail -c 600 gpurun_out/${TAG}_bench_ref.json
timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/${TAG}_fused.json 2> gpurun_out/${TAG}_fused.err; grep "fused m=" gpurun_out/${TAG}_fused.err
timeout 900 python bench.py --workload dit-e5m2 > gpurun_out/${TAG}_dit.json 2> gpurun_out/${TAG}_dit.err; grep "dit-e5m2" gpurun_out/${TAG}_dit.err | tail -n 4
timeout 900 python bench.py --workload t-sweep > gpurun_out/${TAG}_tsweep.json 2> gpurun_out/${TAG}_tsweep.err; grep "t-sweep" gpurun_out/${TAG}_tsweep.err | tail -n 12
timeout 900 python tools/decompress_probe.py 8 > gpurun_out/${TAG}_decompress.json 2> gpurun_out/${TAG}_decompress.err; cat gpurun_out/${TAG}_decompress.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 5 -c 1 -o gpurun_out/${TAG}_full \
    python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > /dev/null 2>&1
for m in 1 256; do timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 2 -c 1 -o gpurun_out/${TAG}_fused_m$m python tools/fused_one.py 28672 8192 $m 3 > /dev/null 2>&1; done
ls gpurun_out/${TAG}_*

#!/bin/bash
# Session re-entry measurement: GPU tests, default + fused + DiT bench lines, reference arm,
# ncu launch list of the bench, full captures of the decode and fused kernels.
mkdir -p gpurun_out
TAG=${1:-r2q}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 3 > gpurun_out/${TAG}_bench_ref.json 2>gpurun_out/${TAG}_bench_ref.err; tail -c 600 gpurun_out/${TAG}_bench_ref.json
timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/${TAG}_fused.json 2> gpurun_out/${TAG}_fused.err; grep "fused m=" gpurun_out/${TAG}_fused.err
timeout 600 python bench.py --workload dit-e5m2 --steps 10 --warmup 3 > gpurun_out/${TAG}_dit.json 2> gpurun_out/${TAG}_dit.err; tail -c 1500 gpurun_out/${TAG}_dit.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 5 -c 1 -o gpurun_out/${TAG}_full \
    python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > gpurun_out/${TAG}_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_gemm -s 2 -c 1 -o gpurun_out/${TAG}_fused_m1 python tools/fused_one.py 28672 8192 1 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_gemm -s 2 -c 1 -o gpurun_out/${TAG}_fused_m256 python tools/fused_one.py 28672 8192 256 3 > /dev/null 2>&1
ls gpurun_out/${TAG}_*

#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2aj_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2aj_pytest.log
timeout 600 python bench.py > gpurun_out/r2aj_bench.json 2> gpurun_out/r2aj_bench.err; cat gpurun_out/r2aj_bench.json
timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/r2aj_fused.json 2> gpurun_out/r2aj_fused.err; grep "fused m=" gpurun_out/r2aj_fused.err
timeout 600 python bench.py --workload llama3.1-8b --steps 20 > gpurun_out/r2aj_8b.json 2> /dev/null; python -c "import json; d=json.load(open('gpurun_out/r2aj_8b.json')); print('8b', d['value'], d['roofline']['frac'])"
timeout 600 python bench.py --workload deepseek-v3-experts --steps 10 > gpurun_out/r2aj_ds.json 2> /dev/null; python -c "import json; d=json.load(open('gpurun_out/r2aj_ds.json')); print('ds', d['value'], d['roofline']['frac'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 5 -c 1 -o gpurun_out/r2aj_full \
    python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/r2aj_launches.csv python bench.py --steps 1 --warmup 3 --layers 8 --e2e-steps 0 --cpu-seconds 0 --no-verify > /dev/null 2>&1

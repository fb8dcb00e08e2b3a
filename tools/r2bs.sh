#!/bin/bash
# Final check: full GPU suite, smoke, default bench, reference arm, fused sweep.
mkdir -p gpurun_out
TAG=r2bs
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; head -c 700 gpurun_out/${TAG}_bench.json; echo
timeout 900 python bench.py --impl reference --steps 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err; head -c 300 gpurun_out/${TAG}_bench_ref.json; echo
timeout 600 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 > gpurun_out/${TAG}_fused.json 2> gpurun_out/${TAG}_fused.err; grep "fused m=" gpurun_out/${TAG}_fused.err

#!/bin/bash
# Final check with the prefetch section table in the 64-bit byte-step kernel (variant 6): GPU suite, smoke, DiT sweep, bench.
mkdir -p gpurun_out
TAG=r3r
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py --workload dit-e5m2 > gpurun_out/${TAG}_dit.json 2> gpurun_out/${TAG}_dit.err; grep "dit-e5m2" gpurun_out/${TAG}_dit.err | tail -n 12
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -c 300 gpurun_out/${TAG}_bench.json

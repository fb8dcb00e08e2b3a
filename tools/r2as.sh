#!/bin/bash
timeout 900 python -m pytest tests/test_e5m2.py -m gpu -q -x > gpurun_out/r2as_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2as_pytest.log
timeout 900 python bench.py --workload dit-e5m2 --steps 10 --warmup 3 > gpurun_out/r2as_dit.json 2> gpurun_out/r2as_dit.err; grep "dit-e5m2" gpurun_out/r2as_dit.err
cat > /tmp/e5one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec, e5m2
x = codec.synth(1.8, 0.05, 256 << 20, 5, fmt="e5m2")
dt = e5m2.E5DeviceTensor(e5m2.encode(x, 256))
assert dt.byte_steps
out = torch.empty(x.size, dtype=torch.uint8, device="cuda")
for _ in range(3): dt.decode_into(out)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:e5_fsm -s 2 -c 1 -o gpurun_out/r2as_e5fsm python /tmp/e5one.py > /dev/null 2>&1

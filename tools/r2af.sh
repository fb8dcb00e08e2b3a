#!/bin/bash
timeout 900 python bench.py --workload dit-e5m2 --steps 10 --warmup 3 > gpurun_out/r2af_dit.json 2> gpurun_out/r2af_dit.err; grep "dit-e5m2" gpurun_out/r2af_dit.err
cat > /tmp/e5one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec, e5m2
x = codec.synth(1.8, 0.05, 256 << 20, 5, fmt="e5m2")
dt = e5m2.E5DeviceTensor(e5m2.encode(x, 256))
out = torch.empty(x.size, dtype=torch.uint8, device="cuda")
for _ in range(3): dt.decode_into(out)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:e5_decode -s 2 -c 1 -o gpurun_out/r2af_e5 python /tmp/e5one.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_warp -s 2 -c 1 -o gpurun_out/r2af_v5 python -c "
import sys, torch
sys.path.insert(0, '.')
from paper_2510_02676_b200 import codec
from paper_2510_02676_b200.device import DeviceTensor
x = codec.synth(1.8, 0.05, 256 << 20, 5, fmt='e5m2')
dt = DeviceTensor(codec.encode_tensor(x, 256))
for _ in range(3): dt.decode()
torch.cuda.synchronize()
" > /dev/null 2>&1
ls gpurun_out/r2af*

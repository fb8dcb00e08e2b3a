#!/bin/bash
for mb in 32 64 128 256; do
  echo "== chunk $mb MB"; ECF8_FUSED_CHUNK_MB=$mb ECF8_BENCH_FUSED_MS=256 timeout 300 python bench.py --workload llama3-70b-fused --steps 10 --warmup 3 --no-verify 2>&1 >/dev/null | grep "fused m="
done
python - <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec
from paper_2510_02676_b200.fused import FusedLinear
import paper_2510_02676_b200.fused as F
w = codec.synth(1.8, 0.05, 28672 * 8192, 5).reshape(28672, 8192)
lin = FusedLinear(w)
x = (torch.randn(256, 8192, device="cuda") * 4).to(torch.float8_e4m3fn)
y = torch.empty(256, 28672, device="cuda")
for _ in range(3): lin(x, 1.0, y)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): lin(x, 1.0, y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"gate 28672x8192 m=256 rows path: host issue {(t1 - t0) / 10 * 1e3:.3f} ms/call, wall {(t2 - t0) / 10 * 1e3:.3f} ms/call")
PY

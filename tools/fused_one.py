"""One decode-fused GEMM call (for ncu): python tools/fused_one.py N K M [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec  # noqa: E402
from paper_2510_02676_b200.fused import FusedLinear  # noqa: E402

n, k, m = (int(a) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
w = codec.synth(1.8, 0.05, n * k, 5).reshape(n, k)
lin = FusedLinear(w)
x = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
y = torch.empty(m, n, device="cuda")
for _ in range(reps):
    lin(x, 1.0, y)
torch.cuda.synchronize()
print("done", lin.split_k)

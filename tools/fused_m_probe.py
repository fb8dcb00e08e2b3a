"""Fused GEMM kernel time vs M on one 28672x8192 weight (CUDA events,
20 back-to-back calls per M), to locate where the M >= 64 cost comes from."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec  # noqa: E402
from paper_2510_02676_b200.fused import FusedLinear  # noqa: E402

n, k = 28672, 8192
w = codec.synth(1.8, 0.05, n * k, 5).reshape(n, k)
lin = FusedLinear(w)
for m in (1, 16, 32, 64, 128, 129, 256):
    x = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
    y = torch.empty(m, n, device="cuda")
    for _ in range(3):
        lin(x, 1.0, y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        lin(x, 1.0, y)
    b.record()
    torch.cuda.synchronize()
    print(f"m={m}: {a.elapsed_time(b) / 20 * 1e3:.1f} us", flush=True)

import sys
import torch
sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec
from paper_2510_02676_b200.fused import FusedLinear
for n, k in [(2048, 2048), (8192, 2048), (2048, 8192), (8192, 8192)]:
    w = codec.synth(1.8, 0.05, n * k, 5).reshape(n, k)
    lin = FusedLinear(w)
    for m in [1, 16, 256]:
        x = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
        print(n, k, m, "split", lin.split_k, flush=True)
        y = lin(x, 1.0)
        torch.cuda.synchronize()
        print("  ok", flush=True)

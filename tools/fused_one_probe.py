import sys, torch
sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec
from paper_2510_02676_b200.fused import FusedLinear
n, k, m = 28672, 8192, 16
w = codec.synth(1.8, 0.05, n * k, 5).reshape(n, k)
lin = FusedLinear(w)
x = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
y = torch.empty(m, n, device="cuda")
for _ in range(5):
    lin(x, 1.0, y)
torch.cuda.synchronize()

"""Decode-fused GEMM timing on Llama-3-70B linear shapes vs decode-then-GEMM
and the plain FP8 GEMM (uncompressed weights).  python tools/fused_probe.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec  # noqa: E402
from paper_2510_02676_b200.device import Batch, DeviceTensor  # noqa: E402
from paper_2510_02676_b200.fused import FusedLinear, fused_layout  # noqa: E402

SHAPES = [("q/o", 8192, 8192), ("gate/up", 28672, 8192), ("down", 8192, 28672)]
MS = [int(a) for a in sys.argv[1:]] or [1, 16, 64, 256]


def t_ms(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name, n, k in SHAPES:
    w = codec.synth(1.8, 0.05, n * k, 5).reshape(n, k)
    lin = FusedLinear(w, threads_per_block=int(__import__("os").environ.get("FUSED_T", "128")))
    enc = codec.encode_tensor(w.reshape(-1), 256)
    dev = DeviceTensor(enc)
    wbuf = torch.empty(n * k, dtype=torch.uint8, device="cuda")
    batch = Batch([dev], [wbuf])
    wt = torch.from_numpy(w).cuda().view(torch.float8_e4m3fn)
    one = torch.tensor(1.0, device="cuda")
    for m in MS:
        x = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
        mp = max(16, (m + 15) // 16 * 16)
        xp = torch.cat([x, x.new_zeros(mp - m, k)]) if mp != m else x
        y = torch.empty(m, n, device="cuda")
        tf = t_ms(lambda: lin(x, 1.0, y))

        def dtg():
            batch.decode()
            torch._scaled_mm(xp, wbuf.view(torch.float8_e4m3fn).view(n, k).t(), scale_a=one, scale_b=one,
                             out_dtype=torch.float32)

        td = t_ms(dtg)
        tdec = t_ms(lambda: batch.decode())
        tp = t_ms(lambda: torch._scaled_mm(xp, wt.t(), scale_a=one, scale_b=one, out_dtype=torch.float32))
        comp = lin.compressed_bytes
        print(f"{name:8s} {n}x{k} m={m:3d}: fused {tf * 1e3:8.1f} us ({m / tf * 1e3:9.0f} tok/s, "
              f"{comp / tf / 1e6:6.0f} GB/s compressed, split_k {lin.split_k}) | decode+gemm {td * 1e3:8.1f} us | "
              f"plain fp8 gemm {tp * 1e3:7.1f} us | decode only {tdec * 1e3:7.1f} us", flush=True)

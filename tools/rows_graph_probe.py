"""Probe: one Llama-3-70B layer (7 linears) as decode-rows (tiled weight ->
row-major chunk in an L2-sized two-slot ring, side stream) + cuBLASLt FP8 GEMM
per chunk, the whole layer captured in one CUDA graph.  Compared with the
fused kernel on the same weights.

python tools/rows_graph_probe.py [chunk_mb ...]
"""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_02676_b200 import codec  # noqa: E402
from paper_2510_02676_b200._lib import check, lib  # noqa: E402
from paper_2510_02676_b200.fused import FusedLinear  # noqa: E402

LLAMA70B = [(8192, 8192), (1024, 8192), (1024, 8192), (8192, 8192), (28672, 8192), (28672, 8192), (8192, 28672)]
chunks_mb = [int(a) for a in sys.argv[1:]] or [16, 32, 64]
MS = [1, 16, 64, 256]

t0 = time.time()
lins = [FusedLinear(codec.synth(1.8, 0.05, n * k, j).reshape(n, k)) for j, (n, k) in enumerate(LLAMA70B)]
print(f"prepared in {time.time() - t0:.0f}s", flush=True)
one = torch.ones((), device="cuda")
st = torch.cuda.Stream()
dec = torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for m in MS:
    xs = [(torch.randn(m, lin.k, device="cuda") * 4).to(torch.float8_e4m3fn) for lin in lins]
    mp = max(16, (m + 15) // 16 * 16)
    xps = [torch.cat([x, x.new_zeros(mp - m, x.shape[1])]) if mp != m else x for x in xs]
    outs = [torch.empty(m, lin.n, device="cuda") for lin in lins]
    ref = []
    with torch.cuda.stream(st):
        for lin, x, o in zip(lins, xs, outs):
            lin(x, 1.0, o, stream=st)
            ref.append(o.clone())

    def fused():
        with torch.cuda.stream(st):
            for lin, x, o in zip(lins, xs, outs):
                lin(x, 1.0, o, stream=st)

    tf = timed(fused)
    res = {"m": m, "fused_ms": round(tf, 4)}
    for cmb in chunks_mb:
        cb = cmb << 20
        slots = [torch.empty(cb + 16, dtype=torch.uint8, device="cuda") for _ in range(2)]
        ev_dec = [torch.cuda.Event() for _ in range(2)]
        ev_use = [torch.cuda.Event() for _ in range(2)]

        def layer():
            dec.wait_stream(st)
            kk = 0
            for lin, xp, o in zip(lins, xps, outs):
                rows = max(128, min(lin.n, cb // lin.k // 128 * 128))
                for r0 in range(0, lin.n, rows):
                    r1 = min(lin.n, r0 + rows)
                    s = kk % 2
                    if kk >= 2:
                        dec.wait_event(ev_use[s])
                    check(lib.ecf8_fused_decode_rows(lin.handle, r0, r1, C.c_void_p(slots[s].data_ptr()),
                                                     C.c_void_p(dec.cuda_stream)))
                    ev_dec[s].record(dec)
                    st.wait_event(ev_dec[s])
                    w = slots[s][: (r1 - r0) * lin.k].view(torch.float8_e4m3fn).view(r1 - r0, lin.k)
                    with torch.cuda.stream(st):
                        y = torch._scaled_mm(xp, w.t(), scale_a=one, scale_b=one, out_dtype=torch.float32)
                        o[:, r0:r1].copy_(y[:m])
                    ev_use[s].record(st)
                    kk += 1
            st.wait_stream(dec)

        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            layer()  # warm (cuBLASLt heuristics, workspace)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            layer()
        def rep():
            with torch.cuda.stream(st):
                g.replay()

        rep()
        torch.cuda.synchronize()
        err = max(float((o - r).abs().max() / (r.abs().max() + 1e-30)) for o, r in zip(outs, ref))
        tg = timed(rep)
        res[f"rows{cmb}MB_graph_ms"] = round(tg, 4)
        res[f"rows{cmb}MB_rel_err_vs_fused"] = float(f"{err:.2e}")
        del g
    print(res, flush=True)

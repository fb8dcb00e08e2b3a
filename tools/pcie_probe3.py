"""PCIe: why chunked copies (76-77 GB/s algorithmic) trail one bulk copy per
direction (92 GB/s).  Variants: one direction chunked, both directions chunked
without the H2D -> D2H dependency, and with it on 1 / 2 / 4 streams per
direction (chunk k on stream k % n)."""
import sys

import torch

sys.path.insert(0, ".")
from bench import build_layer  # noqa: E402

raws, encs = build_layer(0)
algo = sum(e.algorithmic_bytes() for e in encs)
n_out = sum(e.n_elem for e in encs)
n_in = algo - n_out
h_in = torch.empty(n_in, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n_out, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
S_in = [torch.cuda.Stream() for _ in range(4)]
S_out = [torch.cuda.Stream() for _ in range(4)]


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        for s in S_in + S_out:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def run(mb, ns, dep=True, do_in=True, do_out=True):
    c_out = mb << 20
    c_in = c_out * n_in // n_out
    nch = (n_out + c_out - 1) // c_out
    ev = [torch.cuda.Event() for _ in range(nch)]
    for s in S_in + S_out:
        s.wait_stream(torch.cuda.current_stream())
    for k in range(nch):
        si, so = S_in[k % ns], S_out[k % ns]
        if do_in:
            with torch.cuda.stream(si):
                a, b = k * c_in, min(n_in, (k + 1) * c_in)
                if b > a:
                    d_in[a:b].copy_(h_in[a:b], non_blocking=True)
                ev[k].record(si)
        if do_out:
            with torch.cuda.stream(so):
                if dep and do_in:
                    so.wait_event(ev[k])
                a, b = k * c_out, min(n_out, (k + 1) * c_out)
                h_out[a:b].copy_(d_out[a:b], non_blocking=True)


for mb in (32, 8):
    t = timed(lambda: run(mb, 1, do_in=False))
    print(f"{mb} MB: d2h only chunked: {n_out / t / 1e9:.1f} GB/s", flush=True)
    t = timed(lambda: run(mb, 1, do_out=False))
    print(f"{mb} MB: h2d only chunked: {n_in / t / 1e9:.1f} GB/s", flush=True)
    t = timed(lambda: run(mb, 1, dep=False))
    print(f"{mb} MB: both, no dependency, 1 stream each: {algo / t / 1e9:.1f} GB/s", flush=True)
    for ns in (1, 2, 4):
        t = timed(lambda: run(mb, ns))
        print(f"{mb} MB: both, dependency, {ns} streams each: {algo / t / 1e9:.1f} GB/s", flush=True)

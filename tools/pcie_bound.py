"""The e2e path's copy bound on this box: one Llama-3.1-8B layer's compressed
bytes host->device and its FP8 output device->host, from/to pinned memory,
alone and concurrently on two streams (no decode).  The e2e metric
(algorithmic bytes / time) cannot beat algorithmic bytes / concurrent time."""
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
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def h2d(chunk=None):
    with torch.cuda.stream(s1):
        s1.wait_stream(torch.cuda.current_stream())
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        s2.wait_stream(torch.cuda.current_stream())
        h_out.copy_(d_out, non_blocking=True)


t_in = timed(h2d)
t_out = timed(d2h)
t_both = timed(lambda: (h2d(), d2h()))
print(f"h2d {n_in / 1e6:.0f} MB: {n_in / t_in / 1e9:.1f} GB/s; d2h {n_out / 1e6:.0f} MB: {n_out / t_out / 1e9:.1f} GB/s; "
      f"both: {t_both * 1e3:.2f} ms -> copy bound {algo / t_both / 1e9:.1f} GB/s (algorithmic)", flush=True)

# chunked, with the host pipeline's coupling (4 slots: H2D of chunk k+4 waits
# for the D2H of chunk k) or without (a staging buffer per chunk)
for mb, slots in ((8, 4), (16, 4), (32, 4), (4, 0), (8, 0), (16, 0), (32, 0)):
    c_out = mb << 20
    c_in = c_out * n_in // n_out
    nch = (n_out + c_out - 1) // c_out
    ev_in = [torch.cuda.Event() for _ in range(nch)]
    ev_out = [torch.cuda.Event() for _ in range(nch)]

    def chunked():
        s1.wait_stream(torch.cuda.current_stream())
        s2.wait_stream(torch.cuda.current_stream())
        for k in range(nch):
            with torch.cuda.stream(s1):
                if slots and k >= slots:
                    s1.wait_event(ev_out[k - slots])
                a, b = k * c_in, min(n_in, (k + 1) * c_in)
                if b > a:
                    d_in[a:b].copy_(h_in[a:b], non_blocking=True)
                ev_in[k].record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(ev_in[k])
                a, b = k * c_out, min(n_out, (k + 1) * c_out)
                h_out[a:b].copy_(d_out[a:b], non_blocking=True)
                ev_out[k].record(s2)

    t = timed(chunked)
    print(f"chunks of {mb} MB out ({nch}), {slots or 'unbounded'} slots: {t * 1e3:.2f} ms -> {algo / t / 1e9:.1f} GB/s", flush=True)

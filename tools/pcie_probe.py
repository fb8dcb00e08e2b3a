"""PCIe ceiling for the e2e path: pinned H2D, D2H, and both at once."""
import torch

n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        torch.cuda.synchronize()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


h2d = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timeit(lambda: h_out.copy_(d_out, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


bi = timeit(both)
print(f"pcie: H2D {n / h2d / 1e6:.1f} GB/s, D2H {n / d2h / 1e6:.1f} GB/s, "
      f"bidirectional {2 * n / bi / 1e6:.1f} GB/s total ({n / bi / 1e6:.1f} per direction)")

# chunked, dependent pipeline (H2D chunk k on s1 -> D2H chunk k on s2)
for chunk in (1 << 20, 4 << 20, 16 << 20, 64 << 20):
    nch = n // chunk

    def pipe():
        for k in range(nch):
            sl = slice(k * chunk, (k + 1) * chunk)
            with torch.cuda.stream(s1):
                d_in[sl].copy_(h_in[sl], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(ev)
                h_out[sl].copy_(d_out[sl], non_blocking=True)

    t = timeit(pipe, reps=3)
    print(f"chunk {chunk >> 20} MB dependent pipeline: {2 * n / t / 1e6:.1f} GB/s total")

    def indep():
        for k in range(nch):
            sl = slice(k * chunk, (k + 1) * chunk)
            with torch.cuda.stream(s1):
                d_in[sl].copy_(h_in[sl], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[sl].copy_(d_out[sl], non_blocking=True)

    t = timeit(indep, reps=3)
    print(f"chunk {chunk >> 20} MB independent: {2 * n / t / 1e6:.1f} GB/s total")

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

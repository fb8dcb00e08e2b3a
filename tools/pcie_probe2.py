"""Replicate the host pipeline's copy pattern with torch streams (diagnostics)."""
import torch

MB = 1 << 20
h_in = torch.empty(512 * MB, dtype=torch.uint8).pin_memory()
h_out = torch.empty(512 * MB, dtype=torch.uint8).pin_memory()
slots = [torch.empty(64 * MB, dtype=torch.uint8, device="cuda") for _ in range(4)]
s_in, s_run, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def pipe(n_chunks, sizes_in, size_out, relay, slots_wait):
    ev_out = [None] * 4
    off_i = off_o = 0
    for k in range(n_chunks):
        sl = slots[k % 4]
        with torch.cuda.stream(s_in):
            if slots_wait and ev_out[k % 4] is not None:
                s_in.wait_event(ev_out[k % 4])
            o = 0
            for sz in sizes_in:
                sl[o:o + sz].copy_(h_in[off_i:off_i + sz], non_blocking=True)
                o += sz
                off_i = (off_i + sz) % (400 * MB)
            e_in = torch.cuda.Event()
            e_in.record(s_in)
        if relay:
            s_run.wait_event(e_in)
            e_run = torch.cuda.Event()
            e_run.record(s_run)
        else:
            e_run = e_in
        with torch.cuda.stream(s_out):
            s_out.wait_event(e_run)
            h_out[off_o:off_o + size_out].copy_(sl[32 * MB:32 * MB + size_out], non_blocking=True)
            off_o = (off_o + size_out) % (400 * MB)
            e = torch.cuda.Event()
            e.record(s_out)
            ev_out[k % 4] = e


def bench(label, **kw):
    import time
    pipe(**kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe(**kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tot_in = kw["n_chunks"] * sum(kw["sizes_in"])
    tot_out = kw["n_chunks"] * kw["size_out"]
    print(f"{label}: {dt * 1e3:.2f} ms, in {tot_in / dt / 1e9:.1f} GB/s out {tot_out / dt / 1e9:.1f} GB/s")


ours = dict(n_chunks=24, sizes_in=[4 * MB, 256 * 1024, 16 * 1024, 7 * MB], size_out=14 * MB)
bench("ours (4 copies in, relay, slot wait)", relay=True, slots_wait=True, **ours)
bench("no relay", relay=False, slots_wait=True, **ours)
bench("no slot wait", relay=True, slots_wait=False, **ours)
bench("one copy in", relay=True, slots_wait=True, n_chunks=24, sizes_in=[11 * MB], size_out=14 * MB)

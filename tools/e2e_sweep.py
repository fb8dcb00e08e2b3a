"""e2e host path: one Llama-8B layer (and two layers per call) through
ecf8_decode_host_many from pinned buffers; run under different ECF8_CHUNK_*
environments to tune the pipeline."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import build_layer  # noqa: E402
from paper_2510_02676_b200._lib import Sections, check, lib  # noqa: E402

raws, encs = build_layer(0)
algo1 = sum(e.algorithmic_bytes() for e in encs)


def pinned_copy(a):
    t = torch.empty(max(1, a.nbytes), dtype=torch.uint8).pin_memory()
    t.numpy()[: a.nbytes] = a.view(np.uint8).reshape(-1)
    return t


keep, secs = [], []
for e in encs:
    s = e.sections()
    for name, arr in (("encoded", e.encoded), ("gaps", e.gaps), ("outpos", e.outpos), ("packed", e.packed)):
        t = pinned_copy(np.asarray(arr))
        keep.append(t)
        setattr(s, name, t.data_ptr())
    secs.append(s)
for layers in (1, 2, 4):
    ss = secs * layers
    outs = [torch.empty(e.n_elem, dtype=torch.uint8).pin_memory() for e in encs * layers]
    n = len(ss)
    sp = (C.POINTER(Sections) * n)(*[C.pointer(x) for x in ss])
    op = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    ln = (C.c_uint64 * n)(*[e.n_elem for e in encs * layers])
    check(lib.ecf8_decode_host_many(sp, op, ln, n))
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        check(lib.ecf8_decode_host_many(sp, op, ln, n))
        best = min(best, time.perf_counter() - t0)
    ok = all(np.array_equal(o.numpy(), r) for o, r in zip(outs[:7], raws))
    print(f"layers/call {layers}: {best * 1e3 / layers:.2f} ms/layer, {algo1 * layers / best / 1e9:.1f} GB/s, ok={ok}",
          flush=True)

"""e2e host-path probe: one Llama-8B layer through ecf8_decode_host_many,
sections in torch-pinned buffers vs cudaHostRegister'ed library memory."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import LLAMA8B, build_layer  # noqa: E402
from paper_2510_02676_b200._lib import Sections, check, lib  # noqa: E402

raws, encs = build_layer(0)
n7 = len(encs)
outs = [torch.empty(e.n_elem, dtype=torch.uint8).pin_memory() for e in encs]
algo = sum(e.algorithmic_bytes() for e in encs)
h2d = sum(e.compressed_bytes() for e in encs)


def pinned_copy(a):
    t = torch.empty(max(1, a.nbytes), dtype=torch.uint8).pin_memory()
    t.numpy()[: a.nbytes] = a.view(np.uint8).reshape(-1)
    return t


def run(secs, label, reps=5):
    sp = (C.POINTER(Sections) * n7)(*[C.pointer(x) for x in secs])
    op = (C.c_void_p * n7)(*[o.data_ptr() for o in outs])
    ln = (C.c_uint64 * n7)(*[e.n_elem for e in encs])
    check(lib.ecf8_decode_host_many(sp, op, ln, n7))
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        check(lib.ecf8_decode_host_many(sp, op, ln, n7))
        best = min(best, time.perf_counter() - t0)
    ok = all(np.array_equal(o.numpy(), r) for o, r in zip(outs, raws))
    print(f"{label}: {best * 1e3:.2f} ms/layer, {algo / best / 1e9:.1f} GB/s algorithmic, "
          f"H2D {h2d / best / 1e9:.1f} GB/s + D2H {sum(e.n_elem for e in encs) / best / 1e9:.1f} GB/s, ok={ok}")


# (a) torch-pinned section copies
keep = []
secs_a = []
for e in encs:
    s = e.sections()
    for name, arr in (("encoded", e.encoded), ("gaps", e.gaps), ("outpos", e.outpos), ("packed", e.packed)):
        t = pinned_copy(np.asarray(arr))
        keep.append(t)
        setattr(s, name, t.data_ptr())
    secs_a.append(s)
run(secs_a, "torch-pinned sections")
import os
if os.environ.get("ONLY_PINNED"): sys.exit(0)

# (b) cudaHostRegister on the library's own section memory
cudart = torch.cuda.cudart()
regs = []
for e in encs:
    for a in (e.encoded, e.gaps, e.outpos, e.packed):
        rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        regs.append((a.ctypes.data, int(rc)))
print("cudaHostRegister rcs:", sorted({rc for _, rc in regs}))
run([e.sections() for e in encs], "registered sections")
for p, rc in regs:
    if rc == 0:
        cudart.cudaHostUnregister(p)
run([e.sections() for e in encs], "pageable sections")

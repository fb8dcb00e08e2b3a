"""Device encoder throughput on one Llama-3.1-8B layer's FP8 linears
(α 1.8, γ 0.05): histogram + code + encode per tensor, vs the host encoder
(encode_many, all host threads).  Prints FP8 input GB/s."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import LLAMA8B  # noqa: E402
from paper_2510_02676_b200 import codec  # noqa: E402
from paper_2510_02676_b200.device import DeviceTensor, exponent_histogram  # noqa: E402
from paper_2510_02676_b200.codec import build_code  # noqa: E402

raws = [codec.synth(1.8, 0.05, r * c, 1000 + i) for i, (_, r, c) in enumerate(LLAMA8B)]
n_total = sum(r.size for r in raws)
xs = [torch.from_numpy(r).cuda() for r in raws]
codes = [build_code(exponent_histogram(x)) for x in xs]


def run(with_hist):
    out = []
    for x, l in zip(xs, codes):
        lengths = build_code(exponent_histogram(x)) if with_hist else l
        out.append(DeviceTensor.encode(x, lengths, 256))
    torch.cuda.synchronize()
    return out


for with_hist in (False, True):
    run(with_hist)
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        ts = run(with_hist)
        best = min(best, time.perf_counter() - t0)
        del ts
    print(f"device encode{' + histogram' if with_hist else ''}: {best * 1e3:.2f} ms/layer, "
          f"{n_total / best / 1e9:.1f} GB/s of FP8 input", flush=True)

ok = all(np.array_equal(t.decode().cpu().numpy(), r) for t, r in zip(run(False), raws))
t0 = time.perf_counter()
host = codec.encode_many(raws, 256)
dt = time.perf_counter() - t0
print(f"host encode_many: {dt * 1e3:.1f} ms/layer, {n_total / dt / 1e9:.2f} GB/s; device round trip ok={ok}",
      flush=True)

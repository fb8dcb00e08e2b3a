"""Quick decode-throughput probe (development aid; bench.py is the contract).

python tools/probe.py [--n ELEMS] [--count K] [--T 256] [--reps 20]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_02676_b200 import codec  # noqa: E402
from paper_2510_02676_b200.device import Batch, DeviceTensor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=14336 * 4096)
    ap.add_argument("--count", type=int, default=8)
    ap.add_argument("--distinct", type=int, default=2)
    ap.add_argument("--T", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--gamma", type=float, default=0.05)
    a = ap.parse_args()
    t0 = time.time()
    xs = [codec.synth(1.8, a.gamma, a.n, 1000 + i) for i in range(a.distinct)]
    encs = codec.encode_many(xs, a.T)
    print(f"synth+encode {time.time() - t0:.1f}s; bits/sym ~ {8 * encs[0].encoded.size / a.n:.3f}", flush=True)
    dts = [DeviceTensor(encs[i % a.distinct]) for i in range(a.count)]
    outs = [torch.empty(a.n, dtype=torch.uint8, device="cuda") for _ in range(a.count)]
    b = Batch(dts, outs)
    torch.cuda.synchronize()
    for o, i in zip(outs, range(a.count)):
        pass
    b.decode()
    torch.cuda.synchronize()
    ok = all(np.array_equal(outs[i][:1 << 20].cpu().numpy(), xs[i % a.distinct][:1 << 20]) for i in range(a.count))
    ok = ok and np.array_equal(outs[0].cpu().numpy(), xs[0])
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        b.decode()
    torch.cuda.synchronize()
    s.record()
    for _ in range(a.reps):
        b.decode()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.reps
    gbs = b.algorithmic_bytes / (ms * 1e-3) / 1e9
    print(f"bit-exact={ok} count={a.count} n={a.n} T={a.T}: {ms:.3f} ms/step, {gbs:.1f} GB/s algorithmic, "
          f"{a.count * a.n / ms / 1e6:.1f} Gelem/s, launches={b.launches}")
    # single tensor
    s.record()
    for _ in range(a.reps):
        dts[0].decode_into(outs[0])
    e.record()
    torch.cuda.synchronize()
    ms1 = s.elapsed_time(e) / a.reps
    print(f"single tensor: {ms1:.3f} ms, {dts[0].algorithmic_bytes / (ms1 * 1e-3) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()

"""Small-shape cases for compute-sanitizer (memcheck / racecheck / synccheck).

Run on the GPU box as
    compute-sanitizer --tool racecheck --target-processes all python tools/sanitize_cases.py
Every kernel family of the library is launched at least once on inputs small
enough for the sanitizers' replay:
  * decode_warp_kernel<24> (variant 4), its direct-only instance (variant 7),
    <12, WIDE> (variant 5), decode_fsm64_kernel (variant 6), the group
    kernels decode_kernel (T = 1, 2, 512, 1024), verify_gaps_kernel,
    count_window_kernel;
  * a tensor with corrupted gap nibbles (window-by-window walk + exact walk);
  * a batch of tensors of mixed sizes (descriptor search, PDL back-to-back);
  * the decode-fused GEMM (fused_l2_kernel: decode warps -> per-CTA L2 ring
    -> loader bulk copies -> tcgen05.mma; fused_gemm_kernel for 1-bit codes)
    with multi-K-tile CTA runs (ring wrap, stage release, TMEM accumulation
    across K tiles, multi-segment epilogues), m <= 128 and m > 128, E4M3 and
    E5M2;
  * the device encoder (histogram, chunk scan, emit);
  * the native E5M2 decoder (e5_decode_kernel, T 8 / 256 / 1024).
Each output is checked bit-exact against the original bytes (the encoder's
input), so a sanitizer-clean run is also a correct one.  The reference
schedule argument (blocks write disjoint output ranges) is
what racecheck verifies for the shared-memory side here.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2510_02676_b200 import codec  # noqa: E402
from paper_2510_02676_b200.device import Batch, DeviceTensor  # noqa: E402
from paper_2510_02676_b200.fused import FusedLinear, fused_layout  # noqa: E402


def decode_cases(scale):
    for n, T, fmt, seed in [(300_000 * scale, 256, "e4m3", 1), (77_777, 64, "e4m3", 2), (50_001, 8, "e4m3", 3),
                            (200_000 * scale, 128, "e5m2", 4), (20_000, 1, "e4m3", 5), (30_000, 2, "e4m3", 6),
                            (100_000, 512, "e4m3", 7), (100_000, 1024, "e5m2", 8), (0, 256, "e4m3", 9), (1, 256, "e4m3", 10)]:
        x = codec.synth(1.8, 0.05, n, seed, fmt=fmt)
        t = codec.encode_tensor(x, T)
        d = DeviceTensor(t)
        got = d.decode().cpu().numpy()
        assert np.array_equal(got, x), (n, T, fmt)
        print(f"decode n={n} T={T} {fmt} variant={d.kernel_variant} ok", flush=True)
    # corrupted gaps: tiles fail the upload check and take the exact walk
    x = codec.synth(1.8, 0.05, 200_000, 11)
    t = codec.encode_tensor(x, 256)
    want = codec.decode_parallel(t)
    bad = t.copy()
    for w in (5, 700, 1500):
        bad.gaps[w >> 1] ^= 0x30 if w & 1 == 0 else 0x03
    d = DeviceTensor(bad)
    got = d.decode().cpu().numpy()
    assert np.array_equal(got, codec.decode_parallel(bad))
    print(f"corrupt gaps ok (verified tiles {d.verified_tiles()}); clean decode matches: {np.array_equal(want, x)}")
    # a block boundary moved by one symbol: a tile off the direct path (variant 4 with its fallback)
    x = codec.synth(1.8, 0.05, 300_000, 12)
    mv = codec.encode_tensor(x, 256).copy()
    op = mv.outpos
    b = (len(op) - 1) // 2
    op[b + 1] -= 1
    d = DeviceTensor(mv)
    assert d.kernel_variant == 4
    got = d.decode().cpu().numpy()
    ok = np.ones(x.size, bool)
    ok[op[b + 2] - 1] = False
    assert np.array_equal(got[ok], codec.decode_parallel(mv)[ok])
    print("moved block boundary ok (variant 4)", flush=True)
    # batch: mixed tensors, one launch per variant, twice back to back
    xs = [codec.synth(1.8, 0.05, n, 20 + i) for i, n in enumerate([100_000, 3, 65_536, 250_000])]
    ds = [DeviceTensor(codec.encode_tensor(x, 256)) for x in xs]
    outs = [torch.empty(x.size, dtype=torch.uint8, device="cuda") for x in xs]
    b = Batch(ds, outs)
    b.decode()
    b.decode()
    for o, x in zip(outs, xs):
        assert np.array_equal(o.cpu().numpy(), x)
    print("batch ok", flush=True)
    # count_phase known answer (test_codec.cpp:206-212): a 1-bit code over zeros -> 64
    ladder = np.array(list(range(1, 16)) + [15], np.uint8)
    assert codec.count_phase(np.zeros(10, np.uint8), 0, ladder) == 64
    print("count_phase ok", flush=True)


def fused_cases(n, k, ms, fmt):
    w = codec.synth(1.8, 0.05, n * k, 31 + n + k, fmt=fmt).reshape(n, k)
    lin = FusedLinear(w, fmt)
    wt = torch.from_numpy(w).cuda().view(torch.float8_e4m3fn if fmt == "e4m3" else torch.float8_e5m2)
    for m in ms:
        x8 = (torch.randn(m, k, device="cuda") * 2).to(torch.float8_e4m3fn)
        y = lin(x8, 1.0)
        ref = x8.double() @ wt.double().t()
        err = (y.double() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)
        assert err < 1e-4, (n, k, m, err)
        print(f"fused {n}x{k} {fmt} m={m} split_k={lin.split_k} rel err {err:.2e} ok", flush=True)


def e5_cases():
    from paper_2510_02676_b200 import e5m2

    for n, T, seed in [(200_003, 256, 51), (33_000, 8, 52), (70_000, 1024, 53), (1, 32, 54)]:
        x = codec.synth(1.8, 0.05, n, seed, fmt="e5m2")
        got = e5m2.E5DeviceTensor(e5m2.encode(x, T)).decode().cpu().numpy()
        assert np.array_equal(got, x), (n, T)
        print(f"e5m2 native n={n} T={T} ok", flush=True)


def encode_cases():
    x = codec.synth(1.8, 0.05, 300_000, 41)
    xt = torch.from_numpy(x).cuda()
    d = DeviceTensor.encode(xt, threads_per_block=256)
    assert np.array_equal(d.decode().cpu().numpy(), x)
    print("device encode ok", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    if which in ("all", "decode"):
        decode_cases(1)
    if which in ("all", "fused"):
        # 1024 x 4096 = 256 tiles, 2048 x 8192 = 1024 tiles (~7 K tiles per CTA:
        # the 5-stage A ring wraps); k = 128 at n = 128 * 518: 3-4 segments per CTA
        fused_cases(1024, 4096, [16, 200], "e4m3")
        fused_cases(2048, 8192, [1, 130], "e4m3")
        fused_cases(128 * 518, 128, [16, 200], "e4m3")  # m = 200: 2 accumulator buffers reused round-robin
        fused_cases(1024, 2048, [64], "e5m2")
    if which in ("all", "encode"):
        encode_cases()
    if which in ("all", "e5"):
        e5_cases()
    torch.cuda.synchronize()
    print("sanitize cases done")

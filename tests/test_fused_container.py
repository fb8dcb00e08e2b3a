"""A reference-written .ecf8 container served by the decode-fused GEMM.

tests/golden/weights_T256.ecf8 holds two row-major 2-D FP8 weights written
by the reference itself (oracle/_ref: synth_raw + compress_tensors +
serialize, tests/golden/make_golden.py).  FusedLinear.from_container uploads
the row-major ECF8 tensor, decodes it on the GPU, re-tiles it
(ecf8_fused_layout_device) and re-encodes it with the device encoder for the
fused kernel -- no host round trip.  Checked against:
  * the reference-decoded weight (C oracle on the container's own sections,
    and the manifest's SHA-256 of the generating bytes);
  * the plain FP8 GEMM (torch._scaled_mm) on that weight, within the fp32
    accumulation bound of test_fused_large.py;
  * the hook path (ECF8Linear, torch.ops.ecf8.fused_gemm) vs its unfused
    decode-then-GEMM path on the same weight.
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from paper_2510_02676_b200 import codec

from _oracle import tensor_dict

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "weights.json")) as f:
    MANIFEST = json.load(f)
with open(os.path.join(HERE, "golden", MANIFEST["container"]), "rb") as f:
    DATA = f.read()
U = 2.0 ** -24


def test_weights_fixture_is_the_reference_container():
    assert hashlib.sha256(DATA).hexdigest() == MANIFEST["container_sha256"]
    f = codec.parse_container(DATA)
    assert [n for n, _ in f.tensors] == [t["name"] for t in MANIFEST["tensors"]]
    assert f.shapes == [t["shape"] for t in MANIFEST["tensors"]]


@pytest.mark.gpu
def test_fused_layout_device_matches_host_layout():
    from paper_2510_02676_b200.fused import fused_layout, fused_layout_device

    rng = np.random.default_rng(1)
    w = rng.integers(0, 256, (384, 640), dtype=np.uint8)
    dev = fused_layout_device(torch.from_numpy(w).cuda(), 384, 640)
    assert np.array_equal(dev.cpu().numpy(), fused_layout(w))
    back = fused_layout_device(dev, 384, 640, inverse=True)
    assert np.array_equal(back.cpu().numpy().reshape(384, 640), w)


@pytest.mark.gpu
@pytest.mark.parametrize("i", [0, 1])
@pytest.mark.parametrize("m", [1, 37, 256])
def test_container_weight_through_fused_gemm(orc, i, m):
    from paper_2510_02676_b200.fused import FusedLinear

    meta = MANIFEST["tensors"][i]
    n, k = meta["shape"]
    f = codec.parse_container(DATA)
    name, t = f.tensors[i]
    wd = orc.decode_parallel(tensor_dict(t)).reshape(n, k)  # reference-decoded row-major weight
    assert hashlib.sha256(wd.tobytes()).hexdigest() == meta["sha256"]
    lin = FusedLinear.from_container(DATA, name)
    assert lin.n == n and lin.k == k
    g = torch.Generator(device="cuda").manual_seed(m + i)
    x8 = (torch.randn(m, k, device="cuda", generator=g) * 4).to(torch.float8_e4m3fn)
    y = lin(x8, 0.5)
    w8 = torch.from_numpy(wd).cuda().view(torch.float8_e4m3fn)
    y64 = (x8.double() @ w8.double().t()) * 0.5
    bound = (k * U / (1 - k * U) + U) * (x8.double().abs() @ w8.double().abs().t()) * 0.5 + 1e-30
    torch.cuda.synchronize()
    assert ((y.double() - y64).abs() <= bound).all()
    # the op form gives the same bytes
    y_op = torch.ops.ecf8.fused_gemm(x8, lin.handle.value, n, 0.5)
    torch.testing.assert_close(y_op, y, rtol=1e-6, atol=1e-3 * y.abs().max().item())


@pytest.mark.gpu
def test_ecf8_linear_fused_and_unfused_agree():
    from paper_2510_02676_b200.hooks import DecodeArena, ECF8Linear

    f = codec.parse_container(DATA)
    n, k = MANIFEST["tensors"][0]["shape"]
    w = codec.decode_parallel(f.tensors[0][1]).reshape(n, k)
    fused = ECF8Linear(w, scale_w=0.25, arena=DecodeArena())
    plain = ECF8Linear(w, scale_w=0.25, arena=DecodeArena(), fused=False)
    assert fused.fused is not None and plain.fused is None
    x = torch.randn(5, 7, k, device="cuda")
    sx = torch.tensor(0.02, device="cuda")
    ya, yb = fused(x, sx), plain(x, sx)
    assert ya.shape == yb.shape == (5, 7, n)
    torch.testing.assert_close(ya.float(), yb.float(), rtol=1e-2, atol=1e-2 * yb.float().abs().max().item())

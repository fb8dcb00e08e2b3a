"""Decode-fused tcgen05 FP8 GEMM (row a17).

CPU: the tiled layout is a bijection (inverse(layout(W)) == W) with the
swizzle the kernel assumes.
GPU: y = x . W^T from the fused kernel equals the plain FP8 GEMM
(torch._scaled_mm, fp32 out) on the reference-decoded weights within an
fp32-accumulation tolerance (|err| <= 1e-3 * max|y| + 1e-3), for E4M3 and
E5M2 weights, m in {1, 16, 64, 256}, split-K and not.
"""
import numpy as np
import pytest
import torch

from paper_2510_02676_b200 import codec
from paper_2510_02676_b200.fused import fused_layout, fused_layout_inverse

from _oracle import tensor_dict


def test_fused_layout_roundtrip_and_swizzle():
    rng = np.random.default_rng(0)
    w = rng.integers(0, 256, (256, 384), dtype=np.uint8)
    seq = fused_layout(w)
    assert np.array_equal(fused_layout_inverse(seq, 256, 384), w)
    # tile (nt=1, kt=2), row r, byte c -> r*128 + ((c//16 ^ r%8) * 16) + c%16
    tile = seq[(1 * 3 + 2) * 16384:(1 * 3 + 3) * 16384]
    for r, c in [(0, 0), (5, 17), (127, 127), (64, 100)]:
        assert tile[r * 128 + (((c // 16) ^ (r % 8)) * 16) + c % 16] == w[128 + r, 256 + c]


def ref_gemm(orc, lin, x8, scale, fmt):
    seq = orc.decode_parallel(tensor_dict(lin.encoded))  # reference-decoded tiled bytes
    wd = fused_layout_inverse(seq, lin.n, lin.k)
    dt = {"e4m3": torch.float8_e4m3fn, "e5m2": torch.float8_e5m2}[fmt]
    w = torch.from_numpy(wd).cuda().view(dt)
    m = x8.shape[0]
    pad = (-m) % 16
    xp = torch.cat([x8, x8.new_zeros(pad, lin.k)]) if pad else x8
    one = torch.tensor(1.0, device="cuda")
    y = torch._scaled_mm(xp, w.t(), scale_a=one, scale_b=one, out_dtype=torch.float32)[:m]
    return y * scale, wd


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["e4m3", "e5m2"])
@pytest.mark.parametrize("m", [1, 16, 64, 256])
@pytest.mark.parametrize("nk", [(256, 512), (1024, 2048)])
def test_fused_gemm_matches_fp8_gemm_on_reference_decoded_weights(orc, fmt, m, nk):
    from paper_2510_02676_b200.fused import FusedLinear

    n, k = nk
    w = codec.synth(1.8, 0.05, n * k, 77 + n, fmt=fmt).reshape(n, k)
    lin = FusedLinear(w, fmt)
    torch.manual_seed(m)
    x8 = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
    y = lin(x8, scale=0.25)
    torch.cuda.synchronize()
    want, wd = ref_gemm(orc, lin, x8, 0.25, fmt)
    assert np.array_equal(wd, w)
    tol = 1e-3 * want.abs().max().item() + 1e-3
    err = (y - want).abs().max().item()
    assert err <= tol, f"max err {err} > {tol} (split_k={lin.split_k})"


@pytest.mark.gpu
@pytest.mark.parametrize("T", [8, 64, 256])
@pytest.mark.parametrize("m", [1, 200])
def test_fused_gemm_decode_geometries(orc, T, m):
    # every decode-warp geometry of the fused kernel: 4-window lanes (T <= 128),
    # 8-window lanes (T = 256), 24 or 16 decode warps (m <= 128 / m > 128)
    from paper_2510_02676_b200.fused import FusedLinear

    n, k = 512, 1024
    w = codec.synth(1.8, 0.05, n * k, 900 + T, fmt="e4m3").reshape(n, k)
    lin = FusedLinear(w, "e4m3", threads_per_block=T)
    torch.manual_seed(T + m)
    x8 = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
    y = lin(x8, scale=0.5)
    torch.cuda.synchronize()
    want, wd = ref_gemm(orc, lin, x8, 0.5, "e4m3")
    assert np.array_equal(wd, w)
    tol = 1e-3 * want.abs().max().item() + 1e-3
    assert (y - want).abs().max().item() <= tol


@pytest.mark.gpu
def test_back_to_back_decodes_into_one_buffer():
    # consecutive decodes overlap by programmatic dependent launch; the second
    # one's stores must still land after the first one's
    from paper_2510_02676_b200.device import Batch, DeviceTensor

    xs = [codec.synth(1.8, 0.05, 3_000_000, 40 + i) for i in range(3)]
    ds = [DeviceTensor(codec.encode_tensor(x, 256)) for x in xs]
    out = torch.empty(3_000_000, dtype=torch.uint8, device="cuda")
    bs = [Batch([d], [out]) for d in ds]
    for _ in range(4):
        for b in bs:
            b.decode()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), xs[-1])


@pytest.mark.gpu
def test_fused_gemm_back_to_back_and_graph(orc):
    # the GEMM is the programmatic dependent of its X-swizzle kernel, which
    # also zeroes y: back-to-back calls into one y (no host sync) and a CUDA
    # graph replay must give the single-call result
    from paper_2510_02676_b200.fused import FusedLinear

    n, k, m = 512, 1024, 16
    w = codec.synth(1.8, 0.05, n * k, 77).reshape(n, k)
    lin = FusedLinear(w)
    xs = [(torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn) for _ in range(3)]
    want = []
    for x in xs:
        y = torch.empty(m, n, device="cuda")
        lin(x, 1.0, y)
        torch.cuda.synchronize()
        want.append(y.clone())
    y = torch.full((m, n), 7.0, device="cuda")
    for _ in range(3):
        for x in xs:
            lin(x, 1.0, y)
    torch.cuda.synchronize()
    # split-K partial sums are added atomically: equal up to fp32 reassociation
    torch.testing.assert_close(y, want[-1], rtol=1e-5, atol=1e-3)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        lin(xs[0], 1.0, y)  # warm-up on the capture stream
        with torch.cuda.graph(g, stream=s):
            lin(xs[1], 1.0, y)
    torch.cuda.synchronize()
    y.fill_(3.0)
    g.replay()
    torch.cuda.synchronize()
    torch.testing.assert_close(y, want[1], rtol=1e-5, atol=1e-3)

"""Just-in-time per-layer decode (paper_2510_02676_b200/hooks.py).

GPU: the ECF8Linear forward equals the same FP8 GEMM run on the weights
decoded by the CPU oracle (bit-identical bytes -> identical GEMM output), all
layers share one grow-only arena, E4M3 and E5M2.
"""
import numpy as np
import pytest
import torch

from paper_2510_02676_b200 import codec

from _oracle import tensor_dict

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", ["e4m3", "e5m2"])
@pytest.mark.parametrize("m", [1, 16, 33])
def test_ecf8_linear_matches_fp8_gemm_on_reference_decoded_weights(orc, fmt, m):
    from paper_2510_02676_b200.hooks import _FP8, DecodeArena, ECF8Linear

    n, k = 256, 512
    w = codec.synth(1.8, 0.05, n * k, 11, fmt=fmt).reshape(n, k)
    lin = ECF8Linear(w, scale_w=0.5, fmt=fmt, arena=DecodeArena())
    wd = orc.decode_parallel(tensor_dict(lin.encoded)).reshape(n, k)  # reference-decoded W
    assert np.array_equal(wd, w)
    x = torch.randn(m, k, device="cuda")
    sx = torch.tensor(0.01, device="cuda")
    y = lin(x, sx)
    xq = (x / sx).to(torch.float8_e4m3fn)
    pad = (-m) % 16
    xq = torch.cat([xq, xq.new_zeros(pad, k)]) if pad else xq
    wt = torch.from_numpy(wd).cuda().view(_FP8[fmt])
    want = torch._scaled_mm(xq, wt.t(), scale_a=sx, scale_b=torch.tensor(0.5, device="cuda"),
                            out_dtype=torch.bfloat16)[:m]
    # the arena holds exactly the reference-decoded bytes ...
    assert np.array_equal(lin.decode_weight().view(torch.uint8).cpu().numpy(), wd)
    # ... and the GEMM on them matches cuBLASLt on the reference bytes (cuBLASLt
    # may pick a different split per call: equal up to bf16 rounding)
    wf = want.float()
    scale = wf[wf.isfinite()].abs().max().item()
    torch.testing.assert_close(y.float(), wf, rtol=1e-2, atol=1e-2 * scale, equal_nan=True)
    # and against an fp32 dequantised reference within FP8-GEMM tolerance
    ref = (xq[:m].float() * sx) @ (wt.float() * 0.5).t()
    fin = ref.isfinite()
    torch.testing.assert_close(y.float()[fin], ref[fin], rtol=2e-2, atol=2e-2 * ref[fin].abs().max().item())


def test_compress_linears_shares_one_arena():
    from paper_2510_02676_b200.hooks import ECF8Linear, compress_linears

    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(512, 1024), torch.nn.GELU(), torch.nn.Linear(1024, 256),
                                torch.nn.GELU(), torch.nn.Linear(256, 512)).cuda()
    x = torch.randn(8, 512, device="cuda")
    with torch.no_grad():
        ref = model(x)
        mods = compress_linears(model, fused=False)  # the just-in-time decode path
        assert len(mods) == 3 and all(isinstance(m, ECF8Linear) for m in mods.values())
        y = model(x)
        y2 = model(x)
    arena = next(iter(mods.values())).arena
    assert all(m.arena is arena for m in mods.values())
    assert arena.capacity >= 1024 * 512 and arena.allocations <= 3
    assert torch.equal(y, y2)  # re-decoding is deterministic
    rel = (y.float() - ref).norm() / ref.norm()
    assert rel < 0.1  # FP8 weight + activation quantisation error only


def test_compress_linears_fused_matches_decode_then_gemm():
    from paper_2510_02676_b200.hooks import compress_linears

    torch.manual_seed(1)
    make = lambda: torch.nn.Sequential(torch.nn.Linear(512, 1024), torch.nn.GELU(),  # noqa: E731
                                       torch.nn.Linear(1024, 256)).cuda()
    a = make()
    b = make()
    b.load_state_dict(a.state_dict())
    x = torch.randn(8, 512, device="cuda")
    with torch.no_grad():
        ma = compress_linears(a, fused=True)
        mb = compress_linears(b, fused=False)
        assert all(m.fused is not None for m in ma.values()) and all(m.fused is None for m in mb.values())
        ya, yb = a(x), b(x)
    torch.testing.assert_close(ya.float(), yb.float(), rtol=2e-2, atol=2e-2 * yb.float().abs().max().item())

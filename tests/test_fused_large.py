"""Decode-fused tcgen05 FP8 GEMM (row a17) at the shapes the bench times.

With >= 4096 weight tiles every CTA of the fused plan owns a long run of K
tiles, so these tests exercise what the small-shape tests cannot: the A-ring
wrap and the stage-release waits (wait_stage_free / g_consumed), TMEM
accumulation across K tiles, the 2-4 segment epilogues of split-K runs, and
the single-X-stage reissue for m > 128.

Comparators:
  * y_ref  = torch._scaled_mm (cuBLASLt FP8, fp32 out) on the weights the
             reference decoder (C oracle, codec.cpp:256-273 restated) decodes
             from the same ECF8 stream -- the paper's decode-then-use
             (PAPER.md:170-173);
  * y64    = the same product in fp64 (exact: FP8 x FP8 products and their
             sums over K <= 28672 fit the fp64 mantissa).

Stated tolerance (fp32 accumulation, any order, split-K partial sums added
atomically): the classical bound |fl(sum) - sum| <= gamma_K * sum |x_i w_i|
with gamma_K = K u / (1 - K u), u = 2^-24, plus one rounding for the scale:
    |y - y64| <= (gamma_K + u) * scale * (|x| @ |w|^T)     elementwise.
Both the fused kernel and cuBLASLt are held to it.  The test also records the
observed max error relative to max|y64|.
"""
import functools

import numpy as np
import pytest
import torch

from paper_2510_02676_b200 import codec
from paper_2510_02676_b200.fused import fused_layout_inverse

from _oracle import tensor_dict

pytestmark = pytest.mark.gpu

U = 2.0 ** -24
_DT = {"e4m3": torch.float8_e4m3fn, "e5m2": torch.float8_e5m2}


@functools.lru_cache(maxsize=2)
def _weight(n, k, fmt, T):
    """FusedLinear over a synthetic alpha-stable weight, plus the weight the
    reference decoder recovers from its ECF8 stream (row-major [n, k])."""
    from _oracle import oracle
    from paper_2510_02676_b200.fused import FusedLinear

    w = codec.synth(1.8, 0.05, n * k, 1000 + n + 7 * k + T, fmt=fmt).reshape(n, k)
    lin = FusedLinear(w, fmt, threads_per_block=T)
    seq = oracle().decode_parallel(tensor_dict(lin.encoded), nthreads=0)
    wd = fused_layout_inverse(seq, n, k)
    assert np.array_equal(wd, w), "reference decode of the tiled stream != original weight"
    return lin, torch.from_numpy(wd).cuda().view(_DT[fmt])


def _check(lin, w8, m, scale, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x8 = (torch.randn(m, lin.k, device="cuda", generator=g) * 4).to(torch.float8_e4m3fn)
    y = torch.full((m, lin.n), float("nan"), device="cuda")
    lin(x8, scale=scale, out=y)
    # comparators
    pad = (-m) % 16
    xp = torch.cat([x8, x8.new_zeros(pad, lin.k)]) if pad else x8
    one = torch.tensor(1.0, device="cuda")
    y_ref = torch._scaled_mm(xp, w8.t(), scale_a=one, scale_b=one, out_dtype=torch.float32)[:m] * scale
    x64, w64 = x8.double(), w8.double()
    y64 = (x64 @ w64.t()) * scale
    mag = (x64.abs() @ w64.abs().t()) * abs(scale)
    K = lin.k
    gamma = K * U / (1 - K * U)
    bound = (gamma + U) * mag + 1e-30
    torch.cuda.synchronize()
    assert torch.isfinite(y).all(), "fused GEMM left unwritten outputs"
    err = (y.double() - y64).abs()
    err_ref = (y_ref.double() - y64).abs()
    worst = (err / bound).max().item()
    worst_ref = (err_ref / bound).max().item()
    rel = err.max().item() / max(y64.abs().max().item(), 1e-30)
    assert worst <= 1.0, f"fused: max err / bound = {worst:.3f} (rel {rel:.2e}, split_k={lin.split_k})"
    assert worst_ref <= 1.0, f"cuBLASLt comparator outside the stated bound: {worst_ref:.3f}"
    # fused vs the plain FP8 GEMM on reference-decoded weights: both within the bound of y64
    assert ((y.double() - y_ref.double()).abs() <= 2 * bound).all()
    return rel


@pytest.mark.parametrize("m", [1, 16, 64, 128, 129, 256])
def test_fused_llama70b_qo_8192x8192(m):
    lin, w8 = _weight(8192, 8192, "e4m3", 128)
    assert lin.split_k > 1  # 4096 tiles over the SMs: multi-K-tile runs that straddle n-tiles
    _check(lin, w8, m, 0.5, m)


@pytest.mark.parametrize("m", [1, 256])
def test_fused_llama70b_gate_up_28672x8192(m):
    lin, w8 = _weight(28672, 8192, "e4m3", 128)
    _check(lin, w8, m, 1.0, 100 + m)


@pytest.mark.parametrize("m", [16, 200])
def test_fused_llama70b_down_8192x28672(m):
    lin, w8 = _weight(8192, 28672, "e4m3", 128)
    _check(lin, w8, m, 0.25, 200 + m)


@pytest.mark.parametrize("m", [1, 64, 256])
def test_fused_e5m2_8192x8192(m):
    # E5M2 weights carry 1-bit codes at gamma 0.05: the 64-symbol lane geometry
    lin, w8 = _weight(8192, 8192, "e5m2", 128)
    _check(lin, w8, m, 0.5, 300 + m)


@pytest.mark.parametrize("m", [1, 130])
def test_fused_T256_lanes_4096x8192(m):
    # T = 256: 8-window lanes (the standalone decoder's geometry)
    lin, w8 = _weight(4096, 8192, "e4m3", 256)
    _check(lin, w8, m, 1.0, 400 + m)


@pytest.mark.parametrize("m", [16, 200])
@pytest.mark.parametrize("k", [128, 256])
def test_fused_many_segments_per_cta(m, k):
    # K = 1 or 2 tiles per output n-tile: a CTA's run of ~3.5 tiles spans up to
    # five n-tiles; at m > 128 only two 256-column accumulators fit TMEM, so
    # segments reuse them round-robin (flushed by warps 0-3 first)
    n = 128 * 518
    lin, w8 = _weight(n, k, "e4m3", 128)
    _check(lin, w8, m, 1.0, 500 + m + k)


@pytest.mark.parametrize("m", [100, 256])
def test_fused_accumulator_reuse_long_runs(m):
    # 2000 n-tiles of one K tile: every CTA's run of ~13.5 tiles is ~14
    # segments, more than the 4 (m <= 128) or 2 (m > 128) accumulator
    # buffers -- each buffer is flushed and reused several times per CTA
    lin, w8 = _weight(128 * 2000, 128, "e4m3", 128)
    _check(lin, w8, m, 0.5, 600 + m)


def test_fused_out_is_validated():
    lin, _ = _weight(4096, 8192, "e4m3", 256)
    x8 = torch.zeros(4, lin.k, device="cuda").to(torch.float8_e4m3fn)
    for bad in (torch.empty(4, lin.n, device="cuda", dtype=torch.bfloat16),
                torch.empty(3, lin.n, device="cuda"),
                torch.empty(lin.n, 4, device="cuda").t(),
                torch.empty(4, lin.n)):
        with pytest.raises(ValueError):
            lin(x8, 1.0, bad)


@pytest.mark.parametrize("m", [129, 256])
def test_large_m_rows_pipeline_matches(m):
    # m >= LARGE_M: W decoded in chunks of whole 128-row tiles back to
    # row-major (ecf8_fused_decode_rows) + dense FP8 GEMM per chunk; several
    # chunks (the two-slot ring wraps), same bound as the fused kernel
    from paper_2510_02676_b200 import fused

    lin, w8 = _weight(28672, 8192, "e4m3", 128)
    assert lin.rows_ok and 28672 * 8192 > 3 * fused.CHUNK_BYTES
    old, fused.LARGE_M = fused.LARGE_M, 129  # the path is opt-in
    try:
        _check(lin, w8, m, 0.75, 700 + m)
    finally:
        fused.LARGE_M = old


def test_decode_rows_back_to_row_major():
    import torch

    from paper_2510_02676_b200 import _lib

    lin, w8 = _weight(4096, 8192, "e4m3", 256)
    out = torch.empty(1024 * 8192 + 16, dtype=torch.uint8, device="cuda")
    for r0, r1 in ((0, 128), (1920, 2944), (3968, 4096)):
        _lib.check(_lib.lib.ecf8_fused_decode_rows(lin.handle, r0, r1, out.data_ptr(), None))
        torch.cuda.synchronize()
        got = out[: (r1 - r0) * 8192].view(r1 - r0, 8192)
        assert torch.equal(got, w8[r0:r1].view(torch.uint8))
    with pytest.raises(_lib.InvalidArgument, match="whole 128-row tiles"):
        _lib.check(_lib.lib.ecf8_fused_decode_rows(lin.handle, 5, 128, out.data_ptr(), None))


def test_back_to_back_calls_share_the_stream_workspace():
    # Calls on one stream share one workspace (swizzled X, the L2 rings) and
    # chain by programmatic dependent launch: the same weight twice in a row
    # and two weights alternating, every call with its own x and y, all
    # enqueued before one synchronize -- each y within the stated bound.
    lin_a, w_a = _weight(4096, 8192, "e4m3", 128)
    lin_b, w_b = _weight(1024, 8192, "e4m3", 128)
    order = [(lin_a, w_a), (lin_a, w_a), (lin_b, w_b), (lin_a, w_a), (lin_b, w_b), (lin_b, w_b), (lin_a, w_a)]
    calls = []
    for i, (lin, w8) in enumerate(order):
        m = (1, 16, 64, 200)[i % 4]
        g = torch.Generator(device="cuda").manual_seed(500 + i)
        x8 = (torch.randn(m, lin.k, device="cuda", generator=g) * 4).to(torch.float8_e4m3fn)
        y = torch.full((m, lin.n), float("nan"), device="cuda")
        lin(x8, scale=1.0, out=y)
        calls.append((x8, w8, y))
    torch.cuda.synchronize()
    for x8, w8, y in calls:
        x64, w64 = x8.double(), w8.double()
        y64 = x64 @ w64.t()
        K = x8.shape[1]
        gamma = K * U / (1 - K * U)
        bound = (gamma + U) * (x64.abs() @ w64.abs().t()) + 1e-30
        assert torch.isfinite(y).all()
        assert ((y.double() - y64).abs() / bound).max().item() <= 1.0

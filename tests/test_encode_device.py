"""Device encoder and exponent histogram.

GPU cases compare ecf8_encode_device's sections byte for byte with the
oracle's encoder (oracle/ecf8_oracle.c, restating codec.cpp:49-98) and the
host encoder, then decode the GPU-encoded tensor on the GPU.  The histogram
is checked against a numpy count of the exponent field (fp8.hpp:24-30).
CPU cases check argument validation, which comes before the device check.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2510_02676_b200 import _lib, codec

from _oracle import tensor_dict

LADDER = np.array([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 16, 16], np.uint8)
L16 = np.array([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16], np.uint8)  # Kraft 1 - 2^-16


def _encode_raw(n, T, lengths):
    h = C.c_void_p()
    lv = np.ascontiguousarray(np.asarray(lengths, np.uint8))
    return _lib.lib.ecf8_encode_device(None, n, T, lv.ctypes.data_as(C.c_void_p), None, C.byref(h))


def test_validation_before_device():
    with pytest.raises(_lib.InvalidArgument, match="power of two"):
        _lib.check(_encode_raw(0, 3, LADDER))
    with pytest.raises(_lib.InvalidArgument, match="invalid length vector"):
        _lib.check(_encode_raw(0, 256, np.full(16, 1, np.uint8)))
    with pytest.raises(_lib.InvalidArgument, match="invalid length vector"):
        _lib.check(_encode_raw(0, 256, np.zeros(16, np.uint8)))


def test_no_device_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(_lib.CudaError, match="no CUDA device"):
        _lib.check(_encode_raw(0, 256, LADDER))
    counts = np.zeros(16, np.uint64)
    with pytest.raises(_lib.CudaError, match="no CUDA device"):
        _lib.check(_lib.lib.ecf8_exponent_histogram(None, 0, counts.ctypes.data_as(C.POINTER(C.c_uint64)), None))


# ------------------------------------------------------------------ GPU


def _dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _same(got, want, what):
    for k in ("encoded", "gaps", "outpos", "packed"):
        a, b = np.asarray(getattr(got, k)), np.asarray(want[k])
        assert a.shape == b.shape, f"{what}: {k} size {a.shape} vs {b.shape}"
        if not np.array_equal(a, b):
            i = int(np.flatnonzero(a != b)[0])
            raise AssertionError(f"{what}: {k} differs at {i}: {a[i]} vs {b[i]}")
    assert np.array_equal(np.asarray(got.lengths), want["lengths"])


def _roundtrip(orc, x, T, lengths=None):
    from paper_2510_02676_b200.device import DeviceTensor

    if lengths is None:
        lengths = orc.build_code(np.bincount((x >> 3) & 15, minlength=16).astype(np.uint64)) if x.size else LADDER
    dt = DeviceTensor.encode(_dev(x), lengths, T)
    got = dt.to_host()
    _same(got, orc.encode(x, lengths, T), f"T={T} n={x.size}")
    if x.size:
        _same(got, tensor_dict(codec.encode_tensor(x, T, lengths)), f"host encoder T={T} n={x.size}")
        assert np.array_equal(dt.decode().cpu().numpy(), x)
    return dt


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 2, 15, 16, 17, 4095, 4096, 4097, 65537, 1_000_003])
def test_histogram(n):
    from paper_2510_02676_b200.device import exponent_histogram

    rng = np.random.default_rng(n)
    x = rng.integers(0, 256, n + 1, dtype=np.uint8)
    want = np.bincount((x[1:] >> 3) & 15, minlength=16).astype(np.uint64)
    got = exponent_histogram(_dev(x)[1:])  # misaligned start
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("T", [1, 2, 8, 64, 128, 256, 1024])
def test_encode_matches_oracle_synth(orc, T):
    for n, seed in ((1, 1), (4097, 2), (200_003, 3)):
        x = codec.synth(1.8, 0.05, n, seed)
        _roundtrip(orc, x, T)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 63, 64, 65, 4095, 4096, 4097, 8193, 100_000])
def test_encode_sizes_and_distributions(orc, n):
    rng = np.random.default_rng(7 + n)
    for dist in range(3):
        if dist == 0:
            x = rng.integers(0, 256, n, dtype=np.uint8)
        elif dist == 1:
            x = np.where(rng.random(n) < 0.9, 0x38, rng.integers(0, 256, n)).astype(np.uint8)
        else:
            x = np.full(n, 0xB8, np.uint8)  # one symbol: a 1-bit code
        for T in (1, 32, 256):
            _roundtrip(orc, x, T)


@pytest.mark.gpu
def test_encode_long_codes_and_gap15(orc):
    # 16-bit code words (LADDER / L16) and the gap-15 straddle (test_codec.cpp:282-305)
    sym = np.array([0] * 63 + [15, 14] + [0] * 200, np.uint8)
    i = np.arange(sym.size)
    x = ((sym << 3) | ((i % 16) << 4 & 0x80) | (i % 8)).astype(np.uint8)
    for T in (1, 2, 32, 256):
        _roundtrip(orc, x, T, LADDER)
    rng = np.random.default_rng(5)
    s = rng.integers(0, 16, 50_000).astype(np.uint8)
    x = ((s << 3) | (rng.integers(0, 2, s.size) << 7) | rng.integers(0, 8, s.size)).astype(np.uint8)
    for T in (1, 64, 256, 1024):
        _roundtrip(orc, x, T, L16)


@pytest.mark.gpu
def test_encode_e5m2_bytes(orc):
    x = codec.synth(1.8, 0.05, 300_001, 11, fmt="e5m2")
    dt = _roundtrip(orc, x, 256)
    assert dt.kernel_variant in (4, 5, 6, 7)


@pytest.mark.gpu
def test_encode_auto_code_and_tiles():
    import torch

    from paper_2510_02676_b200.device import DeviceTensor

    x = codec.synth(1.8, 0.05, 3_000_000, 21)
    dt = DeviceTensor.encode(torch.from_numpy(x).cuda())  # lengths from the GPU histogram
    host = codec.encode_tensor(x, 256)
    _same(dt.to_host(), tensor_dict(host), "auto code")
    ok, total = dt.verified_tiles()
    assert ok == total > 0
    assert torch.equal(dt.decode().cpu(), torch.from_numpy(x))


@pytest.mark.gpu
def test_encode_absent_symbol():
    import torch

    from paper_2510_02676_b200.device import DeviceTensor

    lengths = np.array([1, 1] + [0] * 14, np.uint8)  # only exponents 0 and 1 have codes
    x = torch.tensor([0x00, 0x08, 0x10], dtype=torch.uint8).cuda()  # exponent 2 has none
    with pytest.raises(_lib.InvalidArgument, match="symbol absent from code table"):
        DeviceTensor.encode(x, lengths, 256)


def test_host_make_stats():
    # container.cpp:386-413 on synth data: savings near the survey's 17.96 % (α 1.8, γ 0.05)
    x = codec.synth(1.8, 0.05, 1 << 20, 1)
    r = codec.make_stats(x, 256, name_len=6, rank=2)
    assert r["n_elem"] == x.size
    assert 2.2 < r["entropy_bits"] < r["bits_per_symbol"] < 2.6
    assert r["bits_per_weight"] == 4.0 + r["bits_per_symbol"]
    # the container's gaps (4 bits per 64-bit window) and offsets cost ~2 points
    assert 0 < r["projected_savings"] - r["actual_savings"] < 0.03
    t = codec.encode_tensor(x, 256)
    sections = t.compressed_bytes() + (2 + 6) + 1 + 2 * 8 + (8 + 4 + 16 + 8 + 8 + 8)  # tensor_section_bytes
    assert r["actual_savings"] == 1.0 - sections / x.size


@pytest.mark.gpu
@pytest.mark.parametrize("n, T", [(0, 256), (1, 1), (4097, 32), (1_000_003, 256), (2_000_000, 1024)])
def test_make_stats_device_matches_host(n, T):
    from paper_2510_02676_b200.device import make_stats_device

    x = codec.synth(1.8, 0.05, n, 3) if n else np.zeros(0, np.uint8)
    want = codec.make_stats(x, T, name_len=9, rank=2)
    got = make_stats_device(_dev(x) if n else _dev(np.zeros(1, np.uint8))[:0], T, name_len=9, rank=2)
    assert got == want

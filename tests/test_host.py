"""Product host library (encoder, codes, container, synth) vs oracle / reference.

CPU-only: nothing here decodes on the device.  Byte-identity of containers
with the reference is the drop-in requirement for the encoder side.
"""
import numpy as np
import pytest

from paper_2510_02676_b200 import codec
from paper_2510_02676_b200._lib import FormatError, InvalidArgument

from _oracle import tensor_dict


def random_hist(rng, k_max=16, c_max=1 << 20):
    h = np.zeros(16, np.uint64)
    for _ in range(int(rng.integers(1, k_max + 1))):
        h[rng.integers(0, 16)] += rng.integers(1, c_max)
    return h


def test_build_code_matches_oracle(orc):
    rng = np.random.default_rng(1)
    for _ in range(500):
        h = random_hist(rng)
        assert np.array_equal(codec.build_code(h), orc.build_code(h))


def test_build_code_exhaustive_small(orc):
    # every histogram over <= 4 symbols with counts 1..6 (test_huffman.cpp:130-163 style)
    import itertools

    for k in range(1, 5):
        for counts in itertools.product(range(1, 7), repeat=k):
            h = np.zeros(16, np.uint64)
            h[[0, 5, 9, 15][:k]] = counts
            assert np.array_equal(codec.build_code(h), orc.build_code(h))


def test_build_lut_matches_oracle(orc):
    rng = np.random.default_rng(2)
    for _ in range(300):
        l = codec.build_code(random_hist(rng))
        e1, n1 = codec.build_lut(l)
        e2, n2 = orc.build_lut(l)
        assert n1 == n2 and np.array_equal(e1, e2)


def test_invalid_lengths_rejected():
    with pytest.raises(InvalidArgument, match="invalid length vector"):
        codec.build_lut(np.zeros(16, np.uint8))
    with pytest.raises(InvalidArgument):
        codec.build_lut(np.ones(16, np.uint8))
    bad = np.zeros(16, np.uint8)
    bad[0] = 17
    with pytest.raises(InvalidArgument):
        codec.build_lut(bad)


@pytest.mark.parametrize("T", [1, 2, 32, 256, 512, 1024])
def test_encoder_byte_identical_to_oracle(orc, T):
    rng = np.random.default_rng(T)
    for n in (1, 7, 64, 65, 1000, 40000):
        x = rng.integers(0, 256, n, dtype=np.uint8)
        mine = tensor_dict(codec.encode_tensor(x, T))
        theirs = orc.encode_auto(x, T)
        for k in ("encoded", "gaps", "outpos", "packed", "lengths"):
            assert np.array_equal(mine[k], theirs[k]), k


def test_encoder_rejects_absent_symbol():
    l = np.zeros(16, np.uint8)
    l[0] = l[1] = 1
    with pytest.raises(InvalidArgument, match="symbol absent"):
        codec.encode_tensor(np.array([0, 8, 16], np.uint8), 256, l)


def test_empty_tensor_encoding():
    t = codec.encode_tensor(np.zeros(0, np.uint8), 256)
    assert t.n_elem == 0 and list(t.encoded) == [0, 0] and list(t.outpos) == [0] and t.gaps.size == 0


def test_decode_reference_api_matches_oracle(orc):
    rng = np.random.default_rng(3)
    x = rng.integers(0, 256, 5000, dtype=np.uint8)
    t = codec.encode_tensor(x, 32)
    assert np.array_equal(codec.decode_reference(t), x)
    assert np.array_equal(orc.decode_reference(tensor_dict(t)), x)


def test_synth_bit_identical_across_threads():
    a = codec.synth(1.8, 0.05, 100003, 11, nthreads=1)
    b = codec.synth(1.8, 0.05, 100003, 11, nthreads=7)
    assert np.array_equal(a, b)


def test_synth_matches_reference(ref):
    for alpha, gamma, seed in ((1.8, 0.05, 1), (2.0, 0.70710678118654752, 9), (1.0, 2.0, 5)):
        assert np.array_equal(codec.synth(alpha, gamma, 50000, seed), ref.synth(alpha, gamma, 50000, seed))


def test_container_byte_identical_to_reference(ref):
    rng = np.random.default_rng(4)
    x = codec.synth(1.8, 0.05, 30000, 2)
    y = rng.integers(0, 256, 999, dtype=np.uint8)
    raw = codec.raw_file([("a", [100, 300], x), ("empty", [0], np.zeros(0, np.uint8)), ("y", [999], y)])
    for T in (1, 2, 32, 256, 1024):
        assert codec.compress_raw(raw, T) == ref.compress_raw(raw, T)


def test_container_parse_roundtrip():
    rng = np.random.default_rng(5)
    x = rng.integers(0, 256, 3000, dtype=np.uint8)
    blob = codec.compress_raw(codec.raw_file([("w", [3000], x)]), 32)
    f = codec.parse_container(blob)
    (name, t), = f.tensors
    assert name == "w" and t.n_elem == 3000 and t.threads_per_block == 32
    assert np.array_equal(codec.decode_reference(t), x)


def _good_container():
    rng = np.random.default_rng(54)
    x = rng.integers(0, 256, 300, dtype=np.uint8)
    return codec.compress_raw(codec.raw_file([("t", [300], x)]), 2)


@pytest.mark.parametrize(
    "mutate,msg",
    [
        (lambda b: b"X" + b[1:], "bad magic"),
        (lambda b: b[:4] + b"\x09" + b[5:], "unsupported version"),
        (lambda b: b + b"\x00", "trailing bytes after last tensor"),
        (lambda b: b[: len(b) // 2], "truncated file"),
    ],
)
def test_container_malformations(mutate, msg):
    # test_container.cpp:103-206 (message strings pinned)
    with pytest.raises(FormatError, match=msg):
        codec.parse_container(mutate(_good_container()))


def test_container_section_checks():
    b = bytearray(_good_container())
    # header 12 + name_len 2 + 't' + rank 1 + dim 8 = 24 -> n_elem at 24, T at 32
    bad = bytearray(b)
    bad[32:36] = (3).to_bytes(4, "little")
    with pytest.raises(FormatError, match="invalid thread count"):
        codec.parse_container(bytes(bad))
    bad = bytearray(b)
    bad[36:52] = bytes([1] * 16)
    with pytest.raises(FormatError, match="invalid length vector in container"):
        codec.parse_container(bytes(bad))
    bad = bytearray(b)
    bad[24:32] = (301).to_bytes(8, "little")
    with pytest.raises(FormatError, match="element count does not match dims"):
        codec.parse_container(bytes(bad))


def test_e4m3_pinned():
    # test_fp8.cpp:98-115 via synth-free path: compare with the reference converter semantics
    import ctypes as C

    from paper_2510_02676_b200._lib import lib  # noqa: F401  (library loads)

    # e4m3 conversion is exercised through synth(); spot-check distribution sanity
    x = codec.synth(2.0, 0.70710678118654752, 200000, 9)
    h = np.bincount((x >> 3) & 15, minlength=16)
    assert int(np.argmax(h)) in (6, 7)  # test_container.cpp:391-426
    assert not np.any((x & 0x7F) == 0x7F)  # never the NaN pattern


def test_e5m2_synth_matches_torch():
    torch = pytest.importorskip("torch")
    x = codec.synth(1.8, 0.05, 50000, 3, fmt="e5m2")
    vals = torch.from_numpy(x.copy()).view(torch.float8_e5m2).float()
    assert torch.isfinite(vals).all()
    # re-quantizing the decoded values with torch reproduces the bytes
    back = vals.to(torch.float8_e5m2).view(torch.uint8).numpy()
    assert np.array_equal(back, x)

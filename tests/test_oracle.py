"""Pin the C oracle (oracle/ecf8_oracle.c) to the reference's own known answers.

Every expected value below is a golden vector from the reference suite
(/root/reference/proj/tests/*.cpp, cited per test).  Where the reference
library itself was built here (oracle/_ref), the oracle is also compared
with it on randomized inputs (test_oracle_vs_reference_*).
"""
import numpy as np
import pytest

LADDER = np.array([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 16, 16], np.uint8)


def hist(counts):
    h = np.zeros(16, np.uint64)
    h[: len(counts)] = counts
    return h


def test_worked_example_lengths_codes(orc):
    # test_huffman.cpp:41-62: counts {3,2,1,2,5} -> lengths {2,4,4,3,1}
    l = orc.build_code(hist([3, 2, 1, 2, 5]))
    assert list(l[:5]) == [2, 4, 4, 3, 1]
    c = orc.canonical_codes(l)
    assert (c[4], c[0], c[3], c[1], c[2]) == (0b0, 0b10, 0b110, 0b1110, 0b1111)


def test_worked_example_stream_bytes(orc):
    # test_codec.cpp:94-118: "aaabbcddeeeee" at T=1 -> ab bb f6, 29 bits
    sym = np.array([0, 0, 0, 1, 1, 2, 3, 3, 4, 4, 4, 4, 4], np.uint8)
    l = orc.build_code(hist([3, 2, 1, 2, 5]))
    t = orc.encode(sym << 3, l, 1)
    assert t["encoded"].size == 10
    assert list(t["encoded"][:3]) == [0xAB, 0xBB, 0xF6]
    assert not t["encoded"][3:].any()
    assert list(t["outpos"]) == [0, 13]
    assert t["gaps"][0] >> 4 == 0
    assert np.array_equal(orc.decode_reference(t), sym << 3)


def test_skewed_and_uniform_codes(orc):
    # test_huffman.cpp:65-98
    assert list(orc.build_code(hist([1, 1, 2, 4]))[:4]) == [3, 3, 2, 1]
    assert list(orc.build_code(np.full(16, 10, np.uint64))) == [4] * 16
    one = np.zeros(16, np.uint64)
    one[9] = 42
    l = orc.build_code(one)
    assert l[9] == 1 and l.sum() == 1


def test_powers_of_two_counts(orc):
    # test_huffman.cpp:100-109
    l = orc.build_code(np.array([1 << s for s in range(16)], np.uint64))
    assert l[0] == 15 and l[1] == 15
    assert [int(l[s]) for s in range(2, 16)] == [16 - s for s in range(2, 16)]


def test_ladder_codes_and_lut(orc):
    # test_huffman.cpp:188-217, test_lut.cpp:105-128
    c = orc.canonical_codes(LADDER)
    assert (c[0], c[13], c[14], c[15]) == (0, 0x3FFE, 0xFFFC, 0xFFFD)
    e, n = orc.build_lut(LADDER)
    assert n == 3 and e[0xFF] == 255
    assert orc.decode_one(e, n, 0xFFFC) == (14, 16)
    assert orc.decode_one(e, n, 0xFFFD) == (15, 16)
    assert orc.decode_one(e, n, 0xFFFE) == (0, 1)
    assert orc.decode_one(e, n, 0xFFFF) == (0, 1)


def test_count_phase_known_answers(orc):
    # test_codec.cpp:206-233
    l = np.zeros(16, np.uint8)
    l[5] = 1
    assert orc.count_phase(np.zeros(10, np.uint8), 0, l) == 64
    l = np.zeros(16, np.uint8)
    l[0], l[15] = 1, 16
    assert orc.canonical_codes(l)[15] == 0x8000
    w = np.zeros(10, np.uint8)
    w[1] = 0x01
    assert orc.count_phase(w, 15, l) == 34
    assert orc.count_phase(np.zeros(10, np.uint8), 15, l) == 49
    assert orc.count_phase(np.zeros(10, np.uint8), 0, l) == 64


def test_dyadic_200_symbols_T2(orc):
    # test_codec.cpp:179-204: 450 bits -> 4 blocks of 2 windows
    l = np.zeros(16, np.uint8)
    l[:4] = [1, 2, 3, 3]
    sym = (np.arange(200) % 4).astype(np.uint8)
    t = orc.encode(sym << 3, l, 2)
    assert t["outpos"].size == 5 and t["outpos"][-1] == 200
    assert np.array_equal(orc.decode_parallel(t), sym << 3)


def test_gap15_straddle(orc):
    # test_codec.cpp:282-305 / acceptance.cpp:127-141
    sym = np.array([0] * 63 + [15, 14] + [0] * 200, np.uint8)
    fp8 = (sym << 3) | ((np.arange(sym.size) % 16) << 4 & 0x80) | (np.arange(sym.size) % 8)
    fp8 = fp8.astype(np.uint8)
    for T in (1, 2, 32, 256):
        t = orc.encode(fp8, LADDER, T)
        assert (t["gaps"][0] & 15) == 15  # window 1: low nibble of byte 0
        assert np.array_equal(orc.decode_parallel(t), fp8)
        assert np.array_equal(orc.decode_reference(t), fp8)


@pytest.mark.parametrize("n", [0, 1, 2, 3, 7, 8, 63, 64, 65, 100, 513, 4096, 100000])
def test_parallel_reference_original_agree(orc, n):
    # test_codec.cpp:307-332 matrix
    rng = np.random.default_rng(41 + n)
    for dist in range(3):
        if dist == 0:
            x = rng.integers(0, 256, n, dtype=np.uint8)
        elif dist == 1:
            x = np.where(rng.random(n) < 0.9, 0x38, rng.integers(0, 256, n)).astype(np.uint8)
        else:
            x = np.full(n, 0xB8, np.uint8)
        for T in (1, 2, 32, 256):
            t = orc.encode_auto(x, T) if n else orc.encode(x, np.array([1] + [0] * 15, np.uint8), T)
            assert np.array_equal(orc.decode_parallel(t), x)
            assert np.array_equal(orc.decode_reference(t), x)


def test_truncated_stream_detected(orc):
    # test_codec.cpp:273-280
    l = orc.build_code(hist([1, 1, 2, 4]))
    t = orc.encode(np.full(100, 3 << 3, np.uint8), l, 1)
    t["n_elem"] = 1 << 20
    t["packed"] = np.zeros((1 << 19) + 1, np.uint8)
    with pytest.raises(ValueError):
        orc.decode_reference(t)


# --------------------------------------------- oracle vs the real reference


def test_oracle_vs_reference_codes(orc, ref):
    rng = np.random.default_rng(7)
    for _ in range(300):
        h = np.zeros(16, np.uint64)
        for _ in range(rng.integers(1, 17)):
            h[rng.integers(0, 16)] += rng.integers(1, 1 << 20)
        l = orc.build_code(h)
        assert np.array_equal(l, ref.build_code(h))
        e1, n1 = orc.build_lut(l)
        e2, n2 = ref.build_lut(l)
        assert n1 == n2 and np.array_equal(e1, e2)


def test_oracle_vs_reference_counts(orc, ref):
    rng = np.random.default_rng(8)
    for _ in range(200):
        h = np.zeros(16, np.uint64)
        for _ in range(rng.integers(1, 17)):
            h[rng.integers(0, 16)] += rng.integers(1, 5000)
        l = orc.build_code(h)
        w = rng.integers(0, 256, 10, dtype=np.uint8)
        g = int(rng.integers(0, 16))
        assert orc.count_phase(w, g, l) == ref.count_phase(w, g, l)


def test_oracle_vs_reference_containers(orc, ref):
    from paper_2510_02676_b200.codec import raw_file

    rng = np.random.default_rng(9)
    for T in (1, 2, 32, 256, 1024):
        x = ref.synth(1.8, 0.05, 20000, 3 + T)
        y = rng.integers(0, 256, 777, dtype=np.uint8)
        blob = ref.compress_raw(raw_file([("x", [20000], x), ("y", [777], y)]), T)
        t = orc.encode_auto(x, T)
        # section bytes of tensor 0 must sit verbatim in the reference container
        assert t["encoded"].tobytes() in blob and t["packed"].tobytes() in blob
        assert np.array_equal(orc.decode_parallel(t), x)


def test_reference_arm_legs_agree(ref):
    """The bench reference arm's CPU legs: decode_parallel_into at 1 and all
    threads, decode_reference, and the x86-64-v4 build decode the same bytes."""
    from _oracle import reference_v4

    from paper_2510_02676_b200.codec import raw_file

    x = ref.synth(1.8, 0.05, 50000, 17)
    blob = ref.compress_raw(raw_file([("x", [50000], x)]), 256)
    (h,) = ref.container_tensors(blob)
    try:
        assert np.array_equal(ref.decode(h, x.size, 0)[0], x)
        assert np.array_equal(ref.decode(h, x.size, 1)[0], x)
        assert np.array_equal(ref.decode_reference(h, x.size)[0], x)
    finally:
        ref.free(h)
    r4 = reference_v4()
    if r4 is not None:
        (h4,) = r4.container_tensors(blob)
        try:
            assert np.array_equal(r4.decode(h4, x.size, 0)[0], x)
        finally:
            r4.free(h4)

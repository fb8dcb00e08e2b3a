"""Device decode tables (csrc/cuda/tables.cpp) vs the reference cascade.

The B200 kernels decode several symbols per shared-memory load from a
multi-symbol table.  These CPU tests prove the table is equivalent to the
reference's decode_one walk (lut.hpp:43-49, built by the oracle):
  * every fast entry's symbols / bit count equal the cascade walk for every
    completion of the bits beyond the index;
  * a numpy model of the kernel's count loop (decode.cu count_window)
    reproduces the oracle's count_phase on random windows.
"""
import numpy as np
import pytest

from paper_2510_02676_b200 import codec


def random_lengths(rng):
    # test_util.hpp:98-117 style Kraft-feasible, possibly incomplete codes
    k = int(rng.integers(1, 17))
    syms = rng.permutation(16)[:k]
    lengths = np.zeros(16, np.uint8)
    remaining = 1 << 16
    for i, s in enumerate(syms):
        reserve = k - 1 - i
        feas = [L for L in range(1, 17) if (1 << (16 - L)) + reserve <= remaining]
        L = int(rng.choice(feas))
        lengths[s] = L
        remaining -= 1 << (16 - L)
    return lengths


LADDER = np.array([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 16, 16], np.uint8)


def cascade_walk(casc, n_luts, stream, pos):
    """Vectorised decode_one on uint64 streams at bit offsets pos (<= 48)."""
    w = (stream >> (np.uint64(48) - pos.astype(np.uint64))) & np.uint64(0xFFFF)
    w = w.astype(np.int64)
    v = casc[w >> 8].astype(np.int64)
    ptr = v >= 240
    v = np.where(ptr, casc[np.where(ptr, (256 - v) * 256 + (w & 255), 0)], v)
    bits = casc[(n_luts - 1) * 256 + v]
    return v, bits.astype(np.int64)


def length_sets():
    rng = np.random.default_rng(2026)
    sets = [LADDER, np.array([1] + [0] * 15, np.uint8), np.array([0] * 11 + [1] + [0] * 4, np.uint8)]
    l = np.zeros(16, np.uint8)
    l[:4] = [1, 2, 3, 3]
    sets.append(l)
    sets.append(codec.build_code(np.array([1 << s for s in range(16)], np.uint64)))
    x = codec.synth(1.8, 0.05, 200000, 1)
    sets.append(codec.build_code(np.bincount((x >> 3) & 15, minlength=16).astype(np.uint64)))
    sets += [random_lengths(rng) for _ in range(40)]
    return sets


@pytest.mark.parametrize("case", range(46))
def test_fast_entries_equal_cascade_walk(case):
    lengths = length_sets()[case]
    fast, smask, casc, n_luts, K = codec.device_tables(lengths)
    assert fast.size == 1 << K
    rng = np.random.default_rng(case)
    idx = np.repeat(np.arange(1 << K, dtype=np.uint64), 8)
    tail = rng.integers(0, 1 << 62, idx.size, dtype=np.uint64) >> np.uint64(K - 2)
    stream = (idx << np.uint64(64 - K)) | tail
    ii = idx.astype(np.int64)
    e = fast[ii].astype(np.int64)
    b, n, syms = e & 31, ((e >> 5) & 31) // 4, e >> 12
    assert np.all(((e >> 5) & 3) == 0) and np.all(n <= 5)
    pos = np.zeros(idx.size, np.int64)
    starts = np.zeros(idx.size, np.int64)
    for i in range(6):
        live = n > i
        if not live.any():
            break
        starts |= np.where(live, 1 << pos, 0)
        s, bits = cascade_walk(casc, n_luts, stream, pos)
        assert np.all(s[live] == ((syms[live] >> (4 * i)) & 15))
        pos = np.where(live, pos + bits, pos)
    assert np.all(pos == b)
    assert np.all(b <= K)
    assert np.array_equal(smask[ii].astype(np.int64), starts)


def count_model(fast, smask, casc, n_luts, K, window10, gap):
    """Python model of decode.cu decode_window (count mode) on one window."""
    bits = np.unpackbits(np.concatenate([window10, np.zeros(8, np.uint8)]))
    stream = int("".join(map(str, bits)), 2)  # 144-bit integer
    nbits = bits.size

    def peek(p, k):
        return (stream >> (nbits - p - k)) & ((1 << k) - 1)

    p, c = gap, 0
    while True:
        idx = peek(p, K)
        e = int(fast[idx])
        b, n = e & 31, ((e >> 5) & 31) // 4
        if n == 0:  # reference cascade on 16 bits
            w = peek(p, 16)
            v = int(casc[w >> 8])
            if v >= 240:
                v = int(casc[(256 - v) * 256 + (w & 255)])
            c, p = c + 1, p + int(casc[(n_luts - 1) * 256 + v])
            if p >= 64:
                return c
            continue
        r = 64 - p
        if b >= r:
            return c + bin(int(smask[idx]) & ((1 << r) - 1)).count("1")
        c, p = c + n, p + b


@pytest.mark.parametrize("case", range(0, 46, 3))
def test_count_model_matches_oracle(orc, case):
    lengths = length_sets()[case]
    fast, smask, casc, n_luts, K = codec.device_tables(lengths)
    rng = np.random.default_rng(100 + case)
    for _ in range(60):
        w = rng.integers(0, 256, 10, dtype=np.uint8)
        if rng.random() < 0.3:
            w[:] = 0
        g = int(rng.integers(0, 16))
        assert count_model(fast, smask, casc, n_luts, K, w, g) == orc.count_phase(w, g, lengths)

"""Byte-step decoder tables (tables.hpp fsm / fsm_cm) and a bit-exact model
of the kernel's lane walk (decode_common.cuh decode_lane_fsm).

CPU only.  Pins:
  * the state machine parses any bit string exactly as the canonical code
    does (huffman.cpp:131-157 words, i.e. the reference's decode_one chain on
    a complete code, lut.hpp:43-49), completion masks included;
  * it is offered exactly for complete codes whose words are all >= 2 bits;
  * the lane model -- pre-shift by the first window's gap, 2-byte pairs, the
    clipped tail bytes at the next window's gap -- returns, for every lane of
    encoder-written streams, the symbols the reference's per-window walks
    emit (count_phase / emit_phase, codec.cpp:133-190, oracle-checked).
"""
import numpy as np
import pytest

from paper_2510_02676_b200 import codec

from test_tables import length_sets


def canonical(lengths):
    """(length, word) -> symbol for the canonical code (huffman.cpp:131-157)."""
    code, words = 0, {}
    prev = 0
    for L in range(1, 17):
        for s in range(16):
            if lengths[s] == L:
                code <<= L - prev
                prev = L
                words[(L, code)] = s
                code += 1
    return words


def parse_bits(bits, words):
    """Sequential prefix-code parse: [(symbol, end_bit)] of the words completed."""
    out, l, v = [], 0, 0
    for i, b in enumerate(bits):
        l += 1
        v = (v << 1) | int(b)
        if (l, v) in words:
            out.append((words[(l, v)], i))
            l, v = 0, 0
    return out


def is_complete(lengths):
    return sum(2.0 ** -int(L) for L in lengths if L) == 1.0


@pytest.mark.parametrize("case", range(46))
def test_fsm_parses_like_the_code(case):
    lengths = length_sets()[case]
    fsm, cm, ok = codec.fsm_tables(lengths)
    present = [L for L in lengths if L]
    want_ok = len(present) >= 2 and min(present) >= 2 and is_complete(lengths)
    assert ok == want_ok
    if not ok:
        return
    words = canonical(lengths)
    rng = np.random.default_rng(case)
    for _ in range(20):
        nbytes = int(rng.integers(1, 60))
        data = rng.integers(0, 256, nbytes, dtype=np.uint8)
        bits = np.unpackbits(data)
        want = parse_bits(bits, words)
        got, st = [], 0
        for j, byte in enumerate(data):
            e = int(fsm[st, byte])
            n = (e & 31) // 4
            assert (e >> 5) & 7 == 0 and n <= 4
            ends = [i for i in range(8) if (int(cm[st, byte]) >> i) & 1]
            assert len(ends) == n
            for k in range(n):
                got.append(((e >> (16 + 4 * k)) & 15, 8 * j + ends[k]))
            assert e >> (16 + 4 * n) == 0  # no stray symbol bits (the sink ORs them in)
            st = (e >> 8) & 0xFF
        assert got == want


def lane_model(fsm, cm, lane_bytes, gap0, gnext, LW=8):
    """decode_lane_fsm, step for step (returns the lane's symbols)."""
    NB, NS = 8 * LW, 2 * LW + 1
    bits = np.unpackbits(np.frombuffer(lane_bytes, np.uint8))
    sbits = np.zeros(32 * NS, np.uint8)
    avail = bits[gap0: gap0 + 32 * NS]
    sbits[:avail.size] = avail
    sbytes = np.packbits(sbits)
    Lp = 64 * LW + gnext - gap0
    Bp, rmask = Lp >> 3, (1 << (Lp & 7)) - 1
    e, syms = 0, []
    for j in range(NB + 2):
        idx = (((e >> 8) & 0xFF), int(sbytes[j]))
        ej = int(fsm[idx])
        if j >= NB - 2 and j >= Bp:
            lm = rmask if j == Bp else 0
            k4 = 4 * bin(int(cm[idx]) & lm).count("1")
            ej = (ej & ((0x10000 << k4) - 0x10000) & 0xFFFFFFFF) | k4
        n = (ej & 31) // 4
        syms += [(ej >> (16 + 4 * k)) & 15 for k in range(n)]
        e = ej
    return syms


@pytest.mark.parametrize("n,T,gamma,seed", [(20_000, 256, 0.05, 1), (9_000, 8, 0.05, 2), (15_000, 64, 0.3, 3),
                                            (12_000, 32, 1.0, 4), (8_000, 128, 0.01, 5)])
def test_lane_model_equals_reference_windows(orc, n, T, gamma, seed):
    x = codec.synth(1.8, gamma, n, seed)
    t = codec.encode_tensor(x, T)
    fsm, cm, ok = codec.fsm_tables(t.lengths)
    if not ok:
        pytest.skip("code has a 1-bit word (no byte-step decoder)")
    enc = np.asarray(t.encoded)
    n_win = (enc.size - 2) // 8
    padded = np.concatenate([enc, np.zeros(64, np.uint8)])
    # reference per-window counts (count_phase, codec.cpp:133-161)
    counts = np.array([orc.count_phase(padded[8 * w: 8 * w + 10], t.gap_at(w), t.lengths) for w in range(n_win)])
    first = np.concatenate([[0], np.cumsum(counts)])
    expo = (x >> 3) & 15
    checked = 0
    for lane in range((n_win - 1) // 8):
        w0 = 8 * lane
        # the window after the lane must own a word (past the last symbol the
        # encoder leaves gap 0, the upload check rejects the tile, and the
        # kernel takes the window-by-window walk)
        if first[w0 + 9] >= n:
            break
        got = lane_model(fsm, cm, padded[8 * w0: 8 * w0 + 72].tobytes(), t.gap_at(w0), t.gap_at(w0 + 8))
        want_n = int(first[w0 + 8] - first[w0])
        assert len(got) == want_n, (lane, len(got), want_n)
        lo, hi = int(first[w0]), min(int(first[w0 + 8]), n)
        assert got[: hi - lo] == list(expo[lo:hi]), lane
        checked += 1
    assert checked > 10

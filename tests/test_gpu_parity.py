"""B200 decode parity: every decode goes through the C ABI on the GPU and is
compared bit-for-bit with the CPU oracle (oracle/ecf8_oracle.c) and the
original bytes.  Cases follow the reference suite
(/root/reference/proj/tests/test_codec.cpp, acceptance.cpp).
"""
import numpy as np
import pytest

from paper_2510_02676_b200 import codec

from _oracle import tensor_dict

pytestmark = pytest.mark.gpu

TS = (1, 2, 32, 256, 512, 1024)
LADDER = np.array([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 16, 16], np.uint8)


def check(orc, x, T, lengths=None):
    t = codec.encode_tensor(x, T, lengths)
    got = codec.decode_parallel(t)
    want = orc.decode_parallel(tensor_dict(t))
    assert np.array_equal(want, x)
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)
        raise AssertionError(f"T={T} n={x.size}: {bad.size} mismatches, first at {bad[0]}")


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 63, 64, 65, 100, 513, 4096, 100000])
def test_sizes_distributions_widths(orc, n):
    # test_codec.cpp:307-332
    rng = np.random.default_rng(41 + n)
    for dist in range(3):
        if dist == 0:
            x = rng.integers(0, 256, n, dtype=np.uint8)
        elif dist == 1:
            x = np.where(rng.random(n) < 0.9, 0x38, rng.integers(0, 256, n)).astype(np.uint8)
        else:
            x = np.full(n, 0xB8, np.uint8)
        for T in TS:
            check(orc, x, T)


def test_empty_tensor():
    t = codec.encode_tensor(np.zeros(0, np.uint8), 256)
    assert codec.decode_parallel(t).size == 0


def test_gap15_straddle(orc):
    # test_codec.cpp:282-305
    sym = np.array([0] * 63 + [15, 14] + [0] * 200, np.uint8)
    i = np.arange(sym.size)
    x = ((sym << 3) | ((i % 16) << 4 & 0x80) | (i % 8)).astype(np.uint8)
    for T in TS:
        check(orc, x, T, LADDER)


def test_all_256_bytes(orc):
    x = (np.arange(100000) & 0xFF).astype(np.uint8)
    for T in TS:
        check(orc, x, T)


def test_alpha_stable_config1(orc):
    # config 1: 4096 x 4096 E4M3, alpha 1.8, gamma 0.05, seed 1, T=256
    x = codec.synth(1.8, 0.05, 4096 * 4096, 1)
    t = codec.encode_tensor(x, 256)
    got = codec.decode_parallel(t)
    assert np.array_equal(got, x)
    assert np.array_equal(orc.decode_parallel(tensor_dict(t), nthreads=0), got)


@pytest.mark.parametrize("gamma", [0.02, 0.05, 1.0])
def test_alpha_stable_widths(orc, gamma):
    x = codec.synth(1.8, gamma, 300001, 7)
    for T in TS:
        check(orc, x, T)


def test_e5m2_bytes(orc):
    x = codec.synth(1.8, 0.05, 200000, 5, fmt="e5m2")
    for T in (32, 256, 1024):
        check(orc, x, T)


def test_crafted_incomplete_codes(orc):
    """Kraft < 1 codes (accepted by parse_container): fallback symbols."""
    from test_tables import random_lengths

    rng = np.random.default_rng(77)
    for _ in range(30):
        l = random_lengths(rng)
        present = np.flatnonzero(l)
        sym = rng.choice(present, 5000).astype(np.uint8)
        x = ((sym << 3) | rng.integers(0, 256, sym.size).astype(np.uint8) & 0x87).astype(np.uint8)
        check(orc, x, int(rng.choice(TS)), l)


def test_decode_block_matches_oracle(orc):
    # test_codec.cpp:334-367: any block, any (permuted) order, same bytes
    rng = np.random.default_rng(43)
    x = rng.integers(0, 256, 40000, dtype=np.uint8)
    for T in (2, 32, 256, 1024):
        t = codec.encode_tensor(x, T)
        out = np.zeros(x.size, np.uint8)
        for b in reversed(range(t.n_blocks)):
            codec.decode_block(t, b, out)
        assert np.array_equal(out, x)


def test_count_phase_known_answers():
    # test_codec.cpp:206-233 on the device count routine
    l = np.zeros(16, np.uint8)
    l[5] = 1
    assert codec.count_phase(np.zeros(10, np.uint8), 0, l) == 64
    l = np.zeros(16, np.uint8)
    l[0], l[15] = 1, 16
    w = np.zeros(10, np.uint8)
    w[1] = 1
    assert codec.count_phase(w, 15, l) == 34
    assert codec.count_phase(np.zeros(10, np.uint8), 15, l) == 49
    assert codec.count_phase(np.zeros(10, np.uint8), 0, l) == 64


def test_count_phase_random_windows(orc):
    from test_tables import length_sets

    rng = np.random.default_rng(5)
    sets = length_sets()
    for k in range(300):
        l = sets[k % len(sets)]
        w = rng.integers(0, 256, 10, dtype=np.uint8)
        g = int(rng.integers(0, 16))
        assert codec.count_phase(w, g, l) == orc.count_phase(w, g, l)


def test_container_streaming_roundtrip():
    # test_container.cpp:227-263 + acceptance criterion 8
    rng = np.random.default_rng(56)
    tensors, largest = [], 0
    for i in range(100):
        n = int(rng.integers(0, 2000))
        largest = max(largest, n)
        tensors.append((f"t{i}", [n], rng.integers(0, 256, n, dtype=np.uint8)))
    raw = codec.raw_file(tensors)
    blob = codec.compress_raw(raw, 256)
    out, allocs, cap = codec.decompress(blob)
    assert out == raw and allocs == 1 and cap == largest


def test_invalid_lengths_rejected_by_device_path():
    t = codec.encode_tensor(np.arange(64, dtype=np.uint8), 32)
    bad = t.copy()
    bad.lengths[:] = 1
    from paper_2510_02676_b200._lib import InvalidArgument

    with pytest.raises(InvalidArgument, match="invalid length vector"):
        codec.decode_parallel(bad)


@pytest.mark.parametrize("T", [8, 64, 256, 1024])
def test_block_range_beyond_window_capacity_rejected(T):
    # outpos steps up to T * 64 pass the reference's container check, but with
    # Lmin >= 2 a block's windows hold at most T * 32 code words; such a block
    # (never encoder output) must be rejected, not decoded past the kernels'
    # Lmin-sized slots and staging tiles
    from paper_2510_02676_b200._lib import InvalidArgument

    x = codec.synth(1.8, 0.05, 40 * T * 32, 11)
    t = codec.encode_tensor(x, T)
    assert int(np.flatnonzero(t.lengths).size) and min(l for l in t.lengths if l) >= 2
    bad = t.copy()
    op = bad.outpos
    assert len(op) >= 4
    op[1] = op[0] + 1  # block 1 now spans (nearly) two blocks' symbols
    assert op[2] - op[1] > T * 32 and op[2] - op[1] <= T * 64
    with pytest.raises(InvalidArgument, match="inconsistent block offsets"):
        codec.decode_parallel(bad)
    import torch  # noqa: F401

    from paper_2510_02676_b200.device import DeviceTensor

    with pytest.raises(InvalidArgument, match="inconsistent block offsets"):
        DeviceTensor(bad)
    assert np.array_equal(codec.decode_parallel(t), x)


def test_decode_many_pipeline_across_tensors(orc):
    # mixed T / sizes / an empty tensor; the 12 M-element tensor spans several
    # 2 MB chunks, so chunk slots are reused within and across tensors
    specs = [(12_000_000, 256, 1), (0, 256, 2), (333, 1, 3), (70_001, 1, 4), (5_000_000, 32, 5),
             (100_000, 1024, 6), (4_096 * 1024, 2, 7), (9, 8, 8)]
    raws = [codec.synth(1.8, 0.05, n, seed) for n, _, seed in specs]
    ts = [codec.encode_tensor(x, T) for x, (_, T, _) in zip(raws, specs)]
    for _ in range(2):  # second pass reuses the warm slots
        got = codec.decode_many(ts)
        for g, x in zip(got, raws):
            assert np.array_equal(g, x)
    # the single-tensor call shares the pipeline
    assert np.array_equal(codec.decode_parallel(ts[0]), raws[0])


def test_decode_many_validates_each_tensor():
    from paper_2510_02676_b200._lib import InvalidArgument

    t = codec.encode_tensor(codec.synth(1.8, 0.05, 1000, 1), 256)
    with pytest.raises(InvalidArgument, match="output size mismatch"):
        codec.decode_many_into([t, t], [np.empty(1000, np.uint8), np.empty(999, np.uint8)])


@pytest.mark.parametrize("n,T,seed", [(5_000_000, 256, 1), (777_777, 64, 2), (123_457, 8, 3), (3_000_001, 128, 4)])
def test_device_path_continuous_walk(orc, n, T, seed):
    # encoder output: the upload gap check passes every tile, so the whole
    # tensor takes the continuous walk
    import torch

    from paper_2510_02676_b200.device import DeviceTensor

    x = codec.synth(1.8, 0.05, n, seed)
    t = codec.encode_tensor(x, T)
    d = DeviceTensor(t)
    # every tile places its lanes directly: the direct-only variant 7
    assert d.kernel_variant == 7
    ok, total = d.verified_tiles()
    assert total == -(-(len(t.outpos) - 1) * T // 256)
    # every tile but possibly the last: windows of the zero padding after the
    # final symbol need not end where the next (empty) window's gap says
    assert ok >= total - 1
    got = d.decode().cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(got, x)


def test_inconsistent_gaps_fall_back_to_reference_semantics(orc):
    # a parseable stream whose gap nibbles disagree with the code words: the
    # reference still decodes it window by window (codec.cpp:201-253); the
    # device path must detect it at upload and produce the same bytes.  Where
    # a corrupted block's windows count fewer symbols than outpos says, the
    # reference leaves that tail of the block to stale scratch contents
    # (codec.cpp:253 copies the whole staging range) -- undefined, so only
    # blocks whose counts cover them are compared.
    from paper_2510_02676_b200.device import DeviceTensor

    x = codec.synth(1.8, 0.05, 400_000, 9)
    t = codec.encode_tensor(x, 256).copy()
    g = np.asarray(t.gaps)
    for j in (37, 1000, 5001):  # windows 2j (high nibble) get a shifted gap
        g[j] = ((((g[j] >> 4) + 3) & 15) << 4) | (g[j] & 15)
    d = tensor_dict(t)
    want = orc.decode_parallel(d)  # the reference's parallel decoder on these gaps
    assert not np.array_equal(want, x)
    T, enc, op = 256, np.asarray(t.encoded), np.asarray(t.outpos)
    defined = np.ones(t.n_elem, bool)
    for b in range(len(op) - 1):
        cnt = sum(orc.count_phase(enc[8 * w:8 * w + 10], t.gap_at(w), d["lengths"]) for w in range(b * T, (b + 1) * T))
        if cnt < op[b + 1] - op[b]:
            defined[op[b]:op[b + 1]] = False
    dev = DeviceTensor(t)
    ok, total = dev.verified_tiles()
    # the upload check rejects the corrupted tiles (a window that starts an
    # 8-window lane is checked only against its successor: each lane runs
    # from its own first gap to its last window's recorded end)
    assert total - 4 <= ok <= total - 2
    got = dev.decode().cpu().numpy()
    assert defined.sum() > 0.9 * t.n_elem
    assert np.array_equal(got[defined], want[defined])
    assert np.array_equal(codec.decode_parallel(t)[defined], want[defined])


@pytest.mark.parametrize("T", [8, 64, 256])
def test_block_decoding_past_its_range_is_clamped(orc, T):
    # one block boundary moved down by one symbol (never encoder output):
    # block b decodes one word more than its range (the reference clamps it,
    # codec.cpp:239-251), block b + 1 one fewer (its last element is stale
    # scratch in the reference: undefined, not compared).  The upload check
    # must take such a tile off the direct-placement path, or block b's extra
    # word would land on block b + 1's first element.
    from paper_2510_02676_b200.device import DeviceTensor

    x = codec.synth(1.8, 0.05, 300_000, 21 + T)
    t = codec.encode_tensor(x, T).copy()
    op = t.outpos
    nb = len(op) - 1
    b = nb // 2
    op[b + 1] -= 1
    d = tensor_dict(t)
    want = orc.decode_parallel(d)
    defined = np.ones(t.n_elem, bool)
    defined[op[b + 2] - 1] = False
    assert not np.array_equal(want[defined], x[defined])
    dev = DeviceTensor(t)
    assert dev.kernel_variant == 4  # a tile off the direct path: the kernel with the fallback
    got = dev.decode().cpu().numpy()
    assert np.array_equal(got[defined], want[defined])
    assert np.array_equal(codec.decode_parallel(t)[defined], want[defined])


@pytest.mark.gpu
def test_batch_decode_in_cuda_graph():
    # the per-layer decode as a captured CUDA graph (programmatic dependent
    # launches inside the graph), replayed: bit-exact every time
    import torch

    from paper_2510_02676_b200.device import Batch, DeviceTensor

    xs = [codec.synth(1.8, 0.05, n, 60 + i) for i, n in enumerate((2_000_000, 750_001, 3_100_000))]
    ds = [DeviceTensor(codec.encode_tensor(x, 256)) for x in xs]
    outs = [torch.empty(x.size, dtype=torch.uint8, device="cuda") for x in xs]
    b = Batch(ds, outs)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        b.decode(s)  # warm-up outside the capture (lazy attribute setup)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        b.decode(s)
        b.decode(s)
    for _ in range(3):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        for o, x in zip(outs, xs):
            assert np.array_equal(o.cpu().numpy(), x)


def test_decompress_to_sink_matches_decompress():
    # decompress_streaming into a caller sink (ecf8_host_decompress_to): same
    # raw bytes, one buffer (pinned for the call), capacity = largest tensor
    rng = np.random.default_rng(57)
    tensors = [(f"t{i}", [n], codec.synth(1.8, 0.05, n, 70 + i)) for i, n in enumerate([5000, 0, 1_200_000, 77])]
    raw = codec.raw_file(tensors)
    blob = codec.compress_raw(raw, 256)
    parts = []
    allocs, cap = codec.decompress_to(blob, lambda mv: parts.append(bytes(mv)))
    assert b"".join(parts) == raw and allocs == 1 and cap == 1_200_000
    from paper_2510_02676_b200._lib import Ecf8Error

    def bad(mv):
        raise OSError("disk full")

    with pytest.raises(Ecf8Error, match="sink write failed"):
        codec.decompress_to(blob, bad)
    assert rng is not None


@pytest.mark.parametrize("T", [8, 32, 128, 256])
@pytest.mark.parametrize("n,fmt,gamma", [(3_000_001, "e5m2", 0.05), (777_777, "e5m2", 1.0), (500_000, "e4m3", 0.002),
                                         (1, "e5m2", 0.05), (4099, "e5m2", 0.05)])
def test_one_bit_codes_take_the_64bit_byte_steps(orc, T, n, fmt, gamma):
    # codes with a 1-bit word (E5M2 bytes through the reference format,
    # small-gamma E4M3): variant 6 when every tile passes the upload check
    from paper_2510_02676_b200.device import DeviceTensor

    x = codec.synth(1.8, gamma, n, 70 + T, fmt=fmt)
    t = codec.encode_tensor(x, T)
    lengths = [l for l in t.lengths if l]
    if len(lengths) < 2 or min(lengths) != 1:
        pytest.skip("no 1-bit word in this code")
    d = DeviceTensor(t)
    assert d.kernel_variant == 6
    got = d.decode().cpu().numpy()
    assert np.array_equal(got, x)
    assert np.array_equal(got, orc.decode_parallel(tensor_dict(t)))


def test_one_bit_code_with_corrupt_gaps_keeps_variant_5(orc):
    from paper_2510_02676_b200.device import DeviceTensor

    x = codec.synth(1.8, 0.05, 400_000, 77, fmt="e5m2")
    t = codec.encode_tensor(x, 256).copy()
    assert min(l for l in t.lengths if l) == 1
    g = np.asarray(t.gaps)
    g[333] = ((((g[333] >> 4) + 5) & 15) << 4) | (g[333] & 15)
    d = DeviceTensor(t)
    assert d.kernel_variant == 5
    want = orc.decode_parallel(tensor_dict(t))
    T, enc, op, dd = 256, np.asarray(t.encoded), np.asarray(t.outpos), tensor_dict(t)
    defined = np.ones(t.n_elem, bool)
    for b in range(len(op) - 1):
        cnt = sum(orc.count_phase(enc[8 * w:8 * w + 10], t.gap_at(w), dd["lengths"]) for w in range(b * T, (b + 1) * T))
        if cnt < op[b + 1] - op[b]:
            defined[op[b]:op[b + 1]] = False
    got = d.decode().cpu().numpy()
    assert np.array_equal(got[defined], want[defined])


def test_batch_mixes_variants_6_and_7(orc):
    import torch

    from paper_2510_02676_b200.device import Batch, DeviceTensor

    xs = [codec.synth(1.8, 0.05, 1_000_003, 81, fmt="e5m2"), codec.synth(1.8, 0.05, 2_000_000, 82),
          codec.synth(1.8, 0.05, 70_000, 83, fmt="e5m2")]
    ds = [DeviceTensor(codec.encode_tensor(x, 256)) for x in xs]
    assert sorted(d.kernel_variant for d in ds) == [6, 6, 7]
    outs = [torch.empty(x.size, dtype=torch.uint8, device="cuda") for x in xs]
    b = Batch(ds, outs)
    for _ in range(2):
        b.decode()
        torch.cuda.synchronize()
        for o, x in zip(outs, xs):
            assert np.array_equal(o.cpu().numpy(), x)


@pytest.mark.gpu
def test_batch_mixes_variants_4_and_7(orc):
    # one tensor with a tile off the direct path (a block boundary moved down
    # by one symbol, as in test_block_decoding_past_its_range_is_clamped)
    # between two encoder outputs: one launch per variant, every output exact
    import torch

    from paper_2510_02676_b200.device import Batch, DeviceTensor

    xs = [codec.synth(1.8, 0.05, 1_500_000, 91 + i) for i in range(3)]
    ts = [codec.encode_tensor(x, 256) for x in xs]
    t1 = ts[1].copy()
    op = t1.outpos
    b = (len(op) - 1) // 2
    op[b + 1] -= 1
    ts[1] = t1
    want1 = orc.decode_parallel(tensor_dict(t1))
    defined = np.ones(t1.n_elem, bool)
    defined[op[b + 2] - 1] = False
    ds = [DeviceTensor(t) for t in ts]
    assert [d.kernel_variant for d in ds] == [7, 4, 7]
    outs = [torch.empty(x.size, dtype=torch.uint8, device="cuda") for x in xs]
    bt = Batch(ds, outs)
    for _ in range(2):
        bt.decode()
        torch.cuda.synchronize()
        assert np.array_equal(outs[0].cpu().numpy(), xs[0])
        assert np.array_equal(outs[1].cpu().numpy()[defined], want1[defined])
        assert np.array_equal(outs[2].cpu().numpy(), xs[2])

"""Python mirror of the ECF8 API (reference names, reference error behaviour).

Thin wrappers over the C ABI; every decode that is not explicitly the
reference's sequential oracle API runs on the B200.  Arrays are numpy uint8.

Reference map (/root/reference/proj):
  build_code            src/huffman.cpp:111-129
  build_lut             src/lut.cpp:47-97
  encode_tensor         src/codec.cpp:100-109
  decode_reference      src/codec.cpp:125-131   (host oracle API)
  count_phase           src/codec.cpp:133-161   (device)
  decode_block          src/codec.cpp:201-254   (device)
  decode_parallel(_into) src/codec.cpp:256-279  (device, the hot path)
  compress_raw          src/container.cpp:291-322 (+ serialize / parse_raw)
  parse_container       src/container.cpp:182-250
  decompress            src/container.cpp:324-352 (device decode)
  synth                 src/container.cpp:482-495 (multi-threaded, identical bytes)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import Sections, check, lib

FAST_BITS = 12


def _ptr(a: np.ndarray | None) -> int | None:
    if a is None:
        return None
    return a.ctypes.data if a.size else None


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


# ------------------------------------------------------------------ codes


def build_code(counts) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    if c.shape != (16,):
        raise ValueError("histogram must have 16 bins")
    out = np.zeros(16, np.uint8)
    check(lib.ecf8_host_build_code(_ptr(c), _ptr(out)))
    return out


def build_lut(lengths) -> tuple[np.ndarray, int]:
    l = _u8(lengths)
    buf = np.zeros(18 * 256, np.uint8)
    n = C.c_uint32()
    check(lib.ecf8_host_build_lut(_ptr(l), _ptr(buf), C.byref(n)))
    return buf[: 256 * n.value].copy(), n.value


def device_tables(lengths) -> tuple[np.ndarray, np.ndarray, np.ndarray, int, int]:
    """(fast u32, start masks u16, cascade bytes, n_luts, fast_bits) as uploaded to HBM."""
    l = _u8(lengths)
    fast = np.zeros(1 << 16, np.uint32)
    smask = np.zeros(1 << 16, np.uint16)
    casc = np.zeros(18 * 256, np.uint8)
    n = C.c_uint32()
    fb = C.c_uint32()
    check(lib.ecf8_host_device_tables(_ptr(l), _ptr(fast), _ptr(smask), _ptr(casc), C.byref(n), C.byref(fb)))
    k = 1 << fb.value
    return fast[:k].copy(), smask[:k].copy(), casc[: 256 * n.value].copy(), n.value, fb.value


def fsm_tables(lengths) -> tuple[np.ndarray, np.ndarray, bool]:
    """(fsm u32 [16, 256], completion masks u8 [16, 256], available) -- the
    byte-step decoder the B200 kernel stages for verified tiles."""
    l = _u8(lengths)
    fsm = np.zeros(16 * 256, np.uint32)
    cm = np.zeros(16 * 256, np.uint8)
    ok = C.c_int()
    check(lib.ecf8_host_fsm_tables(_ptr(l), _ptr(fsm), _ptr(cm), C.byref(ok)))
    return fsm.reshape(16, 256), cm.reshape(16, 256), bool(ok.value)


# --------------------------------------------------------------- tensors


@dataclass
class EncodedTensor:
    """Container sections of one tensor (numpy views kept alive here)."""

    n_elem: int
    threads_per_block: int
    lengths: np.ndarray
    encoded: np.ndarray
    gaps: np.ndarray
    outpos: np.ndarray
    packed: np.ndarray
    _owner: object = None

    @property
    def n_blocks(self) -> int:
        return len(self.outpos) - 1

    def gap_at(self, t: int) -> int:
        return (int(self.gaps[t >> 1]) >> (0 if t & 1 else 4)) & 15

    def sections(self) -> Sections:
        s = Sections()
        s.n_elem = self.n_elem
        s.threads_per_block = self.threads_per_block
        for i in range(16):
            s.lengths[i] = int(self.lengths[i])
        s.encoded, s.encoded_len = _ptr(self.encoded), self.encoded.size
        s.gaps, s.gaps_len = _ptr(self.gaps), self.gaps.size
        s.outpos, s.n_outpos = _ptr(self.outpos), self.outpos.size
        s.packed, s.packed_len = _ptr(self.packed), self.packed.size
        return s

    def compressed_bytes(self) -> int:
        """Bytes the decoder reads (container sections, metadata included)."""
        return self.encoded.size + self.gaps.size + 8 * self.outpos.size + self.packed.size

    def algorithmic_bytes(self) -> int:
        return self.compressed_bytes() + self.n_elem

    def copy(self) -> "EncodedTensor":
        return EncodedTensor(
            self.n_elem,
            self.threads_per_block,
            self.lengths.copy(),
            self.encoded.copy(),
            self.gaps.copy(),
            self.outpos.copy(),
            self.packed.copy(),
        )


def _view(ptr: int | None, n: int, dtype, owner) -> np.ndarray:
    """Zero-copy numpy view of library memory that keeps `owner` alive."""
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    ct = C.c_uint64 if dtype == np.uint64 else C.c_uint8
    arr = (ct * n).from_address(ptr)
    arr._owner = owner  # numpy -> memoryview -> ctypes array -> owner
    return np.ctypeslib.as_array(arr)


class _HostTensor:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        if self.handle and lib is not None:  # lib is None during interpreter teardown
            lib.ecf8_host_tensor_free(self.handle)
            self.handle = None


def _from_handle(h) -> EncodedTensor:
    owner = _HostTensor(h)
    s = Sections()
    check(lib.ecf8_host_tensor_sections(h, C.byref(s)))
    return _from_sections(s, owner)


def _from_sections(s: Sections, owner) -> EncodedTensor:
    return EncodedTensor(
        n_elem=s.n_elem,
        threads_per_block=s.threads_per_block,
        lengths=np.array(list(s.lengths), np.uint8),
        encoded=_view(s.encoded, s.encoded_len, np.uint8, owner),
        gaps=_view(s.gaps, s.gaps_len, np.uint8, owner),
        outpos=_view(s.outpos, s.n_outpos, np.uint64, owner),
        packed=_view(s.packed, s.packed_len, np.uint8, owner),
        _owner=owner,
    )


def encode_tensor(fp8, threads_per_block: int = 256, lengths=None) -> EncodedTensor:
    """Host encoder.  lengths=None: the tensor's own package-merge code."""
    a = _u8(fp8).reshape(-1)
    l = None if lengths is None else _u8(lengths)
    h = C.c_void_p()
    check(lib.ecf8_host_encode(_ptr(a), a.size, threads_per_block, _ptr(l), C.byref(h)))
    return _from_handle(h)


def make_stats(fp8, threads_per_block: int = 256, name_len: int = 1, rank: int = 1) -> dict:
    """make_stats (container.cpp:386-413) of one raw tensor: entropy, code
    length, projected and actual savings (name_len / rank: its container
    overhead)."""
    from ._lib import EntropyReport

    a = _u8(fp8).reshape(-1)
    r = EntropyReport()
    check(lib.ecf8_host_make_stats(_ptr(a), a.size, threads_per_block, name_len, rank, C.byref(r)))
    return r.as_dict()


def encode_many(arrays, threads_per_block: int = 256, nthreads: int = 0) -> list[EncodedTensor]:
    arrs = [_u8(a).reshape(-1) for a in arrays]
    n = len(arrs)
    ptrs = (C.c_void_p * n)(*[_ptr(a) for a in arrs])
    sizes = (C.c_uint64 * n)(*[a.size for a in arrs])
    outs = (C.c_void_p * n)()
    check(lib.ecf8_host_encode_many(ptrs, sizes, n, threads_per_block, outs, nthreads))
    return [_from_handle(C.c_void_p(outs[i])) for i in range(n)]


def decode_reference(t: EncodedTensor) -> np.ndarray:
    out = np.empty(t.n_elem, np.uint8)
    s = t.sections()
    check(lib.ecf8_host_decode_reference(C.byref(s), _ptr(out), out.size))
    return out


def decode_parallel_into(t: EncodedTensor, out: np.ndarray) -> None:
    """The drop-in hot path (host buffers): decode on the B200."""
    if out.dtype != np.uint8 or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous uint8 array")
    s = t.sections()
    check(lib.ecf8_decode_host(C.byref(s), _ptr(out), out.size))


def decode_parallel(t: EncodedTensor) -> np.ndarray:
    out = np.empty(t.n_elem, np.uint8)
    decode_parallel_into(t, out)
    return out


def decode_many_into(ts: list[EncodedTensor], outs: list[np.ndarray]) -> None:
    """decode_parallel_into for a list of tensors in one pipelined call
    (ecf8_decode_host_many): host -> B200 -> host, overlapped across tensors."""
    if len(ts) != len(outs):
        raise ValueError("one output per tensor")
    for o in outs:
        if o.dtype != np.uint8 or not o.flags.c_contiguous:
            raise ValueError("out must be a contiguous uint8 array")
    n = len(ts)
    secs = [t.sections() for t in ts]
    sp = (C.POINTER(Sections) * n)(*[C.pointer(s) for s in secs])
    op = (C.c_void_p * n)(*[_ptr(o) for o in outs])
    lens = (C.c_uint64 * n)(*[o.size for o in outs])
    check(lib.ecf8_decode_host_many(sp, op, lens, n))


def decode_many(ts: list[EncodedTensor]) -> list[np.ndarray]:
    outs = [np.empty(t.n_elem, np.uint8) for t in ts]
    decode_many_into(ts, outs)
    return outs


def decode_block(t: EncodedTensor, block: int, out: np.ndarray) -> None:
    s = t.sections()
    check(lib.ecf8_decode_block_host(C.byref(s), block, _ptr(out), out.size))


def count_phase(window10, gap: int, lengths) -> int:
    w = _u8(window10)
    if w.size != 10:
        raise ValueError("window10 must hold 10 bytes")
    l = _u8(lengths)
    c = C.c_uint32()
    check(lib.ecf8_count_window(_ptr(w), gap, _ptr(l), C.byref(c)))
    return c.value


# ------------------------------------------------------------- container


def _take_malloc(p: C.c_void_p, n: int) -> bytes:
    try:
        return C.string_at(p.value, n) if n else b""
    finally:
        lib.ecf8_host_free(p)


def compress_raw(raw: bytes, threads_per_block: int = 256) -> bytes:
    buf = np.frombuffer(raw, np.uint8)
    p, n = C.c_void_p(), C.c_size_t()
    check(lib.ecf8_host_compress_raw(_ptr(buf), buf.size, threads_per_block, C.byref(p), C.byref(n)))
    return _take_malloc(p, n.value)


class Ecf8File:
    """Parsed container (parse_container); tensors are zero-copy views."""

    def __init__(self, data: bytes):
        buf = np.frombuffer(data, np.uint8)
        h = C.c_void_p()
        check(lib.ecf8_host_parse(_ptr(buf), buf.size, C.byref(h)))
        self._h = h
        self.tensors: list[tuple[str, EncodedTensor]] = []
        self.shapes: list[list[int]] = []
        for i in range(lib.ecf8_host_file_count(h)):
            s, name = Sections(), C.c_char_p()
            check(lib.ecf8_host_file_tensor(h, i, C.byref(s), C.byref(name)))
            self.tensors.append((name.value.decode("utf-8", "replace"), _from_sections(s, self)))
            dims, rank = (C.c_uint64 * 255)(), C.c_int()
            check(lib.ecf8_host_file_shape(h, i, dims, 255, C.byref(rank)))
            self.shapes.append([int(dims[j]) for j in range(rank.value)])

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ecf8_host_file_free(self._h)
            self._h = None


def parse_container(data: bytes) -> Ecf8File:
    return Ecf8File(data)


WRITE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t)


def decompress_to(data: bytes, write) -> tuple[int, int]:
    """decompress_streaming into a sink: write(memoryview) gets the raw file
    in order (ecf8_host_decompress_to).  Returns (buffer_allocations, capacity)."""
    buf = np.frombuffer(data, np.uint8)

    def _w(_ctx, p, n):
        try:
            write(memoryview((C.c_uint8 * n).from_address(p)).cast("B"))
            return 0
        except Exception:  # surfaced as ECF8_EIO "sink write failed"
            return 1

    fn = WRITE_FN(_w)
    a, cap = C.c_uint64(), C.c_uint64()
    check(lib.ecf8_host_decompress_to(_ptr(buf), buf.size, C.cast(fn, C.c_void_p), None, C.byref(a), C.byref(cap)))
    return a.value, cap.value


def decompress(data: bytes) -> tuple[bytes, int, int]:
    """decompress_streaming: (raw file bytes, buffer_allocations, capacity)."""
    buf = np.frombuffer(data, np.uint8)
    p, n = C.c_void_p(), C.c_size_t()
    a, cap = C.c_uint64(), C.c_uint64()
    check(lib.ecf8_host_decompress(_ptr(buf), buf.size, C.byref(p), C.byref(n), C.byref(a), C.byref(cap)))
    return _take_malloc(p, n.value), a.value, cap.value


def synth(alpha: float, gamma: float, n: int, seed: int, fmt: str = "e4m3", nthreads: int = 0) -> np.ndarray:
    """synth_raw data: alpha-stable draws -> RNE saturating FP8 bytes."""
    out = np.empty(n, np.uint8)
    f = {"e4m3": 0, "e5m2": 1}[fmt]
    check(lib.ecf8_host_synth(alpha, gamma, n, seed, f, _ptr(out), nthreads))
    return out


def raw_file(tensors: list[tuple[str, list[int], np.ndarray]]) -> bytes:
    """Serialize an FP8R raw file (container.cpp:128-140) from (name, dims, data)."""
    parts = [b"FP8R", (1).to_bytes(4, "little"), len(tensors).to_bytes(4, "little")]
    for name, dims, data in tensors:
        nb = name.encode()
        parts += [len(nb).to_bytes(2, "little"), nb, bytes([len(dims)])]
        parts += [int(d).to_bytes(8, "little") for d in dims]
        parts.append(_u8(data).tobytes())
    return b"".join(parts)

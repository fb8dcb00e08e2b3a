"""Native E5M2 variant of ECF8 (include/ecf8_e5m2.h).

The reference is E4M3-only.  This variant
entropy-codes the full 5-bit E5M2 exponent (32 symbols) with the reference's
stream, block and code rules, and stores sign + 2 mantissa bits as three bit
planes (3 bits per element instead of the byte split's 4).  Encoding and the
EC5M container run on the host (C++); decoding runs on the B200 only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import E5Sections, check, lib
from .codec import _ptr, _take_malloc, _u8, _view as _arr


def build_code(counts) -> np.ndarray:
    """Code lengths (32 symbols, <= 16 bits) by package-merge with the reference's tie rules."""
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    if c.size != 32:
        raise ValueError("expected 32 counts")
    out = np.zeros(32, np.uint8)
    check(lib.ecf8_e5_build_code(_ptr(c), _ptr(out)))
    return out


class E5Tensor:
    """One encoded tensor: n_elem, T, lengths[32], encoded, gaps, outpos, raw."""

    def __init__(self, n_elem, threads_per_block, lengths, encoded, gaps, outpos, raw, owner=None):
        self.n_elem = int(n_elem)
        self.threads_per_block = int(threads_per_block)
        self.lengths = np.asarray(lengths, np.uint8)
        self.encoded, self.gaps, self.outpos, self.raw = encoded, gaps, outpos, raw
        self._owner = owner

    @classmethod
    def _from_sections(cls, s: E5Sections, owner) -> "E5Tensor":
        return cls(s.n_elem, s.threads_per_block, np.array(s.lengths[:], np.uint8),
                   _arr(s.encoded, s.encoded_len, np.uint8, owner), _arr(s.gaps, s.gaps_len, np.uint8, owner),
                   _arr(s.outpos, s.n_outpos, np.uint64, owner), _arr(s.raw, s.raw_len, np.uint8, owner), owner)

    def sections(self) -> E5Sections:
        s = E5Sections()
        s.n_elem = self.n_elem
        s.threads_per_block = self.threads_per_block
        s.lengths[:] = [int(v) for v in self.lengths]
        for f in ("encoded", "gaps", "outpos", "raw"):
            a = np.ascontiguousarray(getattr(self, f))
            setattr(self, "_k_" + f, a)
            setattr(s, f, _ptr(a) if a.size else None)
        s.encoded_len, s.gaps_len, s.n_outpos, s.raw_len = (self.encoded.size, self.gaps.size, self.outpos.size,
                                                            self.raw.size)
        return s

    def compressed_bytes(self) -> int:
        return int(self.encoded.size + self.gaps.size + 8 * self.outpos.size + self.raw.size)

    def algorithmic_bytes(self) -> int:
        """Decode traffic: compressed sections read + one output byte per element."""
        return self.compressed_bytes() + self.n_elem


class _Handle:
    def __init__(self, h, free):
        self.h, self._free = h, free

    def __del__(self):
        if self.h:
            self._free(self.h)
            self.h = None


def encode(e5m2, threads_per_block: int = 256) -> E5Tensor:
    x = _u8(e5m2)
    h = C.c_void_p()
    check(lib.ecf8_e5_encode(_ptr(x), x.size, threads_per_block, C.byref(h)))
    owner = _Handle(h, lib.ecf8_e5_tensor_free)
    s = E5Sections()
    check(lib.ecf8_e5_tensor_sections(h, C.byref(s)))
    return E5Tensor._from_sections(s, owner)


def decode(t: E5Tensor) -> np.ndarray:
    """Host spans through the B200 (ecf8_e5_decode_host)."""
    out = np.empty(t.n_elem, np.uint8)
    s = t.sections()
    check(lib.ecf8_e5_decode_host(C.byref(s), _ptr(out), out.size))
    return out


class E5DeviceTensor:
    """HBM-resident E5 tensor (ecf8_e5_upload); decode() into a torch CUDA buffer."""

    def __init__(self, t: E5Tensor):
        s = t.sections()
        h = C.c_void_p()
        check(lib.ecf8_e5_upload(C.byref(s), C.byref(h)))
        self._h = _Handle(h, lib.ecf8_e5_free)
        self.n_elem = t.n_elem
        self.algorithmic_bytes = t.algorithmic_bytes()
        self.byte_steps = bool(lib.ecf8_e5_dev_byte_steps(self._h.h))

    def decode_into(self, out, stream=None) -> None:
        import torch

        if out.dtype != torch.uint8 or not out.is_cuda or out.numel() < self.n_elem or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous CUDA uint8 tensor of >= {self.n_elem} elements")
        st = stream if stream is not None else torch.cuda.current_stream()
        check(lib.ecf8_e5_decode_device(self._h.h, C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)))

    def decode(self, stream=None):
        import torch

        out = torch.empty(max(self.n_elem, 16), dtype=torch.uint8, device="cuda")[: self.n_elem]
        self.decode_into(out, stream)
        return out


def compress_raw(raw: bytes, threads_per_block: int = 256) -> bytes:
    """FP8R raw file of E5M2 tensors -> EC5M container."""
    buf = np.frombuffer(raw, np.uint8)
    p, n = C.c_void_p(), C.c_size_t()
    check(lib.ecf8_e5_compress_raw(_ptr(buf), buf.size, threads_per_block, C.byref(p), C.byref(n)))
    return _take_malloc(p, n.value)


class E5File:
    """Parsed EC5M container; tensors are zero-copy views."""

    def __init__(self, data: bytes):
        buf = np.frombuffer(data, np.uint8)
        h = C.c_void_p()
        check(lib.ecf8_e5_parse(_ptr(buf), buf.size, C.byref(h)))
        self._buf = buf
        self._h = _Handle(h, lib.ecf8_e5_file_free)

    def __len__(self) -> int:
        return int(lib.ecf8_e5_file_count(self._h.h))

    def tensor(self, i: int) -> tuple[str, list[int], E5Tensor]:
        s = E5Sections()
        name = C.c_char_p()
        check(lib.ecf8_e5_file_tensor(self._h.h, i, C.byref(s), C.byref(name)))
        dims = (C.c_uint64 * 255)()
        rank = C.c_int()
        check(lib.ecf8_e5_file_shape(self._h.h, i, dims, 255, C.byref(rank)))
        return name.value.decode(), [int(dims[k]) for k in range(rank.value)], E5Tensor._from_sections(s, self)


def decompress(data: bytes) -> bytes:
    """EC5M container -> FP8R raw file (every tensor decoded on the B200)."""
    buf = np.frombuffer(data, np.uint8)
    p, n = C.c_void_p(), C.c_size_t()
    check(lib.ecf8_e5_decompress(_ptr(buf), buf.size, C.byref(p), C.byref(n)))
    return _take_malloc(p, n.value)

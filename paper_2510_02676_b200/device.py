"""Device-resident ECF8 tensors driven from PyTorch streams.

PyTorch is plumbing here: it provides device memory for outputs, the CUDA
stream handle and CUDA events.  The decode itself is the sm_100a kernel in
libecf8_b200.so, reached through the C ABI (include/ecf8_cuda.h).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from ._lib import Sections, check, lib
from .codec import EncodedTensor, build_code


def _fp8_bytes(x: torch.Tensor) -> torch.Tensor:
    if not x.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if x.dtype in (torch.float8_e4m3fn, torch.float8_e5m2):
        x = x.view(torch.uint8)
    if x.dtype != torch.uint8:
        raise ValueError("expected FP8 or uint8 bytes")
    return x.contiguous().reshape(-1)


def exponent_histogram(x: torch.Tensor, stream: torch.cuda.Stream | None = None) -> np.ndarray:
    """ecf8_exponent_histogram: counts of the 16 exponent-field values
    (ExponentHistogram::of_bytes, the first step of make_stats) on the GPU."""
    x = _fp8_bytes(x)
    counts = np.zeros(16, np.uint64)
    check(lib.ecf8_exponent_histogram(C.c_void_p(x.data_ptr() if x.numel() else None), x.numel(),
                                      counts.ctypes.data_as(C.POINTER(C.c_uint64)), _stream_ptr(stream)))
    return counts


def make_stats_device(x: torch.Tensor, threads_per_block: int = 256, name_len: int = 1, rank: int = 1,
                      stream: torch.cuda.Stream | None = None) -> dict:
    """ecf8_make_stats_device: make_stats (container.cpp:386-413) with the
    histogram and the encode on the GPU; same numbers as codec.make_stats."""
    from ._lib import EntropyReport

    x = _fp8_bytes(x)
    r = EntropyReport()
    check(lib.ecf8_make_stats_device(C.c_void_p(x.data_ptr() if x.numel() else None), x.numel(), threads_per_block,
                                     name_len, rank, _stream_ptr(stream), C.byref(r)))
    return r.as_dict()


def _stream_ptr(stream: torch.cuda.Stream | None) -> int | None:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream or None


class DeviceTensor:
    """ecf8_tensor_upload: container sections + decode tables in HBM."""

    def __init__(self, t: EncodedTensor, stream: torch.cuda.Stream | None = None):
        self._sections = t.sections()
        self._src = t  # keep host arrays alive until the async copy completes
        h = C.c_void_p()
        check(lib.ecf8_tensor_upload(C.byref(self._sections), _stream_ptr(stream), C.byref(h)))
        self._adopt(h)

    def _adopt(self, h: C.c_void_p) -> None:
        self.handle = h
        self.n_elem = int(lib.ecf8_tensor_n_elem(h))
        self.algorithmic_bytes = int(lib.ecf8_tensor_algorithmic_bytes(h))
        self.device_bytes = int(lib.ecf8_tensor_device_bytes(h))
        self.kernel_variant = int(lib.ecf8_tensor_kernel_variant(h))

    @classmethod
    def encode(cls, x: torch.Tensor, lengths=None, threads_per_block: int = 256,
               stream: torch.cuda.Stream | None = None) -> "DeviceTensor":
        """ecf8_encode_device: encode_tensor (codec.cpp:49-98) of a CUDA FP8 /
        uint8 tensor on the GPU, straight into HBM.  lengths=None builds the
        code from the GPU exponent histogram (host build_code, huffman.cpp)."""
        x = _fp8_bytes(x)
        if lengths is None:
            lengths = build_code(exponent_histogram(x, stream))
        lv = np.ascontiguousarray(np.asarray(lengths, dtype=np.uint8))
        if lv.size != 16:
            raise ValueError("invalid length vector")
        h = C.c_void_p()
        check(lib.ecf8_encode_device(C.c_void_p(x.data_ptr() if x.numel() else None), x.numel(), threads_per_block,
                                     lv.ctypes.data_as(C.c_void_p), _stream_ptr(stream), C.byref(h)))
        self = cls.__new__(cls)
        self._src = None
        self._adopt(h)
        return self

    def to_host(self) -> EncodedTensor:
        """The tensor's container sections, copied back to host memory."""
        s = Sections()
        check(lib.ecf8_tensor_sections(self.handle, C.byref(s)))
        enc = np.empty(s.encoded_len, np.uint8)
        gaps = np.empty(s.gaps_len, np.uint8)
        outpos = np.empty(s.n_outpos, np.uint64)
        packed = np.empty(s.packed_len, np.uint8)
        check(lib.ecf8_tensor_download(self.handle, enc.ctypes.data_as(C.c_void_p), gaps.ctypes.data_as(C.c_void_p),
                                       outpos.ctypes.data_as(C.c_void_p), packed.ctypes.data_as(C.c_void_p)))
        return EncodedTensor(int(s.n_elem), int(s.threads_per_block), np.array(list(s.lengths), np.uint8), enc, gaps,
                             outpos, packed)

    def verified_tiles(self) -> tuple[int, int]:
        """(tiles decoded by the continuous group walk, all 256-window tiles)."""
        total = C.c_uint64()
        n = int(lib.ecf8_tensor_verified_tiles(self.handle, C.byref(total)))
        return n, int(total.value)

    def decode_into(self, out: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        if out.dtype not in (torch.uint8, torch.float8_e4m3fn, torch.float8_e5m2) or not out.is_cuda:
            raise ValueError("out must be a CUDA uint8/float8 tensor")
        if out.numel() != self.n_elem or not out.is_contiguous():
            raise ValueError("output size mismatch")
        check(lib.ecf8_decode_device(self.handle, C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def decode(self, stream: torch.cuda.Stream | None = None, dtype=torch.uint8) -> torch.Tensor:
        out = torch.empty(self.n_elem, dtype=dtype, device="cuda")
        return self.decode_into(out, stream)

    def free(self):
        if getattr(self, "handle", None):
            lib.ecf8_tensor_free(self.handle)
            self.handle = None

    def __del__(self):
        self.free()


class Batch:
    """ecf8_batch: many tensors decoded by one launch per window width."""

    def __init__(self, tensors: list[DeviceTensor], outs: list[torch.Tensor]):
        if len(tensors) != len(outs):
            raise ValueError("one output per tensor")
        for t, o in zip(tensors, outs):
            if o.numel() != t.n_elem or not o.is_cuda or not o.is_contiguous():
                raise ValueError("output size mismatch")
        n = len(tensors)
        ts = (C.c_void_p * n)(*[t.handle.value for t in tensors])
        os_ = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
        h = C.c_void_p()
        check(lib.ecf8_batch_create(ts, os_, n, C.byref(h)))
        self.handle = h
        self.tensors, self.outs = tensors, outs
        self.launches = int(lib.ecf8_batch_launches(h))
        self.algorithmic_bytes = sum(t.algorithmic_bytes for t in tensors)

    def decode(self, stream: torch.cuda.Stream | None = None) -> None:
        check(lib.ecf8_batch_decode(self.handle, _stream_ptr(stream)))

    def free(self):
        if getattr(self, "handle", None):
            lib.ecf8_batch_free(self.handle)
            self.handle = None

    def __del__(self):
        self.free()

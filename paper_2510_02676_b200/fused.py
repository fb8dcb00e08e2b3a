"""Decode-fused tcgen05 FP8 GEMM (csrc/cuda/fused_gemm.cu).

    y[m, n] = scale * x[m, k] . W[n, k]^T      (fp32 accumulate and output)

W is kept ECF8-compressed in HBM in the *tiled* layout (fused_layout): 128 x
128 tiles, each stored as the swizzled shared-memory image the tensor core
reads, then encoded by the unchanged ECF8 encoder.  The kernel decodes each
K tile straight into shared memory and feeds tcgen05.mma; the decoded
weights never touch HBM.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import codec
from ._lib import check, lib
from .device import DeviceTensor, _stream_ptr


def fused_layout(w: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Row-major [n, k] FP8 bytes <-> the tiled, swizzled sequence (1-D)."""
    w = np.ascontiguousarray(w, dtype=np.uint8)
    if inverse:
        raise TypeError("use fused_layout_inverse(seq, n, k)")
    n, k = w.shape
    out = np.empty(n * k, np.uint8)
    check(lib.ecf8_host_fused_layout(w.ctypes.data, n, k, out.ctypes.data, 0))
    return out


def fused_layout_inverse(seq: np.ndarray, n: int, k: int) -> np.ndarray:
    seq = np.ascontiguousarray(seq, dtype=np.uint8).reshape(-1)
    out = np.empty((n, k), np.uint8)
    check(lib.ecf8_host_fused_layout(seq.ctypes.data, n, k, out.ctypes.data, 1))
    return out


class FusedLinear:
    """An ECF8-compressed FP8 weight [n, k] served by the decode-fused GEMM."""

    def __init__(self, w_fp8: np.ndarray, fmt: str = "e4m3", threads_per_block: int = 128):
        self.n, self.k = map(int, w_fp8.shape)
        self.fmt = fmt
        # T = 128 serves both decode-lane widths (1-bit codes need T <= 128)
        self.encoded = codec.encode_tensor(fused_layout(w_fp8), threads_per_block)
        self.dev = DeviceTensor(self.encoded)
        h = C.c_void_p()
        check(lib.ecf8_fused_create(self.dev.handle, self.n, self.k, {"e4m3": 0, "e5m2": 1}[fmt], C.byref(h)))
        self.handle = h
        self.split_k = int(lib.ecf8_fused_split_k(h))

    def __call__(self, x: torch.Tensor, scale: float = 1.0, out: torch.Tensor | None = None,
                 stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        if x.dtype != torch.float8_e4m3fn or not x.is_cuda or x.dim() != 2 or x.shape[1] != self.k:
            raise ValueError("x must be a CUDA float8_e4m3fn tensor [m, k]")
        x = x.contiguous()
        m = x.shape[0]
        if out is None:
            out = torch.empty(m, self.n, dtype=torch.float32, device=x.device)
        elif (out.dtype != torch.float32 or out.device != x.device or tuple(out.shape) != (m, self.n)
              or not out.is_contiguous()):
            # the kernel zeroes and atomically adds m * n fp32 values at out.data_ptr()
            raise ValueError(f"out must be a contiguous float32 tensor [{m}, {self.n}] on {x.device}")
        check(lib.ecf8_fused_gemm(self.handle, C.c_void_p(x.data_ptr()), m, float(scale),
                                  C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    @property
    def compressed_bytes(self) -> int:
        return self.encoded.compressed_bytes()

    def free(self):
        if getattr(self, "handle", None):
            lib.ecf8_fused_free(self.handle)
            self.handle = None

    def __del__(self):
        self.free()

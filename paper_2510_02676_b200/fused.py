"""Decode-fused tcgen05 FP8 GEMM (csrc/cuda/fused_gemm.cu).

    y[m, n] = scale * x[m, k] . W[n, k]^T      (fp32 accumulate and output)

W is kept ECF8-compressed in HBM in the *tiled* layout (fused_layout): 128 x
128 tiles, each stored as the swizzled shared-memory image the tensor core
reads, then encoded by the unchanged ECF8 encoder.  The kernel decodes each
K tile straight into shared memory and feeds tcgen05.mma; the decoded
weights never touch HBM.

An alternative large-m path (ECF8_FUSED_LARGE_M=<m>): W decoded chunk by
chunk -- ~32 MB of whole 128-row tiles, back to row-major
(ecf8_fused_decode_rows) -- into a two-slot ring meant to stay in L2, each
chunk through a dense FP8 GEMM (cuBLASLt) while the next one decodes on a
side stream.  Measured slower than the fused kernel (host-bound per chunk),
so it is off by default.
"""
from __future__ import annotations

import ctypes as C
import os

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


def fused_layout_device(w: torch.Tensor, n: int, k: int, inverse: bool = False,
                        stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """ecf8_fused_layout_device: the tiled layout on the GPU (row-major <->
    tiled FP8 bytes, n * k uint8 in and out)."""
    if not w.is_cuda or w.numel() != n * k:
        raise ValueError(f"expected {n * k} CUDA bytes")
    src = w.contiguous().view(torch.uint8).reshape(-1)
    out = torch.empty(n * k, dtype=torch.uint8, device=w.device)
    check(lib.ecf8_fused_layout_device(C.c_void_p(src.data_ptr()), n, k, C.c_void_p(out.data_ptr()), int(inverse),
                                       _stream_ptr(stream)))
    return out


# m at which the decode-rows pipeline takes over (off by default: measured slower
# than the fused kernel at m = 256 -- 0.83 ms per Llama-3-70B layer with one chunk
# per linear, 1.95 ms with 32 MB chunks: host-bound per chunk)
LARGE_M = int(os.environ.get("ECF8_FUSED_LARGE_M", "100000"))
CHUNK_BYTES = int(os.environ.get("ECF8_FUSED_CHUNK_MB", "32")) << 20


class _RowsPipe:
    """Per-device state of the large-m path: a two-slot decode ring (L2-resident),
    a side stream for the decodes and the events ordering slot reuse (shared by
    every FusedLinear, so back-to-back calls keep the ring order)."""

    _by_dev: dict = {}

    def __init__(self, dev):
        self.slots = [torch.empty(CHUNK_BYTES + 16, dtype=torch.uint8, device=dev) for _ in range(2)]
        self.dec = torch.cuda.Stream(device=dev)
        self.ev_dec = [torch.cuda.Event() for _ in range(2)]
        self.ev_use = [torch.cuda.Event() for _ in range(2)]
        self.used = [False, False]
        self.k = 0  # chunks issued

    @classmethod
    def get(cls, dev) -> "_RowsPipe":
        key = torch.device(dev).index
        if key not in cls._by_dev:
            cls._by_dev[key] = cls(dev)
        return cls._by_dev[key]


class FusedLinear:
    """An ECF8-compressed FP8 weight [n, k] served by the decode-fused GEMM.

    FusedLinear(w_fp8)                  host bytes, tiled and encoded on the host
    FusedLinear.from_encoded(t, n, k)   a row-major ECF8 tensor (e.g. one tensor
                                        of a reference-written .ecf8 container,
                                        any T) re-tiled on the GPU: decode ->
                                        tiled layout -> device encoder (T = 128)
    """

    def __init__(self, w_fp8: np.ndarray | None, fmt: str = "e4m3", threads_per_block: int = 128,
                 _dev: DeviceTensor | None = None, _nk: tuple[int, int] | None = None):
        if fmt not in ("e4m3", "e5m2"):
            raise ValueError("fmt must be e4m3 or e5m2")
        self.fmt = fmt
        if _dev is None:
            self.n, self.k = map(int, w_fp8.shape)
            # T = 128 serves both decode-lane widths (1-bit codes need T <= 128)
            self.encoded = codec.encode_tensor(fused_layout(w_fp8), threads_per_block)
            self.dev = DeviceTensor(self.encoded)
        else:
            self.n, self.k = _nk
            self.encoded = None
            self.dev = _dev
        h = C.c_void_p()
        check(lib.ecf8_fused_create(self.dev.handle, self.n, self.k, {"e4m3": 0, "e5m2": 1}[fmt], C.byref(h)))
        self.handle = h
        self.split_k = int(lib.ecf8_fused_split_k(h))
        self.rows_ok = bool(lib.ecf8_fused_byte_steps(h))
        self._one = None

    @classmethod
    def from_encoded(cls, t: codec.EncodedTensor, n: int, k: int, fmt: str = "e4m3",
                     stream: torch.cuda.Stream | None = None) -> "FusedLinear":
        """Serve a row-major ECF8 weight (reference container layout) through
        the fused GEMM: decoded, re-tiled and re-encoded on the GPU -- no host
        round trip of the weight."""
        if t.n_elem != n * k or n % 128 or k % 128:
            raise ValueError("fused GEMM needs an n x k weight with n, k multiples of 128")
        rowmajor = DeviceTensor(t, stream)
        w = rowmajor.decode(stream)
        tiled = fused_layout_device(w, n, k, stream=stream)
        del w
        rowmajor.free()
        dev = DeviceTensor.encode(tiled, threads_per_block=128, stream=stream)
        return cls(None, fmt, _dev=dev, _nk=(n, k))

    @classmethod
    def from_container(cls, data: bytes, name: str, fmt: str = "e4m3") -> "FusedLinear":
        """One 2-D tensor of an .ecf8 container (container.hpp:18-30) by name."""
        f = codec.parse_container(data)
        for (tname, t), dims in zip(f.tensors, f.shapes):
            if tname == name:
                if len(dims) != 2:
                    raise ValueError(f"{name}: expected a 2-D weight, got shape {dims}")
                return cls.from_encoded(t, int(dims[0]), int(dims[1]), fmt)
        raise KeyError(name)

    @property
    def compressed_bytes(self) -> int:
        return int(lib.ecf8_tensor_algorithmic_bytes(self.dev.handle)) - self.n * self.k

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
        if m >= LARGE_M and self.rows_ok:
            return self._rows_path(x, scale, out, stream)
        check(lib.ecf8_fused_gemm(self.handle, C.c_void_p(x.data_ptr()), m, float(scale),
                                  C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def _rows_path(self, x: torch.Tensor, scale: float, out: torch.Tensor, stream) -> torch.Tensor:
        """Large m: W decoded in ~32 MB chunks of whole 128-row tiles into an
        L2-resident two-slot ring (ecf8_fused_decode_rows, side stream), each
        chunk multiplied by a dense FP8 GEMM on the caller's stream."""
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        p = _RowsPipe.get(x.device)
        m, k = x.shape
        if self._one is None:
            self._one = torch.ones((), device=x.device)
        pad = (-m) % 16
        xp = torch.cat([x, x.new_zeros(pad, k)]) if pad else x
        sb = torch.full((), float(scale), device=x.device)
        wdt = torch.float8_e4m3fn if self.fmt == "e4m3" else torch.float8_e5m2
        rows = max(128, min(self.n, CHUNK_BYTES // k // 128 * 128))
        for r0 in range(0, self.n, rows):
            r1 = min(self.n, r0 + rows)
            s = p.k % 2
            p.k += 1
            if p.used[s]:
                p.dec.wait_event(p.ev_use[s])  # the GEMM that last read this slot is done
            check(lib.ecf8_fused_decode_rows(self.handle, r0, r1, C.c_void_p(p.slots[s].data_ptr()),
                                             C.c_void_p(p.dec.cuda_stream)))
            p.ev_dec[s].record(p.dec)
            st.wait_event(p.ev_dec[s])
            w = p.slots[s][: (r1 - r0) * k].view(wdt).view(r1 - r0, k)
            with torch.cuda.stream(st):
                y = torch._scaled_mm(xp, w.t(), scale_a=self._one, scale_b=sb, out_dtype=torch.float32)
                out[:, r0:r1].copy_(y[:m])
            p.ev_use[s].record(st)
            p.used[s] = True
        return out

    def free(self):
        if getattr(self, "handle", None) and lib is not None:
            lib.ecf8_fused_free(self.handle)
            self.handle = None

    def __del__(self):
        self.free()


# ---- torch.library op: the fused GEMM as a PyTorch operator (shape-inferable,
# usable from torch.compile'd graphs and CUDA graphs; the handle is the
# FusedLinear's ecf8_fused*)

@torch.library.custom_op("ecf8::fused_gemm", mutates_args=())
def fused_gemm_op(x: torch.Tensor, handle: int, n: int, scale: float) -> torch.Tensor:
    """y[m, n] (fp32) = scale * x[m, k] . W^T for the ECF8 weight behind `handle`."""
    if x.dtype != torch.float8_e4m3fn or not x.is_cuda or x.dim() != 2:
        raise ValueError("x must be a CUDA float8_e4m3fn tensor [m, k]")
    x = x.contiguous()
    out = torch.empty(x.shape[0], n, dtype=torch.float32, device=x.device)
    check(lib.ecf8_fused_gemm(C.c_void_p(handle), C.c_void_p(x.data_ptr()), x.shape[0], float(scale),
                              C.c_void_p(out.data_ptr()), _stream_ptr(None)))
    return out


@fused_gemm_op.register_fake
def _fused_gemm_fake(x: torch.Tensor, handle: int, n: int, scale: float) -> torch.Tensor:
    return x.new_empty(x.shape[0], n, dtype=torch.float32)

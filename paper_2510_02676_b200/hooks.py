"""Just-in-time per-layer decode into one reused HBM buffer.

The paper keeps weights ECF8-compressed in HBM and decodes each layer right
before it is used, into a single pre-allocated buffer (PAPER.md:170-173,
"decode-then-use"); the reference library stops at the host API (SPEC.md:14
lists framework hooks as out of its scope).  Here:

  * ``DecodeArena``  -- one device buffer, sized for the largest layer, that
    every layer decodes into (the device-side ``ReusableBuffer``,
    container.hpp:80-95): grow-only, counts its allocations.
  * ``ECF8Linear``   -- an ``nn.Module`` holding ECF8-compressed FP8 weights
    ([out_features, in_features] E4M3 or E5M2 bytes) resident in HBM.  When
    both feature sizes are multiples of 128 (and m <= 256 tokens), forward is
    the decode-fused tcgen05 GEMM (``torch.ops.ecf8.fused_gemm``: the weight
    is decoded tile by tile into shared memory and never written to HBM; its
    tiled copy is made on the GPU from the row-major ECF8 tensor, fused.py);
    otherwise it decodes the weight with one batched launch into the arena
    and runs the FP8 GEMM (``torch._scaled_mm``, cuBLASLt) on it.
  * ``compress_linears`` -- replaces the ``nn.Linear`` layers of a model with
    ``ECF8Linear`` built from FP8-quantised copies of their weights.

The decode is the sm_100a kernel (libecf8_b200.so); nothing here falls back
to the CPU.
"""
from __future__ import annotations

import numpy as np
import torch
from torch import nn

from . import codec
from .device import Batch, DeviceTensor

_FP8 = {"e4m3": torch.float8_e4m3fn, "e5m2": torch.float8_e5m2}


class DecodeArena:
    """One reused device buffer for just-in-time decoded weights."""

    def __init__(self, device: str | torch.device = "cuda"):
        self.device = torch.device(device)
        self.buf: torch.Tensor | None = None
        self.allocations = 0

    def take(self, n_bytes: int) -> torch.Tensor:
        need = (n_bytes + 255) // 256 * 256
        if self.buf is None or self.buf.numel() < need:
            self.buf = torch.empty(need, dtype=torch.uint8, device=self.device)
            self.allocations += 1
        return self.buf

    @property
    def capacity(self) -> int:
        return 0 if self.buf is None else self.buf.numel()


_default_arena: DecodeArena | None = None


def default_arena() -> DecodeArena:
    global _default_arena
    if _default_arena is None:
        _default_arena = DecodeArena()
    return _default_arena


class ECF8Linear(nn.Module):
    """y = x @ W^T (+ bias) with W kept ECF8-compressed in HBM.

    ``weight_fp8``: uint8 array [out_features, in_features] of FP8 bytes
    (``fmt`` "e4m3" or "e5m2"); ``scale_w``: per-tensor dequant scale.
    Activations are quantised per tensor to E4M3 with ``scale_x`` (computed
    from the batch when None); cuBLASLt has no E5M2 x E5M2 GEMM, E4M3 x E5M2
    is supported."""

    def __init__(self, weight_fp8: np.ndarray, bias: torch.Tensor | None = None, scale_w: float = 1.0,
                 fmt: str = "e4m3", threads_per_block: int = 256, arena: DecodeArena | None = None,
                 fused: bool | None = None):
        super().__init__()
        if weight_fp8.ndim != 2:
            raise ValueError("weight must be [out_features, in_features]")
        self.out_features, self.in_features = map(int, weight_fp8.shape)
        if self.in_features % 16 or self.out_features % 16:
            raise ValueError("FP8 GEMM needs feature sizes that are multiples of 16")
        self.fmt = fmt
        self.encoded = codec.encode_tensor(np.ascontiguousarray(weight_fp8).reshape(-1), threads_per_block)
        self.dev = DeviceTensor(self.encoded)
        self.register_buffer("scale_w", torch.tensor(float(scale_w), dtype=torch.float32, device="cuda"))
        self.bias = None if bias is None else nn.Parameter(bias.detach().to("cuda", torch.bfloat16), False)
        self.arena = arena or default_arena()
        self._batch_key = None
        self._batch = None
        if fused is None:
            fused = self.out_features % 128 == 0 and self.in_features % 128 == 0
        self.fused = None
        if fused:
            from .fused import FusedLinear

            # the tiled copy is made on the GPU from the row-major ECF8 tensor
            self.fused = FusedLinear.from_encoded(self.encoded, self.out_features, self.in_features, fmt)

    @property
    def compressed_bytes(self) -> int:
        return self.encoded.compressed_bytes()

    def decode_weight(self, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Decode W into the arena; returns the [out, in] FP8 view (valid until
        the next decode into the same arena)."""
        n = self.out_features * self.in_features
        buf = self.arena.take(n)
        key = buf.data_ptr()
        if self._batch_key != key:  # arena regrew: rebuild the launch descriptor
            self._batch = Batch([self.dev], [buf[:n]])
            self._batch_key = key
        self._batch.decode(stream)
        return buf[:n].view(_FP8[self.fmt]).view(self.out_features, self.in_features)

    def forward(self, x: torch.Tensor, scale_x: torch.Tensor | None = None) -> torch.Tensor:
        lead = x.shape[:-1]
        x2 = x.reshape(-1, self.in_features)
        act = torch.float8_e4m3fn
        if x2.dtype != act:
            if scale_x is None:
                amax = x2.abs().amax().float().clamp_min(1e-12)
                scale_x = amax / torch.finfo(act).max
            x2 = (x2.float() / scale_x).to(act)
        elif scale_x is None:
            scale_x = torch.tensor(1.0, device=x.device)
        m = x2.shape[0]
        if self.fused is not None and 1 <= m <= 256:
            y = torch.ops.ecf8.fused_gemm(x2, self.fused.handle.value, self.out_features, 1.0)
            y = y * (scale_x.float().reshape(()) * self.scale_w)
            if self.bias is not None:
                y = y + self.bias.float()
            return y.to(torch.bfloat16).reshape(*lead, self.out_features)
        w = self.decode_weight()
        pad = (-m) % 16
        if pad:
            x2 = torch.cat([x2, x2.new_zeros(pad, self.in_features)])
        y = torch._scaled_mm(x2, w.t(), scale_a=scale_x.float().reshape(()), scale_b=self.scale_w,
                             bias=self.bias, out_dtype=torch.bfloat16)
        return y[:m].reshape(*lead, self.out_features)


def quantize_fp8(w: torch.Tensor, fmt: str = "e4m3") -> tuple[np.ndarray, float]:
    """Per-tensor FP8 quantisation (RNE, saturating): (bytes, scale)."""
    dt = _FP8[fmt]
    amax = float(w.detach().abs().max().clamp_min(1e-12))
    scale = amax / torch.finfo(dt).max
    q = (w.detach().float() / scale).clamp(-torch.finfo(dt).max, torch.finfo(dt).max).to(dt)
    return q.view(torch.uint8).cpu().numpy(), scale


def compress_linears(model: nn.Module, fmt: str = "e4m3", arena: DecodeArena | None = None,
                     threads_per_block: int = 256, fused: bool | None = None) -> dict[str, ECF8Linear]:
    """Replace every nn.Linear (feature sizes multiple of 16) by an ECF8Linear
    sharing one decode arena (fused: see ECF8Linear; None = where the shapes
    allow).  Returns {qualified name: module}."""
    arena = arena or DecodeArena()
    done = {}
    for name, mod in list(model.named_modules()):
        for cname, child in list(mod.named_children()):
            if isinstance(child, nn.Linear) and child.in_features % 16 == 0 and child.out_features % 16 == 0:
                q, s = quantize_fp8(child.weight, fmt)
                new = ECF8Linear(q, child.bias, s, fmt, threads_per_block, arena, fused)
                setattr(mod, cname, new)
                done[f"{name}.{cname}" if name else cname] = new
    return done

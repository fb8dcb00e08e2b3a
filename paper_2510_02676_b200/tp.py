"""Tensor-parallel decode-fused linear (BASELINE configs[2]).

Column parallel: W [N, K] is split along N into `world` shards, each shard
ECF8-encoded independently (its own code, container.cpp:291-322) and held
compressed on its rank.  Rank r computes y_r = x . W_r^T with the
decode-fused tcgen05 GEMM (fused.py), then one all-gather over the process
group (NCCL over NVLink on the B200 box) assembles y [M, N].  This gather is
the only collective anywhere in the framework.
"""
from __future__ import annotations

import numpy as np
import torch


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Row range [lo, hi) of rank's column shard; n must split into 128-row tiles."""
    if n % (128 * world):
        raise ValueError(f"N={n} does not split into {world} shards of whole 128-row tiles")
    per = n // world
    return rank * per, (rank + 1) * per


def gather_columns(y_local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[M, N/world] per rank -> [M, N] on every rank (one all_gather)."""
    import torch.distributed as dist

    m, nl = y_local.shape
    if world == 1:
        return y_local
    y_local = y_local.contiguous()
    if dist.get_backend(group) == "nccl":  # one NVLink all-gather into a single buffer
        buf = torch.empty(world, m, nl, dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(buf, y_local, group=group)
    else:  # gloo (CPU tests): list form
        parts = [torch.empty_like(y_local) for _ in range(world)]
        dist.all_gather(parts, y_local, group=group)
        buf = torch.stack(parts)
    return buf.permute(1, 0, 2).reshape(m, world * nl)


class TPFusedLinear:
    """One rank's shard of a column-parallel ECF8 linear."""

    def __init__(self, w_fp8: np.ndarray, rank: int, world: int, fmt: str = "e4m3", local=None):
        n, self.k = map(int, w_fp8.shape)
        self.n = n
        self.rank, self.world = rank, world
        lo, hi = shard_rows(n, world, rank)
        self.rows = (lo, hi)
        shard = np.ascontiguousarray(w_fp8[lo:hi])
        if local is None:
            from .fused import FusedLinear

            local = FusedLinear(shard, fmt)
        self.local = local  # callable (x [m, k], scale) -> y_local [m, hi - lo]

    def __call__(self, x: torch.Tensor, scale: float = 1.0, group=None) -> torch.Tensor:
        y_local = self.local(x, scale)
        return gather_columns(y_local, self.world, group)

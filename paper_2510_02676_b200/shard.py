"""Multi-GPU shard driver: independent ECF8 units partitioned across ranks.

Every tensor (or TP/EP shard of a tensor) is its own ECF8 stream with its own
code (container.cpp:291-322 encodes tensors independently), so
decode needs no exchange between GPUs: each rank decodes the units it owns,
and the only cross-rank traffic is one scalar max-reduce of the elapsed time
(the report, not the data path).  One process per GPU, torch.distributed for
rendezvous (NCCL on the B200 box, gloo in the CPU tests).

Partition policies:
  * ``lpt``      -- dense layers / DiT tensors: longest-processing-time
                    bin packing by compressed bytes (the decode cost);
  * ``round_robin`` -- MoE experts: expert e -> rank e mod world (EP).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from typing import Sequence


def lpt_partition(costs: Sequence[int], world: int) -> list[list[int]]:
    """Greedy LPT: units by decreasing cost, each onto the least-loaded rank.

    Deterministic (ties broken by unit index, then rank index) so every rank
    computes the same plan without communicating.  Returns per-rank unit
    indices in ascending order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-int(costs[i]), i))
    heap = [(0, r) for r in range(world)]
    parts: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        parts[r].append(i)
        heapq.heappush(heap, (load + int(costs[i]), r))
    return [sorted(p) for p in parts]


def round_robin_partition(n_units: int, world: int) -> list[list[int]]:
    """EP placement: unit e on rank e mod world."""
    if world < 1:
        raise ValueError("world must be >= 1")
    return [list(range(r, n_units, world)) for r in range(world)]


def partition(costs: Sequence[int], world: int, policy: str = "lpt") -> list[list[int]]:
    if policy == "lpt":
        return lpt_partition(costs, world)
    if policy == "round_robin":
        return round_robin_partition(len(costs), world)
    raise ValueError(f"unknown shard policy {policy!r}")


def imbalance(costs: Sequence[int], parts: list[list[int]]) -> float:
    """max rank load / mean rank load (1.0 = perfect)."""
    loads = [sum(int(costs[i]) for i in p) for p in parts]
    mean = sum(loads) / max(1, len(loads))
    return max(loads) / mean if mean else 1.0


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (elapsed device time) over the process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: int, dist=None, device=None) -> int:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return int(value)
    import torch

    t = torch.tensor([int(value)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


@dataclass
class ShardPlan:
    """This rank's share of a list of encoded units."""

    rank: int
    world: int
    policy: str
    parts: list[list[int]]
    costs: list[int] = field(default_factory=list)

    @classmethod
    def build(cls, costs: Sequence[int], rank: int, world: int, policy: str = "lpt") -> "ShardPlan":
        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside world {world}")
        return cls(rank, world, policy, partition(costs, world, policy), [int(c) for c in costs])

    @property
    def mine(self) -> list[int]:
        return self.parts[self.rank]

    @property
    def my_cost(self) -> int:
        return sum(self.costs[i] for i in self.mine)

    def imbalance(self) -> float:
        return imbalance(self.costs, self.parts)


class ShardedDecoder:
    """Decode this rank's units on its GPU in one batched launch per group.

    ``units`` is the full, rank-independent list of EncodedTensor (every rank
    builds the same list, or a lazily-materialised one: only ``mine`` is
    touched).  Outputs are device tensors owned by the decoder."""

    def __init__(self, units, rank: int, world: int, policy: str = "lpt", group_size: int = 0, costs=None):
        import torch

        from .device import Batch, DeviceTensor

        if costs is None:
            costs = [u.compressed_bytes() for u in units]
        self.plan = ShardPlan.build(costs, rank, world, policy)
        mine = self.plan.mine
        self.dev = [DeviceTensor(units[i]) for i in mine]
        self.outs = [torch.empty(t.n_elem, dtype=torch.uint8, device="cuda") for t in self.dev]
        g = group_size or max(1, len(mine))
        self.batches = [Batch(self.dev[k:k + g], self.outs[k:k + g]) for k in range(0, len(mine), g)]
        self.algorithmic_bytes = sum(b.algorithmic_bytes for b in self.batches)
        self.launches = sum(b.launches for b in self.batches)

    def decode(self, stream=None) -> None:
        for b in self.batches:
            b.decode(stream)

    def outputs(self) -> dict[int, "object"]:
        """unit index -> decoded device tensor."""
        return dict(zip(self.plan.mine, self.outs))

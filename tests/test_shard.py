"""Multi-GPU shard driver (paper_2510_02676_b200/shard.py).

CPU: partition policies, and a world_size-2 gloo process group in which
each rank plans independently, decodes its own units (with the CPU oracle
standing in for the GPU -- test infrastructure only) and the ranks agree on
coverage, max-over-ranks time and total bytes.
GPU: the ShardedDecoder for every rank of a 2- and 4-way plan, run on one
device, reassembles the whole model bit-exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_02676_b200 import codec
from paper_2510_02676_b200.shard import (ShardPlan, imbalance, lpt_partition, max_over_ranks, partition,
                                         round_robin_partition, sum_over_ranks)


def test_lpt_covers_every_unit_once_and_balances():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        for n in (0, 1, 7, 64, 224):
            costs = rng.integers(1, 1 << 30, n).tolist()
            parts = lpt_partition(costs, world)
            assert len(parts) == world
            assert sorted(i for p in parts for i in p) == list(range(n))
            if n:
                # Graham's LPT bound: makespan <= 4/3 OPT, OPT >= max(mean, max unit)
                opt_lb = max(sum(costs) / world, max(costs))
                assert max(sum(costs[i] for i in p) for p in parts) <= 4 / 3 * opt_lb + 1
    assert lpt_partition([5, 5, 5, 5], 2) == [[0, 2], [1, 3]]


def test_lpt_is_deterministic():
    costs = [3, 3, 3, 2, 2, 2, 1, 1]
    assert lpt_partition(costs, 3) == lpt_partition(list(costs), 3)


def test_llama_layers_lpt_is_balanced():
    # Llama-3.1-8B linears x 32 layers, cost ~ elements: 8 GPUs within 1 %
    shapes = [4096 * 4096, 1024 * 4096, 1024 * 4096, 4096 * 4096, 14336 * 4096, 14336 * 4096, 4096 * 14336]
    costs = shapes * 32
    assert imbalance(costs, lpt_partition(costs, 8)) < 1.01


def test_round_robin_experts():
    parts = round_robin_partition(256, 8)
    assert parts[3][:3] == [3, 11, 19] and all(len(p) == 32 for p in parts)
    assert partition([1] * 10, 4, "round_robin") == round_robin_partition(10, 4)
    with pytest.raises(ValueError):
        partition([1], 2, "bogus")
    with pytest.raises(ValueError):
        ShardPlan.build([1, 2], 2, 2)


def test_single_process_reductions_are_identity():
    assert max_over_ranks(3.5) == 3.5 and sum_over_ranks(7) == 7


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, units_path, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _oracle import oracle, tensor_dict

        data = np.load(units_path, allow_pickle=True)
        raws = list(data["raws"])
        units = codec.encode_many(raws, 64)
        plan = ShardPlan.build([u.compressed_bytes() for u in units], rank, world, "lpt")
        orc = oracle()
        mine = {i: orc.decode_parallel(tensor_dict(units[i])) for i in plan.mine}
        ok = all(np.array_equal(mine[i], raws[i]) for i in plan.mine)
        elapsed = 1.0 + rank  # stand-in per-rank device time
        mx = max_over_ranks(elapsed, dist)
        total = sum_over_ranks(sum(units[i].algorithmic_bytes() for i in plan.mine), dist)
        gathered = [None] * world
        dist.all_gather_object(gathered, plan.mine)
        out_q.put((rank, ok, mx, total, gathered, sum(u.algorithmic_bytes() for u in units)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_partition_and_reduce(tmp_path):
    world = 2
    raws = [codec.synth(1.8, 0.05, n, 40 + k) for k, n in enumerate([5000, 12000, 3000, 9000, 700, 20000])]
    p = tmp_path / "units.npz"
    np.savez(p, raws=np.array(raws, dtype=object))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, str(p), q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    all_bytes = res[0][5]
    for rank, ok, mx, total, gathered, _ in res:
        assert ok
        assert mx == 2.0  # max over ranks of (1 + rank)
        assert total == all_bytes  # every unit decoded exactly once
        assert sorted(i for g in gathered for i in g) == list(range(len(raws)))
    assert res[0][4] == res[1][4]  # identical plans without communication


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_decoder_reassembles_model(world):
    from paper_2510_02676_b200.shard import ShardedDecoder

    sizes = [4096 * 64, 1024 * 64, 14336 * 16, 64 * 14336, 333, 70001, 4096 * 33]
    raws = [codec.synth(1.8, 0.05, n, 900 + k) for k, n in enumerate(sizes)]
    units = codec.encode_many(raws, 256)
    got = {}
    for rank in range(world):
        d = ShardedDecoder(units, rank, world)
        d.decode()
        torch.cuda.synchronize()
        for i, out in d.outputs().items():
            assert i not in got
            got[i] = out.cpu().numpy()
    assert sorted(got) == list(range(len(raws)))
    for i, r in enumerate(raws):
        assert np.array_equal(got[i], r), i

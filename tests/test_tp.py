"""Tensor-parallel decode-fused linear (paper_2510_02676_b200/tp.py).

CPU: world_size-2 gloo group; each rank holds only its column shard (the
local GEMM is a CPU stand-in here, the fused kernel needs the B200) and the
all-gather assembles y = x . W^T exactly.
GPU: the per-shard fused GEMMs concatenated equal the unsharded fused GEMM.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_02676_b200.tp import TPFusedLinear, shard_rows


def _fp8_to_f32(b: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(b)).view(torch.float8_e4m3fn).float()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, q)
    except Exception as e:  # surface failures instead of a queue timeout
        q.put((rank, False, repr(e), None))
    finally:
        dist.destroy_process_group()


def _body(rank, world, q):
    if True:
        rng = np.random.default_rng(0)  # same W and x on every rank
        w = rng.integers(0, 0x7E, (512, 256), dtype=np.uint8)
        x = torch.from_numpy(rng.standard_normal((5, 256)).astype(np.float32))

        def make_local(shard):
            ws = _fp8_to_f32(shard)
            return lambda xx, scale: (xx @ ws.T) * scale

        lo, hi = shard_rows(512, world, rank)
        lin = TPFusedLinear(w, rank, world, local=make_local(w[lo:hi]))
        y = lin(x, 0.5)
        want = (x @ _fp8_to_f32(w).T) * 0.5
        q.put((rank, bool(torch.equal(y, want)), tuple(y.shape), lin.rows))


def test_shard_rows():
    assert shard_rows(1024, 4, 3) == (768, 1024)
    with pytest.raises(ValueError):
        shard_rows(384, 2, 0)


def test_gloo_world2_column_parallel_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] and res[1][1], res
    assert res[0][2] == (5, 512) and res[0][3] == (0, 256) and res[1][3] == (256, 512)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_shards_concatenate_to_full_fused_gemm(world):
    from paper_2510_02676_b200 import codec
    from paper_2510_02676_b200.fused import FusedLinear

    n, k, m = 1024, 1024, 16
    w = codec.synth(1.8, 0.05, n * k, 31).reshape(n, k)
    x = (torch.randn(m, k, device="cuda") * 4).to(torch.float8_e4m3fn)
    full = FusedLinear(w)(x, 0.5)
    parts = [TPFusedLinear(w, r, world).local(x, 0.5) for r in range(world)]
    got = torch.cat(parts, dim=1)
    tol = 1e-3 * full.abs().max().item() + 1e-3
    assert (got - full).abs().max().item() <= tol

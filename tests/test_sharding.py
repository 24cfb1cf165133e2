"""Multi-rank placement and the head-output gather on CPU (gloo, world 2/4)."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_00527_b200.sharding import (
    DecodeShape,
    batch_shard,
    gather_head_outputs,
    head_shard,
    local_queries,
)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("kind", ["batch", "head"])
def test_plans_partition_all_units(world, kind):
    shape = DecodeShape(layers=3, batch=16, q_heads=32, kv_heads=8)
    fn = batch_shard if kind == "batch" else head_shard
    owners = {}
    for r in range(world):
        p = fn(shape, world, r)
        seen = set()
        for layer in range(shape.layers):
            for b in range(shape.batch):
                for h in range(shape.kv_heads):
                    if p.owns(layer, b, h):
                        assert (layer, b, h) not in owners
                        owners[(layer, b, h)] = r
                        seen.add(p.unit_index(layer, b, h))
        assert seen == set(range(p.n_units))  # dense local numbering
        # each layer is a contiguous unit range
        upl = p.units_per_layer
        for layer in range(shape.layers):
            ids = {p.unit_index(layer, b, h) for b in range(p.b0, p.b1) for h in range(p.h0, p.h1)}
            assert ids == set(range(layer * upl, (layer + 1) * upl))
    assert len(owners) == shape.layers * shape.batch * shape.kv_heads


def test_head_shard_more_ranks_than_heads():
    shape = DecodeShape(layers=1, batch=32, q_heads=64, kv_heads=8)
    p = head_shard(shape, 16, 5)
    assert p.kv_heads == 1 and p.batch == 16 and p.h0 == 2
    with pytest.raises(ValueError):
        head_shard(DecodeShape(1, 3, 8, 8), 16, 0)


def test_local_queries_gqa_order():
    shape = DecodeShape(layers=1, batch=2, q_heads=8, kv_heads=4)
    q = torch.arange(2 * 8 * 3, dtype=torch.float32).reshape(2, 8, 3)
    p = head_shard(shape, 2, 1)  # kv heads 2,3 -> q heads 4..7
    lq = local_queries(q, p)
    assert lq.shape == (4, 2, 3)
    assert torch.equal(lq[0, 0], q[0, 4]) and torch.equal(lq[1, 1], q[0, 7]) and torch.equal(lq[3, 0], q[1, 6])


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = DecodeShape(layers=2, batch=4, q_heads=16, kv_heads=4, head_dim=8)
        full = torch.randn(shape.layers, shape.batch, shape.q_heads, 8, generator=torch.Generator().manual_seed(0))
        plan = head_shard(shape, world, rank)
        ok = True
        for layer in range(shape.layers):
            # stand-in for this rank's attention output: its slice of the truth
            local = local_queries(full[layer], plan)
            got = gather_head_outputs(local, plan)
            ok &= bool(torch.equal(got, full[layer]))
        result[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_head_gather(world):
    port = _free_port()
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, port, result), nprocs=world, join=True)
    assert all(result[r] for r in range(world))

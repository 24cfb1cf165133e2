"""Fused decode + head-output gather over peer memory:
two ranks on ONE GPU (this environment has one), sharing their gathered
buffers through CUDA IPC and exchanging handles over gloo.  Each rank checks
the gathered [L, B, Hq, d] against a decode of the full (all-heads) cache."""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _keys(shape, layer, b, h, T):
    from oracle import polar_oracle as po

    return po.synthetic_keys(T, 128, seed=(layer * shape.batch + b) * shape.kv_heads + h, outliers=(0, 1))


def _worker(rank, world, port, G, result_dir, batch=3, T=700, layers=2):
    import torch
    import torch.distributed as dist

    import paper_2502_00527_b200 as pq
    from paper_2502_00527_b200 import sharding as sh

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        shape = sh.DecodeShape(layers=layers, batch=batch, q_heads=2 * G, kv_heads=2)
        plan = sh.head_shard(shape, world, rank)
        rng = np.random.default_rng(0)
        vals = rng.standard_normal((shape.layers, shape.batch, shape.kv_heads, T, 128)).astype(np.float32)
        qs = torch.from_numpy(rng.standard_normal((4, shape.layers, shape.batch, shape.q_heads, 128)).astype(np.float32))
        qs = qs.to(torch.bfloat16).cuda()
        q = qs[0]
        cfg = pq.QuantConfig(4, 4)
        # this rank's shard, units in plan.unit_index order
        cache = pq.PolarKVCache(cfg, plan.n_units, 128, 0, capacity=T)
        for layer in range(shape.layers):
            for b in range(plan.b0, plan.b1):
                for h in range(plan.h0, plan.h1):
                    u = plan.unit_index(layer, b, h)
                    cache.prefill(torch.from_numpy(_keys(shape, layer, b, h, T)).cuda().unsqueeze(0),
                                  torch.from_numpy(vals[layer, b, h]).cuda().unsqueeze(0), unit_start=u)
        dec = sh.HeadShardedDecoder(cache, plan, gather="p2p")
        # four eager steps with different queries and no host barrier between
        # them (the double-buffered gather keeps a fast rank from overwriting
        # rows a slow rank has not read yet)
        eager = [dec.step(qs[i]) for i in range(4)]
        torch.cuda.synchronize()
        eager = [e.float().cpu().numpy() for e in eager]
        got = []
        # CUDA-graph replay (the flags count publications, so replays stay in step)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            dec.step(q)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        dec.begin_step()
        par = dec.peers.parity
        with torch.cuda.graph(graph):
            for layer in range(shape.layers):
                dec.layer(layer, q[layer])
        for _ in range(2):
            dec.peers.out.zero_()
            torch.cuda.synchronize()
            dist.barrier()  # every rank has cleared its buffer before anyone writes again
            graph.replay()
            torch.cuda.synchronize()
            got.append(dec.peers.out[par].float().cpu().numpy())
            dist.barrier()
        # reference: the full cache (all heads) decoded locally, [L, B, Hkv] units
        full = pq.PolarKVCache(cfg, shape.layers * shape.batch * shape.kv_heads, 128, 0, capacity=T)
        for layer in range(shape.layers):
            for b in range(shape.batch):
                for h in range(shape.kv_heads):
                    u = (layer * shape.batch + b) * shape.kv_heads + h
                    full.prefill(torch.from_numpy(_keys(shape, layer, b, h, T)).cuda().unsqueeze(0),
                                 torch.from_numpy(vals[layer, b, h]).cuda().unsqueeze(0), unit_start=u)
        def ref_of(qq):
            qu = qq.reshape(shape.layers * shape.batch * shape.kv_heads, G, 128)
            r = full.decode(qu, out_dtype=torch.float32).reshape(shape.layers, shape.batch, shape.q_heads, 128)
            return r.cpu().numpy()

        def err(g, r):
            return float(np.abs(g - r).max() / max(1.0, np.abs(r).max()))

        ref = ref_of(q)
        errs = [err(g, ref) for g in got] + [err(e, ref_of(qs[i])) for i, e in enumerate(eager)]
        np.save(os.path.join(result_dir, f"rank{rank}.npy"), np.array(errs))
        del graph
        dec.close()  # collective: peers unmapped, own buffers freed
        assert dec.peers is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,shape", [(4, (3, 700, 2)), (8, (3, 700, 2)), (8, (32, 1024, 1))])
def test_peer_gather_two_ranks_one_gpu(tmp_path, G, shape):
    """(8, (32, 1024, 1)): each rank's layer is 32 units of G = 8, so its
    decode runs on the thread-block-cluster path with the peer stores."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, G, str(tmp_path), *shape)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    for r in range(2):
        errs = np.load(tmp_path / f"rank{r}.npy")
        # bf16 gathered outputs vs the fp32 full-cache decode: 2^-7 relative + ulp
        assert (errs <= 2.0 ** -7).all(), errs

"""Multi-GPU placement of cache units and the per-layer head-output gather.

Every (layer, sequence, kv-head) unit is independent in both hot paths
(scales are per unit, kv_cache.py:171; query head hq reads only kv head
hq // G), so the cache shards without any data-path exchange:

* batch sharding  -- each rank owns whole sequences (all layers, all heads):
                     no collective at all; the benchmark's default (weak scaling).
* head sharding   -- each rank owns a contiguous block of KV heads (and, when
                     there are more ranks than KV heads, a slice of the batch).
                     A layer's attention output then spans ranks, so the
                     per-layer [B, Hq, d] output is all-gathered (NCCL over
                     NVLink on the GPU box; gloo in the CPU tests).  This is the
                     only collective on the path (configs[2], configs[3]).
                     ``gather="p2p"`` fuses it into the decode kernel instead:
                     the epilogue stores each output row into every rank's
                     gathered buffer through CUDA IPC peer pointers and the
                     grid's last CTA publishes a per-(layer, rank) flag
                     (PeerGather, pqb_decode_attn_peer / pqb_peer_wait).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class DecodeShape:
    layers: int
    batch: int
    q_heads: int
    kv_heads: int
    head_dim: int = 128

    def __post_init__(self) -> None:
        if self.q_heads % self.kv_heads:
            raise ValueError(f"q_heads {self.q_heads} not a multiple of kv_heads {self.kv_heads}")

    @property
    def group(self) -> int:
        return self.q_heads // self.kv_heads


@dataclass(frozen=True)
class ShardPlan:
    """Units owned by one rank: layers x sequences [b0, b1) x kv heads [h0, h1)."""

    shape: DecodeShape
    world: int
    rank: int
    b0: int
    b1: int
    h0: int
    h1: int

    @property
    def batch(self) -> int:
        return self.b1 - self.b0

    @property
    def kv_heads(self) -> int:
        return self.h1 - self.h0

    @property
    def units_per_layer(self) -> int:
        return self.batch * self.kv_heads

    @property
    def n_units(self) -> int:
        return self.shape.layers * self.units_per_layer

    def unit_index(self, layer: int, b: int, h: int) -> int:
        """Local unit id of global (layer, sequence b, kv head h); layer-major,
        then sequence, then head -- a layer is a contiguous unit range."""
        if not (self.b0 <= b < self.b1 and self.h0 <= h < self.h1):
            raise KeyError((layer, b, h))
        return (layer * self.batch + (b - self.b0)) * self.kv_heads + (h - self.h0)

    def owns(self, layer: int, b: int, h: int) -> bool:
        return self.b0 <= b < self.b1 and self.h0 <= h < self.h1 and 0 <= layer < self.shape.layers


def batch_shard(shape: DecodeShape, world: int, rank: int) -> ShardPlan:
    """Contiguous sequence blocks; all heads local (no collective)."""
    if shape.batch % world:
        raise ValueError(f"batch {shape.batch} not divisible by world {world}")
    per = shape.batch // world
    return ShardPlan(shape, world, rank, rank * per, (rank + 1) * per, 0, shape.kv_heads)


def head_shard(shape: DecodeShape, world: int, rank: int) -> ShardPlan:
    """KV-head blocks; with more ranks than KV heads each head's sequences are
    split further (world = kv_heads * batch_groups)."""
    H = shape.kv_heads
    if world <= H:
        if H % world:
            raise ValueError(f"kv_heads {H} not divisible by world {world}")
        per = H // world
        return ShardPlan(shape, world, rank, 0, shape.batch, rank * per, (rank + 1) * per)
    if world % H or shape.batch % (world // H):
        raise ValueError(f"world {world} must be kv_heads x a divisor of batch")
    groups = world // H
    h, g = rank // groups, rank % groups
    per_b = shape.batch // groups
    return ShardPlan(shape, world, rank, g * per_b, (g + 1) * per_b, h, h + 1)


def local_queries(q_layer: torch.Tensor, plan: ShardPlan) -> torch.Tensor:
    """[B, Hq, d] query rows of one layer -> this rank's [units_per_layer, G, d]."""
    G = plan.shape.group
    q = q_layer[plan.b0 : plan.b1, plan.h0 * G : plan.h1 * G]
    return q.reshape(plan.batch * plan.kv_heads, G, q_layer.shape[-1]).contiguous()


def gather_head_outputs(local_out: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    """All-gather one layer's attention output.

    local_out: [units_per_layer, G, d] in this rank's (sequence, head) order.
    Returns the full [B, Hq, d] on every rank (GQA head order hq = h*G + g)."""
    import torch.distributed as dist

    S = plan.shape
    G, d = S.group, local_out.shape[-1]
    blk = local_out.reshape(plan.batch, plan.kv_heads, G, d).contiguous()
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((plan.world,) + tuple(blk.shape), dtype=blk.dtype, device=blk.device)
        dist.all_gather_into_tensor(buf, blk, group=group)
        parts = list(buf.unbind(0))
    else:
        parts = [torch.empty_like(blk) for _ in range(plan.world)]
        dist.all_gather(parts, blk, group=group)
    full = torch.empty((S.batch, S.kv_heads, G, d), dtype=blk.dtype, device=blk.device)
    for r, part in enumerate(parts):
        p = plan_for(S, plan.world, r, head=True)
        full[p.b0 : p.b1, p.h0 : p.h1] = part
    return full.reshape(S.batch, S.q_heads, d)


def plan_for(shape: DecodeShape, world: int, rank: int, head: bool) -> ShardPlan:
    return head_shard(shape, world, rank) if head else batch_shard(shape, world, rank)


class PeerGather:
    """Gathered per-layer outputs [2, L, B, Hq, d] shared by the ranks of one node.

    Every rank allocates its own buffer and a flag array [L, world] (uint32,
    zero), then all ranks exchange CUDA IPC handles (torch's CUDA tensor
    reduction, sent through ``dist.all_gather_object``) and open each other's
    buffers, so the decode epilogue can store into all of them directly.

    Steps alternate between two buffers (``parity``).  Step k's decode writes
    buffer k % 2 of every peer once the writing rank has seen step k - 1
    complete on all ranks, i.e. once every rank's stream has run its step k - 1
    decodes -- and with them anything it enqueued before them that reads step
    k - 2's outputs (buffer k % 2).  Contract: a rank consumes step k's
    outputs (``out[k % 2]``) on its decode stream before it enqueues step
    k + 2's decode.  With one buffer a fast rank's step k + 1 stores could
    overwrite rows a slow rank had not yet read."""

    def __init__(self, plan: ShardPlan, device, group=None, dtype=torch.bfloat16) -> None:
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        S = plan.shape
        if plan.world > 8:
            raise ValueError("peer gather supports up to 8 ranks")
        self.plan, self.dtype = plan, dtype
        self.out = torch.zeros((2, S.layers, S.batch, S.q_heads, S.head_dim), dtype=dtype, device=device)
        self.flags = torch.zeros((S.layers, plan.world), dtype=torch.int32, device=device)  # counts, peers add
        self.expect = torch.zeros(S.layers, dtype=torch.int32, device=device)  # this rank's per-layer count
        self.parity = 0
        torch.cuda.synchronize(device)
        mine = (reduce_tensor(self.out), reduce_tensor(self.flags))
        handles = [None] * plan.world
        dist.all_gather_object(handles, mine, group=group)
        self.peer_out, self.peer_flags = [], []
        for r, (ho, hf) in enumerate(handles):
            if r == plan.rank:
                self.peer_out.append(self.out)
                self.peer_flags.append(self.flags)
            else:
                self.peer_out.append(ho[0](*ho[1]))
                self.peer_flags.append(hf[0](*hf[1]))
        self._desc = [[self._descriptor(p, layer) for layer in range(S.layers)] for p in range(2)]

    def next_step(self) -> int:
        """Start a step: flip to the other buffer; returns its parity."""
        self.parity ^= 1
        return self.parity

    def descriptor(self, layer: int, parity: int | None = None):
        return self._desc[self.parity if parity is None else parity][layer]

    def gathered(self, layer: int, parity: int | None = None) -> torch.Tensor:
        return self.out[self.parity if parity is None else parity, layer]

    def _descriptor(self, parity: int, layer: int):
        from . import _lib
        from ._device import dtype_code

        p, S = self.plan, self.plan.shape
        d = _lib.PqbPeerOut()
        for k in range(p.world):
            d.out[k] = self.peer_out[k][parity, layer].data_ptr()
            d.flags[k] = self.peer_flags[k][layer].data_ptr()
        d.n_peers, d.rank = p.world, p.rank
        d.batch0, d.head0, d.kv_local, d.q_heads = p.b0, p.h0, p.kv_heads, S.q_heads
        d.out_dtype = dtype_code(self.out)
        return d

    def wait(self, layer: int) -> None:
        """Enqueue the wait for every rank's layer output (replay-safe: counts)."""
        from . import _lib
        from ._device import ptr, stream_ptr

        _lib.call("pqb_peer_wait", ptr(self.flags[layer]), self.plan.world, self.plan.rank, ptr(self.expect[layer:]),
                  stream_ptr(self.out.device))


class HeadShardedDecoder:
    """Per-rank decode over a head-sharded cache + the per-layer head gather.

    ``cache`` is this rank's PolarKVCache holding plan.n_units units in
    plan.unit_index order; ``step(q)`` runs all layers for q [L, B, Hq, d] and
    returns the gathered [L, B, Hq, d] outputs.  gather = "nccl" (decode, then
    the collective) or "p2p" (fused into the decode epilogue, PeerGather)."""

    def __init__(self, cache, plan: ShardPlan, group=None, out_dtype=torch.bfloat16, gather: str = "nccl") -> None:
        if gather not in ("nccl", "p2p"):
            raise ValueError(f"gather must be 'nccl' or 'p2p', got {gather!r}")
        self.cache, self.plan, self.group = cache, plan, group
        upl = plan.units_per_layer
        self.views = [cache.view(layer * upl, (layer + 1) * upl) for layer in range(plan.shape.layers)]
        self.out_dtype = out_dtype
        self.gather = gather
        self.peers = PeerGather(plan, cache.device, group, out_dtype) if gather == "p2p" else None

    def layer(self, layer: int, q_layer: torch.Tensor, wait: bool = True) -> torch.Tensor:
        """One layer of the current step (p2p: into buffer ``peers.parity``;
        call ``begin_step()`` before a step's first layer).  The p2p result is
        a view of the shared buffer, valid until the step after next."""
        q_loc = local_queries(q_layer, self.plan)
        if self.peers is not None:
            self.views[layer].decode_peer(q_loc, self.peers.descriptor(layer))
            if wait:
                self.peers.wait(layer)
            return self.peers.gathered(layer)
        local = self.views[layer].decode(q_loc, out_dtype=self.out_dtype)
        return gather_head_outputs(local, self.plan, self.group)

    def begin_step(self) -> None:
        if self.peers is not None:
            self.peers.next_step()

    def step(self, q: torch.Tensor) -> torch.Tensor:
        """All layers for q [L, B, Hq, d]; returns a fresh [L, B, Hq, d]
        (copied on the decode stream, as the double-buffer contract needs)."""
        self.begin_step()
        return torch.stack([self.layer(layer, q[layer]) for layer in range(self.plan.shape.layers)])

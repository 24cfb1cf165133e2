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


class _DeviceArray:
    """__cuda_array_interface__ view of raw device memory (torch.as_tensor wraps it)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str) -> None:
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (ptr, False),
                                         "strides": None, "version": 3}


def peer_gather_supported(device, world_devices) -> bool:
    """True when ``device`` can store into every device in ``world_devices``
    (the fused gather's peer stores; NVLink/NVSwitch boxes: all pairs)."""
    from . import _lib
    import ctypes

    dev = torch.device(device).index or 0
    for other in world_devices:
        can = _lib.c_i32(0)
        _lib.call("pqb_peer_access", dev, int(other), ctypes.byref(can))
        if not can.value:
            return False
    return True


class PeerGather:
    """Gathered per-layer outputs [2, L, B, Hq, d] shared by the ranks of one node.

    Every rank allocates its own buffer and a flag array [L, world] (uint32,
    zero) with ``pqb_ipc_alloc`` (plain cudaMalloc, so the IPC handle names
    the allocation), the ranks exchange the handles (``dist.all_gather_object``)
    and each maps the others' buffers into ITS OWN device's address space with
    ``pqb_ipc_open`` (peer access enabled on first use), so the decode
    epilogue running on that device can store into all of them over NVLink.

    Steps alternate between two buffers (``parity``).  Step k's decode writes
    buffer k % 2 of every peer once the writing rank has seen step k - 1
    complete on all ranks, i.e. once every rank's stream has run its step k - 1
    decodes -- and with them anything it enqueued before them that reads step
    k - 2's outputs (buffer k % 2).  Contract: a rank consumes step k's
    outputs (``out[k % 2]``) on its decode stream before it enqueues step
    k + 2's decode.  With one buffer a fast rank's step k + 1 stores could
    overwrite rows a slow rank had not yet read.  ``close()`` (collective)
    unmaps the peers' buffers and frees this rank's."""

    def __init__(self, plan: ShardPlan, device, group=None, dtype=torch.bfloat16) -> None:
        import ctypes

        import torch.distributed as dist

        from . import _lib

        S = plan.shape
        if plan.world > 8:
            raise ValueError("peer gather supports up to 8 ranks")
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"peer gather outputs are bf16 or fp32, got {dtype}")
        self.plan, self.dtype, self.group = plan, dtype, group
        self.device = torch.device(device)
        self.dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
        out_shape = (2, S.layers, S.batch, S.q_heads, S.head_dim)
        esz = 2 if dtype == torch.bfloat16 else 4
        self._out_bytes = 2 * S.layers * S.batch * S.q_heads * S.head_dim * esz
        self._layer_bytes = S.batch * S.q_heads * S.head_dim * esz
        self._flag_bytes = S.layers * plan.world * 4
        torch.cuda.synchronize(self.device)
        # every rank must reach every other rank's device (collective verdict, so
        # all ranks raise together and a caller can fall back to the NCCL gather)
        devs = [None] * plan.world
        dist.all_gather_object(devs, self.dev, group=group)
        ok = [None] * plan.world
        dist.all_gather_object(ok, peer_gather_supported(self.device, set(devs)), group=group)
        if not all(ok):
            raise RuntimeError(f"peer gather: no P2P access between the ranks' devices {devs}")
        self._own = []  # (ptr) allocated here, freed by close()
        self._opened = []  # peer mappings, unmapped by close()
        mine = []
        for nbytes in (self._out_bytes, self._flag_bytes):
            p, h = ctypes.c_void_p(), ctypes.create_string_buffer(_lib.PQB_IPC_HANDLE_BYTES)
            _lib.call("pqb_ipc_alloc", self.dev, nbytes, ctypes.byref(p), h)
            self._own.append(p.value)
            mine.append(h.raw)
        raw_out = torch.as_tensor(_DeviceArray(self._own[0], (self._out_bytes // esz,), "<i2" if esz == 2 else "<f4"),
                                  device=self.device)
        self.out = (raw_out.view(torch.bfloat16) if esz == 2 else raw_out).view(out_shape)
        self.flags = torch.as_tensor(_DeviceArray(self._own[1], (S.layers, plan.world), "<i4"),
                                     device=self.device)  # counts, peers add
        self.expect = torch.zeros(S.layers, dtype=torch.int32, device=self.device)  # this rank's per-layer count
        self.parity = 0
        handles = [None] * plan.world
        dist.all_gather_object(handles, mine, group=group)
        self.peer_out, self.peer_flags = [], []  # raw base pointers on this device
        err = ""
        try:
            for r, (ho, hf) in enumerate(handles):
                if r == plan.rank:
                    self.peer_out.append(self._own[0])
                    self.peer_flags.append(self._own[1])
                    continue
                ptrs = []
                for h in (ho, hf):
                    p = ctypes.c_void_p()
                    _lib.call("pqb_ipc_open", self.dev, ctypes.create_string_buffer(h, len(h)), ctypes.byref(p))
                    self._opened.append(p.value)
                    ptrs.append(p.value)
                self.peer_out.append(ptrs[0])
                self.peer_flags.append(ptrs[1])
        except (RuntimeError, ValueError) as exc:
            err = str(exc)
        # every rank must have mapped every peer, or none uses the fused gather
        errs = [None] * plan.world
        dist.all_gather_object(errs, err, group=group)
        if any(errs):
            for p in self._opened:
                _lib.load().pqb_ipc_close(self.dev, p)
            dist.barrier(group=group)  # every importer has unmapped before the owners free
            self.out = self.flags = None
            for p in self._own:
                _lib.load().pqb_ipc_free(self.dev, p)
            self._opened, self._own = [], []
            raise RuntimeError(f"peer gather: mapping the peers' buffers failed: {[e for e in errs if e][0]}")
        self._desc = [[self._descriptor(p, layer) for layer in range(S.layers)] for p in range(2)]

    def close(self) -> None:
        """Collective: unmap the peers' buffers, then free this rank's own
        (every rank must have unmapped it first)."""
        import torch.distributed as dist

        from . import _lib

        if not self._own:
            return
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for p in self._opened:
            _lib.call("pqb_ipc_close", self.dev, p)
        self._opened = []
        dist.barrier(group=self.group)
        self.out = self.flags = None
        for p in self._own:
            _lib.call("pqb_ipc_free", self.dev, p)
        self._own = []

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
            d.out[k] = self.peer_out[k] + (parity * S.layers + layer) * self._layer_bytes
            d.flags[k] = self.peer_flags[k] + layer * p.world * 4
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

    def close(self) -> None:
        """Collective (p2p): release the shared gather buffers (PeerGather.close)."""
        if self.peers is not None:
            self.peers.close()
            self.peers = None

    def step(self, q: torch.Tensor) -> torch.Tensor:
        """All layers for q [L, B, Hq, d]; returns a fresh [L, B, Hq, d]
        (copied on the decode stream, as the double-buffer contract needs)."""
        self.begin_step()
        return torch.stack([self.layer(layer, q[layer]) for layer in range(self.plan.shape.layers)])

"""Sharding layer for one node of B200s (one process per GPU, torch.distributed).

Partition rule = the reference's `_chunks` (pmx/interp.py:273-276): rank r of W
owns elements [r*n//W, (r+1)*n//W).  Independent elements (map, map2, loop,
RK4 parameters, k-NN queries, HMM signals) need no collective.  A reduce folds
each shard from `acc` (as each reference chunk does, interp.py:332-333), then
the per-rank partials are exchanged with ONE all-gather and folded left in
rank order (interp.py:334-336) — deterministic and identical on every rank.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def chunk(n: int, world: int, rank: int) -> tuple[int, int]:
    return rank * n // world, (rank + 1) * n // world


def chunks(n: int, world: int) -> list[tuple[int, int]]:
    """Non-empty chunks only, as in the reference."""
    return [(lo, hi) for lo, hi in (chunk(n, world, i) for i in range(world)) if lo < hi]


def world_rank() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def local_slice(x, world: Optional[int] = None, rank: Optional[int] = None):
    """This rank's contiguous shard of a host or device sequence."""
    w, r = world_rank()
    world = w if world is None else world
    rank = r if rank is None else rank
    lo, hi = chunk(len(x), world, rank)
    return x[lo:hi]


def gather_partials(partial: torch.Tensor) -> torch.Tensor:
    """All-gather one partial per rank, in rank order: one collective (NCCL on
    GPUs; gloo in the CPU tests)."""
    w, _ = world_rank()
    flat = partial.reshape(-1).contiguous()
    if w == 1:
        return flat.reshape(1, -1)
    if dist.get_backend() == "nccl":
        out = torch.empty((w, flat.numel()), dtype=flat.dtype, device=flat.device)
        dist.all_gather_into_tensor(out, flat)
        return out
    parts = [torch.empty_like(flat) for _ in range(w)]
    dist.all_gather(parts, flat)
    return torch.stack(parts)


def nonempty_ranks(n: int, world: int) -> list[int]:
    return [r for r in range(world) if chunk(n, world, r)[0] < chunk(n, world, r)[1]]


def ordered_fold(partials: list, ranks: list[int], fold2: Callable):
    """Left fold of the non-empty ranks' partials in rank order
    (interp.py:334-336; empty chunks are dropped, interp.py:276)."""
    total = None
    for r in ranks:
        v = partials[r]
        total = v if total is None else fold2(total, v)
    return total


class PeerMailboxes:
    """Every rank's reduce mailbox mapped into this process (CUDA IPC over
    NVLink): the handles are exchanged once through the process group, after
    which reduce partials move GPU to GPU inside the reduce kernel
    (pmx_map_reduce_peers), with no collective call per reduction."""

    def __init__(self):
        import ctypes as C
        from . import _lib
        self.world, self.rank = world_rank()
        lib = self.lib = _lib.load()
        own = C.c_void_p()
        handle = (C.c_uint8 * _lib.IPC_HANDLE_BYTES)()
        _lib.check(lib.pmx_peer_mailbox_create(C.byref(own), handle), "peer mailbox")
        self.own = own.value
        handles = [bytes(handle)]
        if self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(handle))
        self.opened = []
        self.group = _lib.PeerGroup()
        self.group.rank, self.group.world, self.group.epoch = self.rank, self.world, 0
        for r, h in enumerate(handles):
            if r == self.rank:
                self.group.mbox[r] = self.own
                continue
            p = C.c_void_p()
            buf = (C.c_uint8 * _lib.IPC_HANDLE_BYTES).from_buffer_copy(h)
            _lib.check(lib.pmx_peer_open(buf, C.byref(p)), f"peer open (rank {r})")
            self.group.mbox[r] = p.value
            self.opened.append(p.value)

    def next(self):
        """The group for the next exchange (epoch + 1, same on every rank)."""
        self.group.epoch += 1
        return self.group

    def close(self):
        for p in self.opened:
            self.lib.pmx_peer_close(p)
        self.opened = []
        if self.own:
            self.lib.pmx_peer_mailbox_destroy(self.own)
            self.own = None


class ShardedMapReduce:
    """reduce op acc (map f s) over a sequence sharded across the ranks.

    Each rank launches the fused device kernel on its shard (folding from
    `acc`, like each reference chunk), the per-rank partials are all-gathered
    (one NCCL call) and folded in rank order on the device."""

    def __init__(self, f, op, acc, local_seq, n_global: int, ctx=None, peers: Optional[PeerMailboxes] = None):
        from .skeletons import PreparedMapReduce
        self.world, self.rank = world_rank()
        self.ranks = nonempty_ranks(n_global, self.world)
        self.prep = PreparedMapReduce(f, op, acc, local_seq, ctx)
        self.op = op
        # fused peer-memory combine when the operator pair has a templated
        # kernel and the mailboxes are mapped; else one all-gather + fold
        self.peers = peers if (peers is not None and self.world > 1 and self.prep.has_peer_kernel()) else None

    def launch(self) -> torch.Tensor:
        if self.peers is not None:
            return self.prep.launch_peers(self.peers)   # one kernel: shard + exchange + fold
        part = self.prep.launch()                 # this shard (from acc)
        if self.world == 1:
            return part
        g = gather_partials(part).reshape(-1)
        if len(self.ranks) == self.world:
            return self.prep.fold_partials(g)     # device, rank order
        # n < world: some chunks are empty (tiny inputs); compact the non-empty
        # partials with device-to-device copies, then fold them in rank order
        packed = torch.empty(len(self.ranks), dtype=g.dtype, device=g.device)
        for i, r in enumerate(self.ranks):
            packed[i:i + 1].copy_(g[r:r + 1])
        return self.prep.fold_partials(packed)

"""Sharding layer for one node of B200s (one process per GPU, torch.distributed).

Partition rule = the reference's `_chunks` (pmx/interp.py:273-276): rank r of W
owns elements [r*n//W, (r+1)*n//W).  Independent elements (map, map2, loop,
RK4 parameters, k-NN queries, HMM / k-mer / Viterbi signals) need no
collective: `ShardedMap`, `ShardedMap2`, `ShardedLoop` and the `sharded_*`
case-study entry points run each rank's shard through the single-GPU
operators, with element / iteration indices kept global.

A reduce applies `acc` once, on rank 0 (the single-GPU semantics: the N = 1
and N > 1 results agree for any associative operator): rank 0 folds its shard
from `acc`, every other rank folds its shard alone (from the operator's
identity when the library recognises it, else from the shard's first
element), and the partials fold left in rank order (interp.py:334-336) —
fused into the reduce kernel over NVLink peer memory (`PeerMailboxes`), or
one all-gather + a device fold.  Deterministic and identical on every rank.
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


# identities of the operators the library recognises (pmx_program_kind role 1,
# csrc/jit.h FastKind): folding a shard from one of these equals folding it alone
_IDENTITY = {10: -0.0, 11: 1.0, 12: float("inf"), 13: float("-inf"),
             20: 0, 21: 1, 22: (1 << 63) - 1, 23: -(1 << 63)}


def _global_index_lam(f, n_params: int, lo: int, index_pos: int):
    """f with its `index_pos`-th parameter (the element / iteration index) made
    global: lam(a.., i..) -> lam(a.., _g) let i = _g + lo in body."""
    from . import lambdas as L
    fl = L.as_lam(f)
    if lo == 0 or len(fl.params) <= index_pos:
        return fl
    params = list(fl.params)
    name = params[index_pos]
    params[index_pos] = f"_gidx_{name}"
    return L.Lam(params, L.let(name, L.addi(L.Var(params[index_pos]), lo), fl.body))


def _local_seq(x, lo: int, hi: int):
    """Rows [lo, hi) of a device sequence (or host / torch array) as a device sequence."""
    from .runtime import DeviceSeq, seq_to_device
    from .skeletons import _materialize
    x = _materialize(x)
    if isinstance(x, DeviceSeq):
        if x.offsets is not None:
            raise ValueError("sharding an irregular nested sequence is not supported")
        row = 1
        for d in x.shape[1:]:
            row *= d
        return DeviceSeq(x.data[lo * row:hi * row], (hi - lo,) + tuple(x.shape[1:]), x.dtype_code,
                         elem_tag=x.elem_tag)
    return seq_to_device(x[lo:hi])


class ShardedMap:
    """map f s over a sequence of n_global elements sharded by _chunks: each rank
    maps its own rows [lo, hi) (no collective).  `s` is this rank's shard
    (local=True) or the whole sequence (sliced here).  The element index a
    two-parameter lambda receives is global."""

    def __init__(self, f, s, n_global: Optional[int] = None, *, local: bool = False, ctx=None):
        self.world, self.rank = world_rank()
        n_global = len(s) if n_global is None else n_global
        self.lo, self.hi = chunk(n_global, self.world, self.rank)
        self.seq = _local_seq(s, 0, self.hi - self.lo) if local else _local_seq(s, self.lo, self.hi)
        self.f = _global_index_lam(f, 2, self.lo, 1)
        self.ctx = ctx

    def launch(self):
        """This rank's y[lo:hi] (a device sequence)."""
        from .skeletons import _materialize, eval_map
        return _materialize(eval_map(self.f, self.seq, self.ctx))

    def gather(self, local) -> torch.Tensor:
        return gather_rows(local.data, self.hi - self.lo)


class ShardedMap2:
    """map2 f s1 s2 sharded by _chunks (no collective); the lengths must agree
    globally (interp.py:151-154)."""

    def __init__(self, f, s1, s2, *, ctx=None):
        from .diagnostics import runtime_error
        if len(s1) != len(s2):
            raise runtime_error(f"map2 over sequences of different lengths ({len(s1)} and {len(s2)})")
        self.world, self.rank = world_rank()
        self.lo, self.hi = chunk(len(s1), self.world, self.rank)
        self.s1, self.s2 = _local_seq(s1, self.lo, self.hi), _local_seq(s2, self.lo, self.hi)
        self.f = _global_index_lam(f, 3, self.lo, 2)
        self.ctx = ctx

    def launch(self):
        from .skeletons import eval_map2
        return eval_map2(self.f, self.s1, self.s2, self.ctx)


class ShardedLoop:
    """loop n f (interp.py:346-358) with the iterations [0, n) sharded by _chunks:
    rank r runs f(i) for its global i in [lo, hi) (no collective).  The body's
    tensors are views of this rank's device memory; iterations must write
    disjoint elements, as the reference's parallel loop requires."""

    def __init__(self, n: int, f, *, ctx=None):
        self.world, self.rank = world_rank()
        self.lo, self.hi = chunk(int(n), self.world, self.rank)
        self.f = _global_index_lam(f, 1, self.lo, 0)
        self.ctx = ctx

    def launch(self) -> dict:
        from .skeletons import eval_loop
        return eval_loop(self.hi - self.lo, self.f, self.ctx)


class ShardedMapReduce:
    """reduce op acc (map f s) over a sequence sharded across the ranks, with
    `acc` applied once (rank 0), so the result equals the single-GPU one.

    Rank 0 folds its shard from `acc`; rank r > 0 folds its shard from the
    operator's identity (recognised operators) or from its first element (any
    other operator: f(x[lo]) is read once at construction).  The partials fold
    left in rank order — in the reduce kernel itself over NVLink peer memory
    when `peers` is given and the operator pair has a fused kernel, else by one
    all-gather and a device fold.  `local_seq` is this rank's shard."""

    def __init__(self, f, op, acc, local_seq, n_global: int, ctx=None, peers: Optional[PeerMailboxes] = None):
        from .skeletons import NO_SPAN, PreparedMapReduce, _compile
        import ctypes as C
        from . import _lib
        self.world, self.rank = world_rank()
        n_local = len(local_seq)
        # rank 0 always contributes (it carries acc); others only when non-empty
        self.ranks = [0] + [r for r in nonempty_ranks(n_global, self.world) if r != 0]
        self.op = op
        f_g = _global_index_lam(f, 2, chunk(n_global, self.world, self.rank)[0], 1) if f is not None else None
        acc_t = "float" if isinstance(acc, float) else "int"
        kind = _lib.load().pmx_program_kind(C.byref(_compile(op, [acc_t, acc_t], NO_SPAN).program), 1)
        seq, init = local_seq, acc
        if self.rank > 0 and n_local > 0:
            if kind in _IDENTITY:
                init = _IDENTITY[kind]
            else:
                init, seq = self._first(f_g, local_seq, acc_t), _local_seq(local_seq, 1, n_local)
        self.prep = PreparedMapReduce(f_g, op, init, seq, ctx)
        # fused peer-memory combine when the operator pair has a templated
        # kernel and the mailboxes are mapped; else one all-gather + fold
        self.peers = peers if (peers is not None and self.world > 1 and self.prep.has_peer_kernel()) else None

    @staticmethod
    def _first(f, s, acc_t):
        """f(s[0]) read to the host: a shard's fold without acc starts from it."""
        from .skeletons import _materialize, eval_map
        one = _local_seq(s, 0, 1)
        v = (_materialize(eval_map(f, one)) if f is not None else one).data[:1].to("cpu").item()
        return float(v) if acc_t == "float" else int(v)

    def launch(self) -> torch.Tensor:
        if self.peers is not None:
            return self.prep.launch_peers(self.peers)   # one kernel: shard + exchange + fold
        part = self.prep.launch()                 # this shard's partial
        if self.world == 1:
            return part
        g = gather_partials(part).reshape(-1)
        if len(self.ranks) == self.world:
            return self.prep.fold_partials(g)     # device, rank order
        # n < world: some chunks are empty (tiny inputs); compact the contributing
        # partials with device-to-device copies, then fold them in rank order
        packed = torch.empty(len(self.ranks), dtype=g.dtype, device=g.device)
        for i, r in enumerate(self.ranks):
            packed[i:i + 1].copy_(g[r:r + 1])
        return self.prep.fold_partials(packed)


def gather_rows(local: torch.Tensor, n_local: int) -> torch.Tensor:
    """All ranks' shards of a sharded result concatenated in rank order (the
    global result on every rank): one all-gather of equal-size padded blocks."""
    w, _ = world_rank()
    flat = local.reshape(n_local, -1) if n_local else local.reshape(0, max(1, local.numel()))
    if w == 1:
        return flat
    sizes = [None] * w
    dist.all_gather_object(sizes, int(n_local))
    m = max(sizes)
    buf = torch.zeros((m, flat.shape[1]), dtype=flat.dtype, device=flat.device)
    buf[:n_local].copy_(flat)
    if dist.get_backend() == "nccl":
        out = torch.empty((w, m, flat.shape[1]), dtype=flat.dtype, device=flat.device)
        dist.all_gather_into_tensor(out.reshape(-1), buf.reshape(-1))
        parts = [out[r, :sizes[r]] for r in range(w)]
    else:
        bufs = [torch.empty_like(buf.cpu()) for _ in range(w)]
        dist.all_gather(bufs, buf.cpu())
        parts = [bufs[r][:sizes[r]].to(flat.device) for r in range(w)]
    return torch.cat(parts)


# ------------------------------------------------- sharded case studies
# Each runs this rank's _chunks shard of the independent elements through the
# single-GPU entry point (model / train data replicated); no collective.

def _shard_rows(x):
    w, r = world_rank()
    lo, hi = chunk(len(x), w, r)
    return x[lo:hi]


def sharded_rk4_sweep(params, init4, steps: int, h: float):
    """rk4_sweep over this rank's parameter sets (programs/rk4.pmx:42-45)."""
    from .casestudies import rk4_sweep
    return rk4_sweep(_shard_rows(params), init4, steps, h)


def sharded_knn_classify(train, labels, queries, k: int, ncls: int, return_indices: bool = False):
    """knn_classify of this rank's queries against the replicated train set."""
    from .casestudies import knn_classify
    return knn_classify(train, labels, _shard_rows(queries), k, ncls, return_indices=return_indices)


def sharded_hmm_forward(trans, emit, init, obs):
    """hmm_forward of this rank's signals (model replicated)."""
    from .casestudies import hmm_forward
    return hmm_forward(trans, emit, init, _shard_rows(obs))


def sharded_hmm_kmer_forward(kmer: int, p_stay: float, p_step: float, emit, obs):
    """hmm_kmer_forward of this rank's signals (the nanopore config: 8k signals over 8 GPUs)."""
    from .casestudies import hmm_kmer_forward
    return hmm_kmer_forward(kmer, p_stay, p_step, emit, _shard_rows(obs))


def sharded_viterbi(trans, emit, init, obs):
    """viterbi of this rank's signals (programs/viterbi.pmx:23-59)."""
    from .casestudies import viterbi
    return viterbi(trans, emit, init, _shard_rows(obs))

"""Host logic of the sharded (N > 1) path with world_size 2 gloo on CPU:
partition rule, rank-ordered gather of partials, reference fold order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_00621_b200 import shard


def test_chunk_rule_matches_reference():
    # _chunks (pmx/interp.py:273-276): i*n//w .. (i+1)*n//w, empties dropped
    assert shard.chunks(10, 4) == [(0, 2), (2, 5), (5, 7), (7, 10)]
    assert shard.chunks(2, 4) == [(0, 1), (1, 2)]
    assert shard.nonempty_ranks(2, 4) == [1, 3]
    assert shard.chunks(3, 8) == [(0, 1), (1, 2), (2, 3)]
    for n in range(0, 40):
        for w in range(1, 9):
            spans = [shard.chunk(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_ordered_fold_is_left_fold_in_rank_order():
    parts = [100, 1, 2, 3]
    assert shard.ordered_fold(parts, [0, 1, 2, 3], lambda a, b: a - b) == 94
    assert shard.ordered_fold(parts, [1, 3], lambda a, b: a - b) == -2


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys, pathlib
        sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "oracle"))
        import oracle as O
        from paper_2211_00621_b200.lambdas import addi, lam, muli, subi
        n = 1000
        xs = list(range(n))
        local = shard.local_slice(xs)
        lo, hi = shard.chunk(n, world, rank)
        assert local == xs[lo:hi]
        # each shard folds from acc like a reference chunk (interp.py:332-333)
        f = lam("x", muli("x", "x"))
        part = O.ir_fold(addi, 0, O.ir_map(f, local))
        g = shard.gather_partials(torch.tensor([part], dtype=torch.int64)).reshape(-1).tolist()
        total = shard.ordered_fold(g, shard.nonempty_ranks(n, world), lambda a, b: O.ir_apply(addi, a, b))
        want = O.ir_reduce(addi, 0, O.ir_map(f, xs), workers=world)
        # non-associative operator: the rank-order fold reproduces the reference's
        # chunked result with workers = world
        part2 = O.ir_fold(subi, 7, local)
        g2 = shard.gather_partials(torch.tensor([part2], dtype=torch.int64)).reshape(-1).tolist()
        total2 = shard.ordered_fold(g2, shard.nonempty_ranks(n, world), lambda a, b: O.ir_apply(subi, a, b))
        want2 = O.ir_reduce(subi, 7, xs, workers=world)
        q.put((rank, total == want, total2 == want2, g))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_reduce_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok1 and ok2 for _, ok1, ok2, _ in res)
    # every rank saw the same gathered partials (rank order)
    assert len({tuple(g) for *_, g in res}) == 1


def test_global_index_lambdas():
    # ShardedMap / ShardedMap2 / ShardedLoop keep element and iteration indices
    # global: the shard's local index j becomes lo + j (checked with the oracle's
    # evaluator of the lambda IR)
    import sys, pathlib
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "oracle"))
    import oracle as O
    from paper_2211_00621_b200.lambdas import addi, lam, muli
    f = lam("x", "i", addi(muli("x", 10), "i"))
    g = shard._global_index_lam(f, 2, 37, 1)
    assert [O.ir_apply(g, 3, j) for j in range(4)] == [30 + 37 + j for j in range(4)]
    assert shard._global_index_lam(f, 2, 0, 1) is not None
    body = lam("i", muli("i", 2))
    assert O.ir_apply(shard._global_index_lam(body, 1, 5, 0), 1) == 12
    # a one-parameter map lambda does not see the index: unchanged
    h = lam("x", muli("x", 3))
    assert O.ir_apply(shard._global_index_lam(h, 2, 99, 1), 4) == 12


def test_identities_of_recognised_operators():
    # rank r > 0 folds its shard from the operator's identity: e (+) x == x for
    # every x the reduce can see (signed zeros, infinities, extreme ints)
    import math
    import sys, pathlib
    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent / "oracle"))
    import oracle as O
    from paper_2211_00621_b200.lambdas import addf, addi, gtf, gti, if_, lam, ltf, lti, mulf, muli
    ops = {10: addf, 11: mulf, 12: lam("a", "b", if_(ltf("a", "b"), "a", "b")),
           13: lam("a", "b", if_(gtf("a", "b"), "a", "b")), 20: addi, 21: muli,
           22: lam("a", "b", if_(lti("a", "b"), "a", "b")), 23: lam("a", "b", if_(gti("a", "b"), "a", "b"))}
    fvals = [0.0, -0.0, 1.5, -2.25, math.inf, -math.inf, 1e308, -5e-324]
    ivals = [0, 1, -1, (1 << 63) - 1, -(1 << 63), 123456789]
    for kind, op in ops.items():
        e = shard._IDENTITY[kind]
        for v in (fvals if kind < 20 else ivals):
            r = O.ir_apply(op, e, v)
            assert r == v and (kind >= 20 or math.copysign(1, r) == math.copysign(1, v)), (kind, v, r)


def _rows_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 11
        lo, hi = shard.chunk(n, world, rank)
        local = torch.arange(lo * 3, hi * 3, dtype=torch.float64).reshape(hi - lo, 3)
        full = shard.gather_rows(local, hi - lo)
        q.put((rank, full.tolist()))
    finally:
        dist.destroy_process_group()


def test_gather_rows_gloo():
    # uneven _chunks shards (n = 11 over 2 ranks: 5 + 6 rows) come back in rank
    # order on every rank
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = torch.arange(33, dtype=torch.float64).reshape(11, 3).tolist()
    assert res[0] == want and res[1] == want

"""Fused peer-memory reduce (pmx_map_reduce_peers) with 2 ranks.

The box has one GPU, so both ranks run on cuda:0 as separate processes: the
mailboxes are still exchanged through CUDA IPC and written with system-scope
release stores / read with acquire loads exactly as across NVLink, so the
protocol (epochs, parity double-buffering, rank-ordered fold, empty shards) is
exercised end to end. Handles travel over a gloo process group."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import time
        import paper_2211_00621_b200 as P
        from paper_2211_00621_b200 import _lib, shard
        from paper_2211_00621_b200.runtime import DeviceSeq
        P.load_library()
        peers = shard.PeerMailboxes()
        out = {}
        rng = np.random.default_rng(7)
        # 1) float sum over non-exact data: total = p0 + p1 (rank order), p0
        #    folded from acc, p1 alone
        n = 1_000_003
        x = rng.standard_normal(n)
        lo, hi = shard.chunk(n, world, rank)
        dx = torch.from_numpy(x[lo:hi].copy()).cuda()
        seq = DeviceSeq(dx, (hi - lo,), _lib.PMX_F64)
        smr = shard.ShardedMapReduce(P.lam("x", P.addf(P.mulf(3.0, "x"), 0.5)), P.addf, 0.0, seq, n, peers=peers)
        assert smr.peers is not None
        vals = []
        for it in range(200):
            if rank == 1 and it % 17 == 0:
                time.sleep(0.01)           # uneven arrival exercises the epoch parity
            vals.append(smr.launch().clone())
        torch.cuda.synchronize()
        out["sum"] = [float(v.item()) for v in vals]
        local = smr.prep.launch().item()   # this rank's chunk partial (collective-free)
        out["local"] = float(local)
        # 2) int product / max, and an empty shard (n < world)
        xi = torch.arange(1, 5, dtype=torch.int64)
        lo, hi = shard.chunk(4, world, rank)
        si = DeviceSeq(xi[lo:hi].cuda(), (hi - lo,), _lib.PMX_I64)
        out["prod"] = int(shard.ShardedMapReduce(None, P.muli, 1, si, 4, peers=peers).launch().item())
        mx = P.lam("a", "b", P.if_(P.gti("a", "b"), "a", "b"))
        out["max"] = int(shard.ShardedMapReduce(P.lam("x", P.addi(P.muli(-2, "x"), 9)), mx, -100, si, 4,
                                                peers=peers).launch().item())
        lo, hi = shard.chunk(1, world, rank)     # rank 0 empty, rank 1 holds the element
        se = DeviceSeq(torch.tensor([41], dtype=torch.int64)[lo:hi].cuda(), (hi - lo,), _lib.PMX_I64)
        out["one"] = int(shard.ShardedMapReduce(None, P.addi, 1, se, 1, peers=peers).launch().item())
        sz = DeviceSeq(torch.empty(0, dtype=torch.int64).cuda(), (0,), _lib.PMX_I64)
        out["none"] = int(shard.ShardedMapReduce(None, P.addi, 5, sz, 0, peers=peers).launch().item())
        # acc applied once (rank 0): N = 1 and N = 2 agree for a non-neutral acc
        out["acc10"] = int(shard.ShardedMapReduce(None, P.addi, 10, si, 4, peers=peers).launch().item())
        lo8, hi8 = shard.chunk(8, world, rank)
        xf = torch.tensor([0.5, -1.25, 2.0, 3.5, -0.75, 8.0, 1.5, 4.0], dtype=torch.float64)
        sf = DeviceSeq(xf[lo8:hi8].cuda(), (hi8 - lo8,), _lib.PMX_F64)
        mnf = P.lam("a", "b", P.if_(P.ltf("a", "b"), "a", "b"))
        out["minf"] = float(shard.ShardedMapReduce(None, mnf, -3.0, sf, 8, peers=peers).launch().item())
        out["mulf"] = float(shard.ShardedMapReduce(None, P.mulf, 2.0, sf, 8, peers=peers).launch().item())
        # an associative operator the library does not recognise (ordered generic
        # tree, collective combine): rank 1 folds from its first element
        gop = P.lam("a", "b", P.addi("a", P.muli("b", 1)))
        g = shard.ShardedMapReduce(P.lam("x", P.muli("x", "x")), gop, 100, si, 4, peers=peers)
        assert g.peers is None
        out["generic"] = int(g.launch().item())
        # generic map (run-time specialised kernel) with the peer combine
        sq = shard.ShardedMapReduce(P.lam("x", P.mulf("x", "x")), P.addf, 0.0, seq, n, peers=peers)
        out["sq"] = float(sq.launch().item())
        out["sq_local"] = float(sq.prep.launch().item())
        P.skeletons.default_ctx().check_errors()
        torch.cuda.synchronize()
        dist.barrier()
        peers.close()
        q.put((rank, out))
    except Exception as exc:  # report to the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_peer_reduce_two_ranks_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in res[r], res[r]["error"]
    s0, s1 = res[0]["sum"], res[1]["sum"]
    # identical on both ranks, every launch, and = p0 + p1 in rank order
    want = np.float64(res[0]["local"]) + np.float64(res[1]["local"])
    assert all(v == float(want) for v in s0), (s0[:3], want)
    assert s0 == s1
    # product: rank0 1*1*2 ; rank1 3*4 -> 2*12
    assert res[0]["prod"] == res[1]["prod"] == 24
    # max of 9-2x over [1,2] and [3,4] from -100
    assert res[0]["max"] == res[1]["max"] == 7
    # rank 0's shard is empty but it carries acc: 1 + 41
    assert res[0]["one"] == res[1]["one"] == 42
    assert res[0]["sq"] == res[1]["sq"] == res[0]["sq_local"] + res[1]["sq_local"]
    # all chunks empty: reduce over [] returns acc
    assert res[0]["none"] == res[1]["none"] == 5
    # acc once, as on one GPU (the reference's debug semantics, interp.py:329-330)
    assert res[0]["acc10"] == res[1]["acc10"] == 10 + 1 + 2 + 3 + 4
    assert res[0]["minf"] == res[1]["minf"] == -3.0
    assert res[0]["mulf"] == res[1]["mulf"] == 2.0 * 0.5 * -1.25 * 2.0 * 3.5 * -0.75 * 8.0 * 1.5 * 4.0
    assert res[0]["generic"] == res[1]["generic"] == 100 + 1 + 4 + 9 + 16

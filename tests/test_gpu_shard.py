"""Product-level sharding with 2 ranks on one GPU.

Each rank runs its _chunks shard (pmx/interp.py:273-276) of map / map2 / loop
and of the case studies through the sharded entry points; the shards,
concatenated in rank order, must equal the single-GPU result bit for bit, and
element / iteration indices must stay global.  Both ranks share cuda:0 (the
box has one GPU); the process group is gloo."""
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


def _single(fn):
    """Run fn on one GPU as world 1 (before the group exists)."""
    return fn()


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        import paper_2211_00621_b200 as P
        from paper_2211_00621_b200 import _lib, shard, synth
        from paper_2211_00621_b200.runtime import DeviceSeq, DeviceTensor, _Root, seq_to_host
        P.load_library()
        n = 10_007
        x = np.arange(n, dtype=np.float64) * 0.25 - 7.0
        y = np.arange(n, dtype=np.float64)[::-1].copy()
        f = P.lam("v", "i", P.addf(P.mulf("v", "v"), P.int2float("i")))      # uses the global index
        g = P.lam("a", "b", "i", P.subf(P.mulf("a", "b"), P.int2float(P.muli("i", 3))))
        # single-GPU references (world 1: computed before the process group)
        ref = {}
        ref["map"] = seq_to_host(P.skeletons._materialize(P.eval_map(f, x)))
        ref["map2"] = seq_to_host(P.eval_map2(g, x, y))
        A, E, pi = synth.hmm_model(64, 8)
        obs = synth.hmm_obs(37, 20, 8)
        ref["hmm"] = seq_to_host(P.hmm_forward(A, E, pi, obs))
        Xk, Lk, Qk = synth.knn_train(3000, 16), synth.knn_labels(3000, 5), synth.knn_query(301, 16)
        ref["knn"] = seq_to_host(P.knn_classify(Xk, Lk, Qk, 8, 5))
        ps = synth.rk4_params(333)
        ref["rk4"] = seq_to_host(P.rk4_sweep(ps, synth.RK4_INIT, 50, synth.RK4_H))
        vr = P.viterbi(A, E, pi, obs)
        ref["vit"] = seq_to_host(vr["path"])
        Ekm = synth.kmer_emission(4, 8)
        obk = synth.hmm_obs(9, 30, 8)
        ref["kmer"] = seq_to_host(P.hmm_kmer_forward(4, 0.5, 0.125, Ekm, obk))
        ref["red"] = P.eval_reduce(P.addf, 3.5, P.eval_map(P.lam("v", P.mulf(2.0, "v")), x)).get()
        torch.cuda.synchronize()

        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = {"ref": ref}
        # map / map2: this rank's rows, gathered in rank order
        sm = shard.ShardedMap(f, x)
        out["map"] = sm.gather(sm.launch()).reshape(-1).cpu().numpy()
        s2 = shard.ShardedMap2(g, x, y)
        loc = s2.launch()
        out["map2"] = shard.gather_rows(loc.data, s2.hi - s2.lo).reshape(-1).cpu().numpy()
        # loop: every rank writes its iterations i of a full-size output tensor
        yt = torch.zeros(n, dtype=torch.float64, device="cuda")
        xt = torch.from_numpy(x).cuda()
        tx = DeviceTensor(_Root(xt, 0, 0, n, _lib.PMX_F64), 0, (n,), "float")
        ty = DeviceTensor(_Root(yt, 1, 0, n, _lib.PMX_F64), 0, (n,), "float")
        body = P.lam("i", P.tensor_set(ty, ["i"], P.addf(P.tensor_get(tx, ["i"]), P.int2float("i"))))
        sl = shard.ShardedLoop(n, body)
        sl.launch()
        torch.cuda.synchronize()
        mine = yt[sl.lo:sl.hi].clone()
        out["loop"] = shard.gather_rows(mine, sl.hi - sl.lo).reshape(-1).cpu().numpy()
        out["loop_untouched"] = bool(torch.all(torch.cat([yt[:sl.lo], yt[sl.hi:]]) == 0).item())
        # case studies: shards gathered in rank order
        def gath(seq):
            loc = seq.data
            rows = seq.shape[0]
            return shard.gather_rows(loc, rows).cpu().numpy()
        out["hmm"] = gath(shard.sharded_hmm_forward(A, E, pi, obs)).reshape(-1)
        out["knn"] = gath(shard.sharded_knn_classify(Xk, Lk, Qk, 8, 5)).reshape(-1)
        out["rk4"] = gath(shard.sharded_rk4_sweep(ps, synth.RK4_INIT, 50, synth.RK4_H))
        out["vit"] = gath(shard.sharded_viterbi(A, E, pi, obs)["path"])
        out["kmer"] = gath(shard.sharded_hmm_kmer_forward(4, 0.5, 0.125, Ekm, obk)).reshape(-1)
        # sharded fused map -> reduce with a non-neutral acc (collective combine)
        lo, hi = shard.chunk(n, world, rank)
        seq = DeviceSeq(torch.from_numpy(x[lo:hi].copy()).cuda(), (hi - lo,), _lib.PMX_F64)
        out["red"] = float(shard.ShardedMapReduce(P.lam("v", P.mulf(2.0, "v")), P.addf, 3.5, seq, n)
                           .launch().item())
        P.skeletons.default_ctx().check_errors()
        torch.cuda.synchronize()
        dist.barrier()
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_sharded_operators_and_case_studies_match_one_gpu():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in res[r], res[r]["error"]
    for r in range(world):
        o, ref = res[r], res[r]["ref"]
        for key in ("map", "map2", "hmm", "knn", "rk4", "vit", "kmer"):
            assert np.array_equal(np.asarray(o[key]).reshape(-1), np.asarray(ref[key]).reshape(-1)), key
        assert np.array_equal(o["loop"], np.arange(10_007) * 0.25 - 7.0 + np.arange(10_007))
        assert o["loop_untouched"]
        # acc once: equals the single-GPU fold exactly (every partial sum is a
        # dyadic rational well inside fp64, so the grouping does not matter)
        assert o["red"] == ref["red"]

"""Small, fixed launches of each hot kernel for ncu captures.

    ncu --set full --clock-control none --import-source on -k regex:<kernel> -s <skip> -c 1 \
        -o gpurun_out/prof_<case> python tools/profile_cases.py <case>

Sizes are the BASELINE configs except where a persistent kernel's time grows
with the step count (HMM T, k-mer T), where T is reduced so the ~40 ncu
replays stay short; per-step behaviour is unchanged.
"""
from __future__ import annotations

import pathlib
import sys

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2211_00621_b200 as P  # noqa: E402
from paper_2211_00621_b200 import _lib, casestudies as CS, synth  # noqa: E402
from paper_2211_00621_b200.runtime import DeviceSeq  # noqa: E402
from paper_2211_00621_b200.skeletons import PreparedMapReduce, default_ctx  # noqa: E402


def mapreduce(reps=3):
    n = 1 << 28
    x = synth.mapreduce_x_device(n, torch.device("cuda"))
    f = P.lam("x", P.addf(P.mulf(2.0, "x"), 1.0))
    seq = DeviceSeq(x, (n,), _lib.PMX_F32)
    prep = PreparedMapReduce(f, P.addf, 0.0, seq)
    y = torch.empty_like(x)
    pmap = PreparedMapReduce(f, P.addf, 0.0, seq, materialize=y, reduce=False)
    pred = PreparedMapReduce(None, P.addf, 0.0, DeviceSeq(y, (n,), _lib.PMX_F32))
    for _ in range(reps):
        prep.launch()
        pmap.launch()
        pred.launch()
    torch.cuda.synchronize()


def generic(reps=2):
    """Run-time specialised kernels (jit.cu): map / loop on unrecognised lambdas."""
    from paper_2211_00621_b200.runtime import DeviceTensor, _Root
    n = 1 << 28
    x = synth.mapreduce_x_device(n, torch.device("cuda"))
    xs = DeviceSeq(x, (n,), _lib.PMX_F32)
    yt = torch.empty_like(x)
    tx = DeviceTensor(_Root(x, 0, 0, n, _lib.PMX_F32), 0, (n,), "float")
    ty = DeviceTensor(_Root(yt, 1, 0, n, _lib.PMX_F32), 0, (n,), "float")
    f = P.lam("x", P.addf(P.mulf("x", "x"), 1.0))
    body = P.lam("i", P.tensor_set(ty, ["i"], P.addf(P.mulf(2.0, P.tensor_get(tx, ["i"])), 1.0)))
    ms_ = 1 << 24
    s_state = DeviceSeq(torch.arange(ms_, dtype=torch.float64, device="cuda") % 97, (ms_,), _lib.PMX_F64)
    stencil = P.lam("x", "j", "t", P.mulf(0.5, P.addf("x", P.get(P.PREV, P.modi(P.addi("j", 1), ms_)))))
    gop = P.lam("a", "b", P.addf("a", P.mulf("b", 1.0)))
    for _ in range(reps):
        P.eval_map(f, xs).materialize()
        P.eval_loop(n, body)
        P.seq_loop(20, stencil, s_state)
        P.eval_reduce(gop, 0.0, xs)
    torch.cuda.synchronize()


def rk4(reps=2):
    ps = torch.from_numpy(synth.rk4_params(10_000)).cuda()
    s0 = torch.from_numpy(synth.RK4_INIT).cuda()
    for _ in range(reps):
        CS.rk4_sweep(ps, s0, 1000, synth.RK4_H)
    torch.cuda.synchronize()


def hmm(reps=2, T=200):
    S, K, nsig = 1024, 8, 4096
    A, E, pi = synth.hmm_model(S, K)
    Ad = torch.from_numpy(A.astype(np.float32)).cuda()
    lE = torch.from_numpy(np.log(E).astype(np.float32)).cuda()
    lpi = torch.from_numpy(np.log(pi).astype(np.float32)).cuda()
    obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).cuda()
    out = torch.empty(nsig, dtype=torch.float64, device="cuda")
    ws = torch.empty(_lib.load().pmx_hmm_forward_workspace_bytes(S, nsig), dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        CS.hmm_forward_raw(lpi, Ad, lE, obs, S, K, nsig, T, out, ws)
    torch.cuda.synchronize()


def knn(reps=2, ntr=1 << 18):
    nq, d, k, c = 1 << 16, 64, 8, 10
    X = torch.from_numpy(synth.knn_train(ntr, d)).cuda()
    Q = torch.from_numpy(synth.knn_query(nq, d)).cuda()
    L = torch.from_numpy(synth.knn_labels(ntr, c)).cuda()
    out = torch.empty(nq, dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.load().pmx_knn_workspace_bytes(ntr, nq, d, k), dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        CS.knn_raw(X, L, Q, ntr, nq, d, k, c, out, None, ws)
    torch.cuda.synchronize()


def knn_full(reps=1):
    """k-NN at the BASELINE config (2^20 train x 2^16 queries)."""
    knn(reps, ntr=1 << 20)


def kmer(reps=2, T=100):
    km, K, nsig = 8, 8, 1024
    lE = torch.from_numpy(np.log(synth.kmer_emission(km, K)).astype(np.float32)).cuda()
    obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).cuda()
    out = torch.empty(nsig, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    ws = torch.empty(lib.pmx_hmm_kmer_workspace_bytes(km, nsig), dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        _lib.check(lib.pmx_hmm_kmer_forward_f32(km, 0.5, 0.125, lE.data_ptr(), K, obs.data_ptr(), nsig, T,
                                                out.data_ptr(), ws.data_ptr(), ws.numel(),
                                                torch.cuda.current_stream().cuda_stream), "kmer")
    torch.cuda.synchronize()


def viterbi(reps=2, T=100):
    S, K, nsig = 1024, 8, 148 * 8
    A, E, pi = synth.hmm_model(S, K)
    lA, lE, lpi = (torch.from_numpy(np.log(a)).cuda() for a in (A, E, pi))
    obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).cuda()
    path = torch.empty(nsig * T, dtype=torch.int32, device="cuda")
    logp = torch.empty(nsig, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    ws = torch.empty(lib.pmx_viterbi_workspace_bytes(S, nsig, T), dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        _lib.check(lib.pmx_viterbi_f64(lpi.data_ptr(), lA.data_ptr(), lE.data_ptr(), S, K, obs.data_ptr(), nsig, T,
                                       path.data_ptr(), logp.data_ptr(), ws.data_ptr(), ws.numel(),
                                       torch.cuda.current_stream().cuda_stream), "viterbi")
    torch.cuda.synchronize()
    v = lib.pmx_viterbi_visited_cells(ws.data_ptr(), S, nsig, T, torch.cuda.current_stream().cuda_stream)
    print("viterbi visited cells per launch", v, "of", S * S * (T - 1) * nsig)


def nn(reps=2):
    npts, nin, nout = 1 << 20, 64, 16
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(npts * nin, dtype=torch.float64, device="cuda", generator=g) * 0.5
    y = torch.randint(0, nout, (npts,), dtype=torch.int32, device="cuda", generator=g)
    w = torch.randn(nin * nout, dtype=torch.float64, device="cuda", generator=g) * 0.3
    b = torch.randn(nout, dtype=torch.float64, device="cuda", generator=g) * 0.1
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    dw = torch.empty(nin * nout, dtype=torch.float64, device="cuda")
    db = torch.empty(nout, dtype=torch.float64, device="cuda")
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    ws = torch.zeros(lib.pmx_nn_workspace_bytes(npts, nin, nout), dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        _lib.check(lib.pmx_nn_softmax_grad_f64(x.data_ptr(), y.data_ptr(), w.data_ptr(), b.data_ptr(), npts, nin,
                                               nout, loss.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(),
                                               ws.numel(), err.data_ptr(), torch.cuda.current_stream().cuda_stream),
                   "nn")
    torch.cuda.synchronize()


if __name__ == "__main__":
    P.load_library()
    for name in sys.argv[1:] or ["mapreduce"]:
        globals()[name]()
    default_ctx().check_errors()
    print("done", sys.argv[1:])

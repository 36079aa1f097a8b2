"""Case-study kernels on the B200 vs the reference's golden outputs and the
CPU oracle.  Tolerances (north_star): integer/index outputs bit-exact, fp64
rel 1e-9, fp32 rel 1e-5 with log-likelihoods compared in fp64."""
import math
import pathlib

import numpy as np
import pytest
import torch

import oracle as O
import paper_2211_00621_b200 as P
from paper_2211_00621_b200 import (
    accelerate, hmm_forward, hmm_kmer_forward, knn_classify, rk4_sweep, synth, viterbi,
)

pytestmark = pytest.mark.gpu

FP64_REL = 1e-9
LL_REL = 1e-5


# ------------------------------------------------------------------ RK4
def test_rk4_reference_program(golden):
    # programs/rk4.pmx: p_k = 0.5 + 0.1k, k < 16, 100 steps (test_acceptance.py:385-394)
    ps = np.array([0.5 + 0.1 * float(k) for k in range(16)])
    got = accelerate(lambda p, s0: rk4_sweep(p, s0, 100, 0.01), ps, synth.RK4_INIT)
    lines = [l for l in golden["program_rk4"]["stdout"].splitlines() if l.strip()]
    assert got.shape == (16, 4)
    for k, line in enumerate(lines):
        for g, w in zip(got[k], map(float, line.split())):
            assert math.isclose(g, w, rel_tol=FP64_REL), (k, g, w)


def test_rk4_param_variant_golden(golden):
    for e in golden["rk4_param"]:
        got = accelerate(lambda p, s0: rk4_sweep(p, s0, e["M"], 0.01), synth.rk4_params(e["N"]), synth.RK4_INIT)
        lines = [l for l in e["stdout"].splitlines() if l.strip()]
        for k, line in enumerate(lines):
            for g, w in zip(got[k], map(float, line.split())):
                assert math.isclose(g, w, rel_tol=FP64_REL)


def test_rk4_vs_oracle_config_steps():
    n = 2000
    ps = synth.rk4_params(n)
    got = accelerate(lambda p, s0: rk4_sweep(p, s0, 1000, synth.RK4_H), ps, synth.RK4_INIT)
    want = O.rk4(ps, synth.RK4_INIT, 1000, synth.RK4_H)
    assert np.allclose(got, want, rtol=FP64_REL, atol=1e-12)


@pytest.mark.parametrize("m", [0, 1, 7, 33])
def test_rk4_odd_and_short_step_counts(m):
    # two steps per straight-line block plus a single-step tail (csrc/rk4.cu)
    ps = synth.rk4_params(257)
    got = accelerate(lambda p, s0: rk4_sweep(p, s0, m, synth.RK4_H), ps, synth.RK4_INIT)
    want = O.rk4(ps, synth.RK4_INIT, m, synth.RK4_H)
    assert np.allclose(got, want, rtol=FP64_REL, atol=1e-12)


def test_rk4_angles_outside_the_fast_reduction_range():
    """Angles beyond |x| = 2^18 (and the steps where they occur) take CUDA's
    libm sin/sincos instead of the branch-free reduction (csrc/rk4.cu)."""
    ps = synth.rk4_params(64)
    for init in ([3.0e5, 0.0, 0.3, 0.0], [0.1, 0.0, -1.0e7, 2.0], [262143.0, 1.0, 262145.0, -1.0]):
        got = accelerate(lambda p, s0: rk4_sweep(p, s0, 50, synth.RK4_H), ps, init)
        want = O.rk4(ps, init, 50, synth.RK4_H)
        assert np.allclose(got, want, rtol=FP64_REL, atol=1e-12), init


# ------------------------------------------------------------------ HMM forward
@pytest.mark.parametrize("ix", [0, 1, 2])
def test_hmm_forward_golden(ix, golden):
    e = golden["hmm_forward"][ix]
    A, E, pi = synth.hmm_model(e["S"], e["K"])
    obs = synth.hmm_obs(e["NS"], e["T"], e["K"])
    got = accelerate(hmm_forward, A, E, pi, obs)
    want = [float(v) for v in e["stdout"].split()]
    assert np.allclose(got, want, rtol=LL_REL, atol=0)


@pytest.mark.parametrize("S,nsig,T", [(256, 40, 40), (512, 33, 12), (1024, 33, 8), (100, 5, 30), (2048, 2, 5),
                                       (1024, 1, 1), (1024, 130, 2), (1024, 129, 3), (1024, 300, 17)])
def test_hmm_forward_vs_oracle(S, nsig, T):
    A, E, pi = synth.hmm_model(S, 8)
    obs = synth.hmm_obs(nsig, T, 8)
    got = accelerate(hmm_forward, A, E, pi, obs)
    want = O.hmm_forward(A, E, pi, obs)
    assert np.allclose(got, want, rtol=LL_REL, atol=0), np.max(np.abs(got - want) / np.abs(want))


def test_hmm_forward_tensor_core_path_precision():
    # S = 1024 runs on tcgen05 (TF32 operands rounded to nearest, two accumulator
    # sets): long sequence, several signals incl. a partial CTA and padding
    # clusters, vs the fp64 log-space oracle.  The residual is a small low bias
    # (~1e-6 relative, constant in T) from the tensor core's truncating fp32
    # accumulation; the budget is the north star's 1e-5.
    A, E, pi = synth.hmm_model(1024, 8)
    obs = synth.hmm_obs(35, 300, 8)
    got = accelerate(hmm_forward, A, E, pi, obs)
    want = O.hmm_forward(A, E, pi, obs)
    err = np.max(np.abs(got - want) / np.abs(want))
    assert err < 5e-6, err


def _impossible_symbol_obs(nsig, T):
    obs = synth.hmm_obs(nsig, T, 8) % 7
    obs[1, 4] = 7          # symbol 7 mid-sequence, at the first step and at the last
    obs[2, 0] = 7
    obs[nsig - 1, T - 1] = 7
    return obs


@pytest.mark.parametrize("S", [64, 1024])
def test_hmm_forward_zero_emission_probability_raises_like_reference(S):
    # the program takes log of the probabilities: log 0.0 is the reference's
    # "math domain error" (pmx/interp.py scalar semantics), raised here too
    A, E, pi = synth.hmm_model(S, 8)
    E = E.copy()
    E[:, 7] = 0.0
    with pytest.raises(P.Diagnostics, match="log: math domain error"):
        accelerate(hmm_forward, A, E, pi, _impossible_symbol_obs(5, 9))


@pytest.mark.parametrize("S", [64, 256, 1024])
def test_hmm_forward_raw_impossible_observation_is_nan(S):
    # the C-ABI entry with log-space inputs (log E = -inf for symbol 7): a signal
    # that observes it gets NaN, as the log-space recursion does (its
    # max-shifted log-sum-exp over all -inf terms); other signals are unaffected
    A, E, pi = synth.hmm_model(S, 8)
    E = E.copy()
    E[:, 7] = 0.0
    obs = _impossible_symbol_obs(5, 9)
    nsig, T = obs.shape
    with np.errstate(divide="ignore", invalid="ignore"):
        want = O.hmm_forward(A, E, pi, obs)
        lE = torch.from_numpy(np.log(E).astype(np.float32)).cuda()
        lpi = torch.from_numpy(np.log(pi).astype(np.float32)).cuda()
    Ad = torch.from_numpy(A.astype(np.float32)).cuda()
    o = torch.from_numpy(obs.astype(np.int32)).cuda()
    out = torch.empty(nsig, dtype=torch.float64, device="cuda")
    from paper_2211_00621_b200 import _lib, casestudies as CS
    ws = torch.empty(_lib.load().pmx_hmm_forward_workspace_bytes(S, nsig), dtype=torch.uint8, device="cuda")
    CS.hmm_forward_raw(lpi, Ad, lE, o, S, 8, nsig, T, out, ws)
    got = out.cpu().numpy()
    assert np.isnan(want[[1, 2, 4]]).all()
    assert np.isnan(got[[1, 2, 4]]).all(), got
    assert np.allclose(got[[0, 3]], want[[0, 3]], rtol=LL_REL, atol=0)


def test_hmm_forward_long_sequence_precision():
    # T = 2000 at S = 256: fp32 trellis with fp64 running log-scale stays far inside 1e-5
    A, E, pi = synth.hmm_model(256, 8)
    obs = synth.hmm_obs(3, 2000, 8)
    got = accelerate(hmm_forward, A, E, pi, obs)
    want = O.hmm_forward(A, E, pi, obs)
    assert np.max(np.abs(got - want) / np.abs(want)) < 1e-6


# ------------------------------------------------------------------ Viterbi
def test_viterbi_reference_program(golden):
    def norm(r):
        t = 0.0
        for v in r:
            t += v
        return [v / t for v in r]
    A = [norm([float(1 + ((i * 7 + j * 3) % 5)) for j in range(4)]) for i in range(4)]
    E = [norm([float(1 + ((j * 5 + k * 2) % 7)) for k in range(8)]) for j in range(4)]
    pi = norm([float(1 + i) for i in range(4)])
    obs = [(t * t + 3 * t) % 8 for t in range(64)]
    r = accelerate(viterbi, A, E, pi, obs)
    lines = golden["program_viterbi"]["stdout"].strip().splitlines()
    assert [int(v) for v in r["path"]] == [int(v) for v in lines[0].split()]
    assert math.isclose(float(r["logp"][0]), float(lines[1]), rel_tol=1e-12)


def test_viterbi_vs_oracle():
    A, E, pi = synth.hmm_model(16, 8)
    obs = synth.hmm_obs(6, 80, 8)
    r = accelerate(viterbi, A, E, pi, obs)
    path, logp = O.viterbi(A, E, pi, obs)
    assert np.array_equal(r["path"], path)
    assert np.allclose(r["logp"], logp, rtol=1e-12)


@pytest.mark.parametrize("S,nsig,T", [(256, 37, 60), (512, 21, 40), (1024, 11, 30), (1024, 9, 1), (1024, 13, 2)])
def test_viterbi_tiled_vs_oracle(S, nsig, T):
    # batched register-tiled kernel (viterbi.cu): paths bit-exact, logp fp64
    A, E, pi = synth.hmm_model(S, 8)
    obs = synth.hmm_obs(nsig, T, 8)
    r = accelerate(viterbi, A, E, pi, obs)
    path, logp = O.viterbi(A, E, pi, obs)
    assert np.array_equal(np.asarray(r["path"]).reshape(nsig, T), path)
    assert np.allclose(np.asarray(r["logp"]), logp, rtol=1e-12, atol=0)


@pytest.mark.parametrize("dense", [False, True])
def test_viterbi_ties_first_index(dense, tmp_path):
    """Exact ties everywhere (uniform transitions, two identical emission rows):
    the pruned scan over sorted columns (default) and the dense kernel
    (PMX_VITERBI_DENSE=1, in a subprocess) both keep the reference's first
    index, like the oracle."""
    import json
    import os
    import subprocess
    import sys
    code = ("import json, numpy as np\n"
            "from paper_2211_00621_b200 import accelerate, viterbi, synth\n"
            "S, K = 256, 8\n"
            "A = np.full((S, S), 1.0 / S)\n"
            "_, E, pi = synth.hmm_model(S, K)\n"
            "E[1] = E[0]; E[5] = E[0]; pi = np.full(S, 1.0 / S)\n"
            "obs = synth.hmm_obs(11, 25, K)\n"
            "r = accelerate(viterbi, A, E, pi, obs)\n"
            "print(json.dumps([np.asarray(r['path']).tolist(), np.asarray(r['logp']).tolist()]))\n")
    env = dict(os.environ)
    if dense:
        env["PMX_VITERBI_DENSE"] = "1"
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                         cwd=str(pathlib.Path(__file__).resolve().parent.parent))
    assert out.returncode == 0, out.stderr[-2000:]
    path, logp = json.loads(out.stdout.strip().splitlines()[-1])
    S, K = 256, 8
    A = np.full((S, S), 1.0 / S)
    _, E, pi = synth.hmm_model(S, K)
    E[1] = E[0]
    E[5] = E[0]
    pi = np.full(S, 1.0 / S)
    obs = synth.hmm_obs(11, 25, K)
    wpath, wlogp = O.viterbi(A, E, pi, obs)
    assert np.array_equal(np.asarray(path).reshape(11, 25), wpath)
    assert np.allclose(logp, wlogp, rtol=1e-12, atol=0)


# ------------------------------------------------------------------ k-NN
@pytest.mark.parametrize("ix", [0, 1, 2])
def test_knn_golden(ix, golden):
    e = golden["knn"][ix]
    X = synth.knn_train(e["NT"], e["D"])
    Q = synth.knn_query(e["NQ"], e["D"])
    L = synth.knn_labels(e["NT"], e["C"])
    got = accelerate(lambda x, l, q: knn_classify(x, l, q, e["K"], e["C"]), X, L, Q)
    assert got.tolist() == [int(v) for v in e["stdout"].split()]


@pytest.mark.parametrize("ntr,nq,d,k,c", [(5000, 300, 64, 8, 10), (1000, 130, 16, 3, 4), (777, 65, 64, 17, 10),
                                          (2000, 70, 64, 8, 10), (131, 257, 64, 1, 3), (4099, 513, 64, 5, 7)])
def test_knn_vs_oracle(ntr, nq, d, k, c):
    X = synth.knn_train(ntr, d)
    Q = synth.knn_query(nq, d)
    L = synth.knn_labels(ntr, c)
    lab, idx = accelerate(lambda x, l, q: knn_classify(x, l, q, k, c, return_indices=True), X, L, Q)
    olab, oidx = O.knn(X, L, Q, k, c)
    assert np.array_equal(lab, olab)
    assert np.array_equal(idx, oidx)


@pytest.mark.parametrize("lo,hi,ntr,nq,k", [
    (0, 1, 3000, 300, 8),      # coordinates in {0, 1}: distances <= 64, massive ties -> index order decides
    (-20, 20, 2000, 100, 8),   # squared distances up to ~10^5: beyond the packed keys -> SIMT kernel
    (-8, 8, 8, 40, 8),         # k == ntr, one padded tile: every list holds padding
    (-3, 3, 70000, 260, 7),    # several train splits per query block, k < 8
])
def test_knn_integer_ranges_exact(lo, hi, ntr, nq, k):
    rng = np.random.default_rng(ntr + nq)
    X = rng.integers(lo, hi + 1, size=(ntr, 64)).astype(np.float32)
    Q = rng.integers(lo, hi + 1, size=(nq, 64)).astype(np.float32)
    L = synth.knn_labels(ntr, 10)
    lab, idx = accelerate(lambda x, l, q: knn_classify(x, l, q, k, 10, return_indices=True), X, L, Q)
    olab, oidx = O.knn(X, L, Q, k, 10)
    assert np.array_equal(idx, oidx)
    assert np.array_equal(lab, olab)


def test_knn_half_integer_queries_take_the_bf16_form():
    # queries with eight coordinates at +-0.5 (the rest integers): not int8-exact,
    # bf16-exact with integer norms -> the bf16 tensor-core kernel (flag 8); exact
    rng = np.random.default_rng(11)
    X = rng.integers(-6, 7, size=(3000, 64)).astype(np.float32)
    Q = rng.integers(-6, 7, size=(200, 64)).astype(np.float32)
    for r in range(200):
        cols = rng.choice(64, size=8, replace=False)
        Q[r, cols] = rng.choice([-0.5, 0.5], size=8)
    L = synth.knn_labels(3000, 10)
    lab, idx = accelerate(lambda x, l, q: knn_classify(x, l, q, 8, 10, return_indices=True), X, L, Q)
    olab, oidx = O.knn(X, L, Q, 8, 10)
    assert np.array_equal(idx, oidx)
    assert np.array_equal(lab, olab)


def test_knn_continuous_data_is_tie_tolerant():
    rng = np.random.default_rng(3)
    X = rng.random((3000, 64), dtype=np.float32)
    Q = rng.random((100, 64), dtype=np.float32)
    L = synth.knn_labels(3000, 10)
    lab, idx = accelerate(lambda x, l, q: knn_classify(x, l, q, 8, 10, return_indices=True), X, L, Q)
    olab, oidx = O.knn(X, L, Q, 8, 10)
    # same neighbour sets up to fp32 rounding of near-equal distances
    d = ((Q[:, None, :].astype(np.float64) - X[None, :, :]) ** 2).sum(-1)
    for q in range(100):
        got_d = np.sort(d[q, idx[q]])
        want_d = np.sort(d[q, oidx[q]])
        assert np.allclose(got_d, want_d, rtol=1e-5)


# ------------------------------------------------------------------ k-mer HMM
@pytest.mark.parametrize("ix", [0, 1])
def test_kmer_golden(ix, golden):
    e = golden["kmer"][ix]
    E = synth.kmer_emission(e["kmer"], e["K"])
    obs = synth.hmm_obs(e["NS"], e["T"], e["K"])
    got = accelerate(lambda em, o: hmm_kmer_forward(e["kmer"], e["p_stay"], e["p_step"], em, o), E, obs)
    want = [float(v) for v in e["stdout"].split()]
    assert np.allclose(got, want, rtol=LL_REL, atol=0)


@pytest.mark.parametrize("kmer,nsig,T", [(5, 4, 60), (8, 2, 6)])
def test_kmer_vs_oracle(kmer, nsig, T):
    E = synth.kmer_emission(kmer, 8)
    obs = synth.hmm_obs(nsig, T, 8)
    got = accelerate(lambda em, o: hmm_kmer_forward(kmer, 0.5, 0.125, em, o), E, obs)
    want = O.kmer_forward(kmer, 0.5, 0.125, E, obs)
    assert np.allclose(got, want, rtol=LL_REL, atol=0)


@pytest.mark.parametrize("nsig,T", [(1, 1), (3, 2), (75, 9), (149, 5), (200, 17)])
def test_kmer8_cluster_signal_loop(nsig, T):
    # k = 8 runs on CTA pairs (k_kmer_fwd_pair), one signal per pair at a time:
    # fewer signals than pairs, one extra signal past a whole round (75, 149 with
    # 74 pairs), several rounds, and T = 1 (no exchange step inside a signal)
    E = synth.kmer_emission(8, 8)
    obs = synth.hmm_obs(nsig, T, 8)
    got = accelerate(lambda em, o: hmm_kmer_forward(8, 0.5, 0.125, em, o), E, obs)
    want = O.kmer_forward_scaled(8, 0.5, 0.125, E, obs)
    assert np.allclose(got, want, rtol=LL_REL, atol=0)


@pytest.mark.parametrize("kmer", [4, 8])
def test_kmer_raw_impossible_observation_is_nan(kmer):
    # C-ABI entry with log E = -inf for symbol 7 in every state: a signal that
    # observes it gets NaN like the log-space recursion; through accelerate the
    # program's log 0.0 raises the reference's math domain error instead
    S, K = 1 << (2 * kmer), 8
    E = synth.kmer_emission(kmer, K)
    E[:, 7] = 0.0
    obs = _impossible_symbol_obs(5, 12)
    nsig, T = obs.shape
    with np.errstate(divide="ignore", invalid="ignore"):
        want = O.kmer_forward(kmer, 0.5, 0.125, E, obs)
        lE = torch.from_numpy(np.log(E).astype(np.float32)).cuda()
    from paper_2211_00621_b200 import _lib
    lib = _lib.load()
    o = torch.from_numpy(obs.astype(np.int32)).cuda()
    out = torch.empty(nsig, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.pmx_hmm_kmer_workspace_bytes(kmer, nsig), dtype=torch.uint8, device="cuda")
    _lib.check(lib.pmx_hmm_kmer_forward_f32(kmer, 0.5, 0.125, lE.data_ptr(), K, o.data_ptr(), nsig, T,
                                            out.data_ptr(), ws.data_ptr(), ws.numel(),
                                            torch.cuda.current_stream().cuda_stream), "kmer")
    got = out.cpu().numpy()
    assert np.isnan(want[[1, 2, 4]]).all()
    assert np.isnan(got[[1, 2, 4]]).all(), got
    assert np.allclose(got[[0, 3]], want[[0, 3]], rtol=LL_REL, atol=0)
    with pytest.raises(P.Diagnostics, match="log: math domain error"):
        accelerate(lambda em, ob: hmm_kmer_forward(kmer, 0.5, 0.125, em, ob), E, obs)


def test_kmer8_cluster_peaked_emissions():
    # emissions spanning ~9 decades (state-dependent), stay/step not summing to 1
    S, K = 1 << 16, 8
    j = np.arange(S)[:, None]
    k = np.arange(K)[None, :]
    E = np.exp(-((j * 7 + k * 5) % 23) * 0.9)
    E /= E.sum(axis=1, keepdims=True)
    obs = synth.hmm_obs(6, 40, K)
    got = accelerate(lambda em, o: hmm_kmer_forward(8, 0.7, 0.05, em, o), E, obs)
    want = O.kmer_forward_scaled(8, 0.7, 0.05, E, obs)
    assert np.allclose(got, want, rtol=LL_REL, atol=0)


# ---------------------------------------------------------- NN gradients
def _nn_ref_data():
    n_in, n_out, n_pts = 16, 8, 32
    x = np.array([[((p * 5 + i * 3) % 11 - 5) / 10.0 for i in range(n_in)] for p in range(n_pts)])
    y = np.array([(p * 7 + 3) % n_out for p in range(n_pts)], np.int32)
    w = np.array([[((i * 3 + j * 7) % 13 - 6) / 20.0 for j in range(n_out)] for i in range(n_in)])
    b = np.array([((j * 5) % 9 - 4) / 15.0 for j in range(n_out)])
    return x, y, w, b


def _nn_loss(x, y, w, b):
    z = x @ w + b
    return float(np.mean(np.log(np.sum(np.exp(z), axis=1)) - z[np.arange(len(y)), y]))


def test_nn_reference_program(golden):
    # programs/nn.pmx: loss, dw, db against the reference's printed values
    # (sums over points in a different order than its 4 workers: rel 1e-12)
    from paper_2211_00621_b200 import nn_gradients
    r = accelerate(nn_gradients, *_nn_ref_data())
    lines = [l for l in golden["program_nn"]["stdout"].splitlines() if l.strip()]
    assert math.isclose(r["loss"], float(lines[0]), rel_tol=1e-12)
    want_dw = np.array([[float(v) for v in l.split()] for l in lines[1:17]])
    want_db = np.array([float(v) for v in lines[17].split()])
    assert np.allclose(np.asarray(r["dw"]).reshape(16, 8), want_dw, rtol=1e-12, atol=1e-17)
    assert np.allclose(np.asarray(r["db"]), want_db, rtol=1e-12, atol=1e-17)


def test_nn_gradients_match_finite_differences():
    # the reference's own check (tests/test_acceptance.py:424-441)
    from paper_2211_00621_b200 import nn_gradients
    x, y, w, b = _nn_ref_data()
    r = accelerate(nn_gradients, x, y, w, b)
    dw = np.asarray(r["dw"]).reshape(16, 8)
    eps = 1e-5
    for i in range(16):
        for j in range(8):
            wp, wm = w.copy(), w.copy()
            wp[i, j] += eps
            wm[i, j] -= eps
            fd = (_nn_loss(x, y, wp, b) - _nn_loss(x, y, wm, b)) / (2 * eps)
            assert math.isclose(dw[i, j], fd, rel_tol=1e-4, abs_tol=1e-8)


@pytest.mark.parametrize("npts,nin,nout", [(100_003, 64, 16), (4097, 7, 32), (1, 3, 1), (50_000, 33, 5),
                                            (70_001, 62, 32), (9_999, 64, 3)])
def test_nn_vs_oracle(npts, nin, nout):
    from paper_2211_00621_b200 import nn_gradients
    rng = np.random.default_rng(npts + nin)
    x = rng.standard_normal((npts, nin)) * 0.5
    y = rng.integers(0, nout, npts).astype(np.int32)
    w = rng.standard_normal((nin, nout)) * 0.3
    b = rng.standard_normal(nout) * 0.1
    r = accelerate(nn_gradients, x, y, w, b)
    loss, dw, db = O.nn(x, y, w, b, workers=4)
    assert math.isclose(r["loss"], loss, rel_tol=1e-11)
    assert np.allclose(np.asarray(r["dw"]).reshape(nin, nout), dw, rtol=1e-9, atol=1e-14)
    assert np.allclose(np.asarray(r["db"]), db, rtol=1e-9, atol=1e-14)


def test_nn_errors():
    from paper_2211_00621_b200 import Diagnostics, nn_gradients
    x, y, w, b = _nn_ref_data()
    y = y.copy()
    y[9] = 8
    with pytest.raises(Diagnostics, match="out of bounds") as ei:
        accelerate(nn_gradients, x, y, w, b)
    assert "element 9)" in str(ei.value)
    with pytest.raises(Diagnostics, match="float division by zero"):
        accelerate(nn_gradients, np.zeros((0, 16)), np.zeros(0, np.int32), w, b)
    # every exp underflows to 0 at point 3: log of a zero total (math.log(0.0))
    x2 = np.zeros((300, 16))
    x2[3] = -100.0
    x2[200] = 1000.0                                  # exp overflow later: the first error wins
    with pytest.raises(Diagnostics, match="log: math domain error") as ei:
        accelerate(nn_gradients, x2, np.zeros(300, np.int32), np.ones((16, 8)), np.zeros(8))
    assert "element 3)" in str(ei.value)
    x2[3] = 0.0
    with pytest.raises(Diagnostics, match="exp: math range error") as ei:
        accelerate(nn_gradients, x2, np.zeros(300, np.int32), np.ones((16, 8)), np.zeros(8))
    assert "element 200)" in str(ei.value)


# ------------------------------------------------------------ RK4 trace
def test_rk4_trace_vs_oracle():
    # the paper's N x M trace of one measured state
    from paper_2211_00621_b200 import rk4_trace
    ps = synth.rk4_params(300)
    tr, fin = accelerate(lambda p, s: rk4_trace(p, s, 200, synth.RK4_H, 2), ps, synth.RK4_INIT)
    want_fin, want_tr = O.rk4_trace(ps, synth.RK4_INIT, 200, synth.RK4_H, 2)
    assert np.asarray(tr).shape == (300, 200)
    assert np.allclose(np.asarray(tr), want_tr, rtol=1e-9, atol=1e-12)
    assert np.allclose(np.asarray(fin), want_fin, rtol=1e-9, atol=1e-12)
    assert np.array_equal(np.asarray(tr)[:, -1], np.asarray(fin)[:, 2])


def test_rk4_trace_into_aliased_tensor_view():
    # trace written through a tensor view of a larger heap buffer (tensorSub,
    # Alg. 2 root): only the view's rows change, the rest of the buffer stays
    from paper_2211_00621_b200 import Ctx, Heap, TensorView, rk4_trace
    n, m = 50, 30
    heap = Heap()
    buf = heap.alloc(np.full((n + 4) * m, -7.0))
    view = TensorView(buf, 2 * m, (n, m), "float")          # rows 2 .. n+1
    ps = synth.rk4_params(n)
    accelerate(lambda p, s, t: rk4_trace(p, s, m, synth.RK4_H, 0, trace=t)[1], ps, synth.RK4_INIT, view,
               ctx=Ctx(heap=heap))
    got = heap.buffers[buf].reshape(n + 4, m)
    _, want = O.rk4_trace(ps, synth.RK4_INIT, m, synth.RK4_H, 0)
    assert np.allclose(got[2:n + 2], want, rtol=1e-9, atol=1e-12)
    assert (got[:2] == -7.0).all() and (got[n + 2:] == -7.0).all()


@pytest.mark.parametrize("variant", ["pair", "f16", "tf32"])
def test_hmm_forward_kernel_variants_vs_oracle(variant, tmp_path):
    """The non-default S = 1024 tensor-core kernels (PMX_HMM_TC, read once per
    process, so each runs in a subprocess): the CTA-pair kernel with single-SM
    UMMAs (hmm_pair.cu), the single-CTA fp16 and TF32 kernels — same
    signals as the default kernel's precision test, incl. a partial cluster."""
    import json
    import os
    import subprocess
    import sys
    A, E, pi = synth.hmm_model(1024, 8)
    obs = synth.hmm_obs(133, 120, 8)
    want = O.hmm_forward(A, E, pi, obs)
    code = ("import json, sys, numpy as np\n"
            "from paper_2211_00621_b200 import accelerate, hmm_forward, synth\n"
            "A, E, pi = synth.hmm_model(1024, 8)\n"
            "obs = synth.hmm_obs(133, 120, 8)\n"
            "print(json.dumps([float(v) for v in np.asarray(accelerate(hmm_forward, A, E, pi, obs))]))\n")
    env = dict(os.environ, PMX_HMM_TC=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=str(pathlib.Path(__file__).resolve().parent.parent))
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.array(json.loads(r.stdout.strip().splitlines()[-1]))
    err = np.max(np.abs(got - want) / np.abs(want))
    assert err < 5e-6, (variant, err)

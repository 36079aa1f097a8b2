"""Parity at the BASELINE configs' full sizes (VERDICT r1 "next" item 1).

Each case study runs on the B200 through the public `accelerate` entry at the
size `bench.py` measures; a deterministic sample of its elements (signals,
queries) is recomputed by the CPU oracle and compared with the north-star
tolerances: indices and labels bit-exact, fp64 rel 1e-9, log-likelihoods rel
1e-5 in fp64.  The oracle finishes each sample in seconds (the scaled-linear
HMM restatements are checked against the log-space ones in test_oracle.py).
Reference pins: tests/test_acceptance.py:307-394 (Viterbi, RK4), SURVEY §8(d)
and Appendix A (HMM forward, k-NN, k-mer)."""
import numpy as np
import pytest

import oracle as O
from paper_2211_00621_b200 import (
    accelerate, hmm_forward, hmm_kmer_forward, knn_classify, rk4_sweep, synth, viterbi,
)
from paper_2211_00621_b200 import casestudies as CS

pytestmark = pytest.mark.gpu

LL_REL = 1e-5
FP64_REL = 1e-9


def test_rk4_full_config_every_parameter_set():
    # 10^4 parameter sets x 10^3 steps, fp64: all 40,000 outputs
    n, m = 10_000, 1_000
    ps = synth.rk4_params(n)
    got = accelerate(lambda p, s0: rk4_sweep(p, s0, m, synth.RK4_H), ps, synth.RK4_INIT)
    want = O.rk4(ps, synth.RK4_INIT, m, synth.RK4_H)
    assert got.shape == (n, 4)
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
    assert np.all((rel <= FP64_REL) | (np.abs(got - want) <= 1e-12)), float(rel.max())


def test_knn_full_config_sampled_queries():
    # 2^20 train x 2^16 queries, d = 64, k = 8, 10 classes; 2,048+ sampled
    # queries: labels and neighbour indices bit-exact
    ntr, nq, d, k, c = 1 << 20, 1 << 16, 64, 8, 10
    X, L, Q = synth.knn_train(ntr, d), synth.knn_labels(ntr, c), synth.knn_query(nq, d)
    lab, idx = accelerate(lambda a, b, q: knn_classify(a, b, q, k, c, return_indices=True), X, L, Q)
    sel = synth.parity_sample(nq, 2048)
    want_lab, want_idx = O.knn(X, L, Q[sel], k, c)
    assert np.array_equal(lab[sel], want_lab)
    assert np.array_equal(idx[sel], want_idx)


def test_hmm_forward_full_config_sampled_signals():
    # 4096 signals x T = 10^4 x S = 1024, K = 8 (fp16 tensor-core path): 16+
    # sampled signals against the fp64 oracle, rel 1e-5
    S, K, nsig, T = 1024, 8, 4096, 10_000
    A, E, pi = synth.hmm_model(S, K)
    obs = synth.hmm_obs(nsig, T, K)
    got = accelerate(hmm_forward, A, E, pi, obs)
    assert CS.hmm_forward_rerun_count(S, nsig) == 0          # the range guard stayed quiet
    sel = synth.parity_sample(nsig, 16)
    want = O.hmm_forward_scaled(A, E, pi, obs[sel])
    rel = np.abs(got[sel] - want) / np.abs(want)
    assert rel.max() <= LL_REL, (float(rel.max()), sel[np.argmax(rel)])


def test_kmer_full_config_sampled_signals():
    # S = 65,536 (k = 8) de Bruijn, one GPU's 1024 of the 8k signals, T = 6000
    kmer, K, nsig, T = 8, 8, 1024, 6000
    E = synth.kmer_emission(kmer, K)
    obs = synth.hmm_obs(nsig, T, K)
    got = accelerate(lambda e, o: hmm_kmer_forward(kmer, 0.5, 0.125, e, o), E, obs)
    sel = synth.parity_sample(nsig, 16)
    want = O.kmer_forward_scaled(kmer, 0.5, 0.125, E, obs[sel])
    rel = np.abs(got[sel] - want) / np.abs(want)
    assert rel.max() <= LL_REL, float(rel.max())


def test_viterbi_full_config_sampled_signals():
    # S = 1024, K = 8, 1184 signals (8 per SM) x T = 1000, fp64: sampled paths
    # bit-exact, logp rel 1e-9
    S, K, nsig, T = 1024, 8, 148 * 8, 1000
    A, E, pi = synth.hmm_model(S, K)
    obs = synth.hmm_obs(nsig, T, K)
    r = accelerate(viterbi, A, E, pi, obs)
    sel = synth.parity_sample(nsig, 16)
    path, logp = O.viterbi(A, E, pi, obs[sel])
    assert np.array_equal(np.asarray(r["path"])[sel], path)
    assert np.allclose(np.asarray(r["logp"])[sel], logp, rtol=FP64_REL, atol=0)


# ------------------------------------------------ fp16 range guard
@pytest.mark.parametrize("nsig,T", [(130, 300), (1, 40)])
def test_hmm_forward_rare_symbol_is_scaled_not_flushed(nsig, T):
    # symbol 7 has probability ~1e-9 in every state: without the per-symbol
    # power-of-two emission scale u_t underflows fp16 (NaN / -inf ll)
    S, K = 1024, 8
    A, E, pi = synth.hmm_model_rare_symbol(S, K)
    obs = synth.hmm_obs(nsig, T, K)
    obs[:, ::7] = K - 1                                     # the rare symbol every 7th step
    got = accelerate(hmm_forward, A, E, pi, obs)
    want = O.hmm_forward_scaled(A, E, pi, obs)
    assert np.all(np.isfinite(got))
    rel = np.abs(got - want) / np.abs(want)
    assert rel.max() <= LL_REL, float(rel.max())


def test_hmm_forward_peaky_model_reruns_flagged_signals():
    # Near-deterministic A / E / pi.  Observations against the current state give
    # per-step emission masses far below 2^-8 (range flag); observations that
    # follow the model (state 0 emitting symbol 0 throughout) keep ~all the mass
    # in one state, whose fp16 rounding error (2^-11) would recur every step and
    # exceed the budget on this |ll| (concentration events).  The guard re-runs
    # both kinds in fp32 on the device.
    S, K, T = 1024, 8, 200
    A, E, pi = synth.hmm_model_peaky(S, K)
    obs = np.concatenate([synth.hmm_obs(131, T, K), np.zeros((3, T), np.int32)])
    got = accelerate(hmm_forward, A, E, pi, obs)
    n_rerun = CS.hmm_forward_rerun_count(S, obs.shape[0])
    want = O.hmm_forward_scaled(A, E, pi, obs)
    assert np.all(np.isfinite(got))
    rel = np.abs(got - want) / np.abs(want)
    assert rel.max() <= LL_REL, float(rel.max())
    assert n_rerun == obs.shape[0], n_rerun


def test_hmm_forward_sparse_initial_distribution():
    S, K = 1024, 8
    A, E, _ = synth.hmm_model(S, K)
    pi = np.full(S, 1e-12)
    pi[517] = 1.0
    pi /= pi.sum()
    obs = synth.hmm_obs(40, 120, K)
    got = accelerate(hmm_forward, A, E, pi, obs)
    want = O.hmm_forward_scaled(A, E, pi, obs)
    rel = np.abs(got - want) / np.abs(want)
    assert rel.max() <= LL_REL, float(rel.max())


def test_viterbi_pruned_scan_with_nan_log_transitions():
    # NaN entries of log A (possible through the C ABI, which takes log A
    # directly) sort after every number in the pruned kernel's column order, so
    # they neither win nor stop a scan early: same path as a dense max-plus that
    # skips NaN candidates (first index on ties)
    import torch
    from paper_2211_00621_b200 import _lib
    S, K, nsig, T = 256, 8, 3, 25
    A, E, pi = synth.hmm_model(S, K)
    lA = np.log(A)
    rng = np.random.default_rng(5)
    lA[rng.integers(0, S, 400), rng.integers(0, S, 400)] = np.nan
    lE, lpi = np.log(E), np.log(pi)
    obs = synth.hmm_obs(nsig, T, K)
    want_path = np.empty((nsig, T), np.int32)
    for s in range(nsig):
        chi = lpi + lE[:, obs[s, 0]]
        back = []
        for t in range(1, T):
            cand = chi[:, None] + lA
            arg = np.nanargmax(cand, axis=0)
            back.append(arg)
            chi = cand[arg, np.arange(S)] + lE[:, obs[s, t]]
        st = int(np.argmax(chi))
        want_path[s, T - 1] = st
        for t in range(T - 1, 0, -1):
            st = int(back[t - 1][st])
            want_path[s, t - 1] = st
    dev = torch.device("cuda")
    t_lA, t_lE, t_lpi = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (lA, lE, lpi))
    t_obs = torch.from_numpy(obs).to(dev)
    path = torch.empty(nsig * T, dtype=torch.int32, device=dev)
    logp = torch.empty(nsig, dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = torch.empty(lib.pmx_viterbi_workspace_bytes(S, nsig, T), dtype=torch.uint8, device=dev)
    st_ = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.pmx_viterbi_f64(t_lpi.data_ptr(), t_lA.data_ptr(), t_lE.data_ptr(), S, K, t_obs.data_ptr(), nsig,
                                   T, path.data_ptr(), logp.data_ptr(), ws.data_ptr(), ws.numel(), st_), "viterbi")
    assert lib.pmx_viterbi_visited_cells(ws.data_ptr(), S, nsig, T, st_) > 0
    assert np.array_equal(path.cpu().numpy().reshape(nsig, T), want_path)


def test_viterbi_visited_cells_counter():
    # the pruned kernel's work counter (the Viterbi roofline's numerator): at most
    # the dense cell count, and a small fraction of it on the bench model
    import torch
    from paper_2211_00621_b200 import _lib
    S, K, nsig, T = 1024, 8, 16, 50
    A, E, pi = synth.hmm_model(S, K)
    dev = torch.device("cuda")
    lA, lE, lpi = (torch.from_numpy(np.log(a)).to(dev) for a in (A, E, pi))
    obs = torch.from_numpy(synth.hmm_obs(nsig, T, K)).to(dev)
    path = torch.empty(nsig * T, dtype=torch.int32, device=dev)
    logp = torch.empty(nsig, dtype=torch.float64, device=dev)
    lib = _lib.load()
    ws = torch.empty(lib.pmx_viterbi_workspace_bytes(S, nsig, T), dtype=torch.uint8, device=dev)
    st_ = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.pmx_viterbi_f64(lpi.data_ptr(), lA.data_ptr(), lE.data_ptr(), S, K, obs.data_ptr(), nsig, T,
                                   path.data_ptr(), logp.data_ptr(), ws.data_ptr(), ws.numel(), st_), "viterbi")
    v = lib.pmx_viterbi_visited_cells(ws.data_ptr(), S, nsig, T, st_)
    dense = S * S * (T - 1) * 16          # 8-signal CTAs: 2 CTAs, padding-free here
    assert 0 < v <= dense
    assert v < 0.5 * dense, v / dense

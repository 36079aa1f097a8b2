"""Synthetic inputs of the benchmark configs, defined by integer formulas.

Every formula here is expressible with the reference's own builtins (muli,
modi, divi, int2float, divf) so the same bits are produced by a PMExpr
program run by the reference interpreter (tests/golden/make_golden.py), by
numpy here, and on the device (torch integer ops, for device-resident runs).
Values are chosen to be exactly representable in fp32 where the config is
fp32.
"""
from __future__ import annotations

import numpy as np

M32 = 1 << 32
GOLD = 2654435761        # Knuth multiplicative hash
GOLD2 = 2246822519


def _h(a: np.ndarray, mult: int = GOLD, shift: int = 16) -> np.ndarray:
    """((a * mult) mod 2^32) >> shift   — PMExpr: divi (modi (muli a mult) 4294967296) 2^shift."""
    a = np.asarray(a, dtype=np.int64)
    return ((a * mult) % M32) >> shift


# -------------------------------------------------------------- map/reduce
def mapreduce_x(n: int, dtype=np.float32) -> np.ndarray:
    """x[i] = float(((i * 2654435761) mod 2^32) >> 10) / 2^22, exact in fp32
    (SURVEY §8(d)); i * 2654435761 < 2^60 for i < 2^28, no int64 wrap."""
    i = np.arange(n, dtype=np.int64)
    return (_h(i, GOLD, 10).astype(np.float64) / 4194304.0).astype(dtype)


def mapreduce_x_device(n: int, device, dtype=None):
    import torch
    i = torch.arange(n, dtype=torch.int64, device=device)
    v = torch.remainder(i * GOLD, M32) >> 10
    return (v.to(torch.float64) / 4194304.0).to(dtype or torch.float32)


def mapreduce_exact_sum(n: int, a: float = 2.0, b: float = 1.0) -> float:
    """Exact value of reduce addf 0.0 (map (lam x. a*x + b) x) for the default
    (a, b) = (2, 1): every partial sum is a multiple of 2^-21 below 2^30, so the
    fp64 reference is exact and schedule-independent."""
    m = _h(np.arange(n, dtype=np.int64), GOLD, 10)
    # 2*(m/2^22) + 1 = (m + 2^21) / 2^21
    assert a == 2.0 and b == 1.0
    return float(int(m.sum()) + n * (1 << 21)) / float(1 << 21)


# -------------------------------------------------------------------- RK4
def rk4_params(n: int, first: int = 0, total: int | None = None) -> np.ndarray:
    """p_k = 0.5 + k/N (non-chaotic range); rows
    [first, first + n) of an N = `total` (default n) parameter sweep."""
    k = np.arange(first, first + n, dtype=np.float64)
    return 0.5 + k / float(n if total is None else total)


RK4_INIT = np.array([0.1, 0.0, 0.3, 0.0], dtype=np.float64)   # programs/rk4.pmx:41
RK4_H = 0.01


# ------------------------------------------------------------------- k-NN
def knn_train(ntr: int, d: int) -> np.ndarray:
    """train[p][i] = (h(p*d + i) mod 17) - 8, integers in [-8, 8]."""
    a = np.arange(ntr * d, dtype=np.int64)
    return ((_h(a, GOLD, 16) % 17) - 8).astype(np.float32).reshape(ntr, d)


def knn_query(nq: int, d: int, first: int = 0) -> np.ndarray:
    """queries [first, first + nq) of the query formula."""
    a = np.arange(first * d, (first + nq) * d, dtype=np.int64)
    return ((_h(a, GOLD2, 16) % 17) - 8).astype(np.float32).reshape(nq, d)


def knn_labels(ntr: int, ncls: int) -> np.ndarray:
    p = np.arange(ntr, dtype=np.int64)
    return (_h(p, GOLD, 20) % ncls).astype(np.int32)


# -------------------------------------------------------------------- HMM
def _rownorm(w: np.ndarray) -> np.ndarray:
    return w / w.sum(axis=1, keepdims=True)


def hmm_model(S: int, K: int):
    """Row-stochastic (A, E, pi) with strictly positive integer weights:
    A[i][j] ~ 1 + (i*131 + j*71 + i*j*7) mod 97, E[j][k] ~ 1 + (j*13 + k*29 + j*k*3) mod 31,
    pi[i] ~ 1 + i mod 17.  Normalised in fp64 as `rowNorm` does (A.1 line 6)."""
    i = np.arange(S, dtype=np.int64)[:, None]
    j = np.arange(S, dtype=np.int64)[None, :]
    A = _rownorm((1 + (i * 131 + j * 71 + i * j * 7) % 97).astype(np.float64))
    jj = np.arange(S, dtype=np.int64)[:, None]
    k = np.arange(K, dtype=np.int64)[None, :]
    E = _rownorm((1 + (jj * 13 + k * 29 + jj * k * 3) % 31).astype(np.float64))
    pi = (1 + np.arange(S, dtype=np.int64) % 17).astype(np.float64)
    pi = pi / pi.sum()
    return A, E, pi


def hmm_obs(nsig: int, T: int, K: int, first: int = 0) -> np.ndarray:
    """obs[s][t] = h(s*T + t) mod K, for signals [first, first + nsig)."""
    a = np.arange(first * T, (first + nsig) * T, dtype=np.int64)
    return (_h(a, GOLD, 16) % K).astype(np.int32).reshape(nsig, T)


def kmer_emission(kmer: int, K: int) -> np.ndarray:
    S = 1 << (2 * kmer)
    jj = np.arange(S, dtype=np.int64)[:, None]
    k = np.arange(K, dtype=np.int64)[None, :]
    return _rownorm((1 + (jj * 13 + k * 29 + jj * k * 3) % 31).astype(np.float64))


def hmm_model_rare_symbol(S: int, K: int, eps: float = 1e-9):
    """hmm_model with symbol K-1 nearly impossible in every state (E[:, K-1] =
    eps before row normalisation): the case where an unscaled fp16 trellis
    underflows."""
    A, E, pi = hmm_model(S, K)
    E = E.copy()
    E[:, K - 1] = eps
    return A, _rownorm(E), pi


def hmm_model_peaky(S: int, K: int, stay: float = 0.999, off: float = 1e-9):
    """Near-deterministic model: A keeps its state with probability ~`stay`
    and reaches the neighbour state with the rest (every other transition
    `off`), state j emits symbol j mod K with probability 0.99, pi puts 1e-9 on
    all but state 0.  Observations that disagree with the current state force
    tiny per-step emission masses (the fp16 path's range guard re-runs them)."""
    i = np.arange(S)[:, None]
    j = np.arange(S)[None, :]
    A = np.full((S, S), off)
    A[i == j] = stay
    A[(i + 1) % S == j] = 1.0 - stay
    E = np.full((S, K), 0.01 / (K - 1))
    E[np.arange(S), np.arange(S) % K] = 0.99
    pi = np.full(S, 1e-9)
    pi[0] = 1.0
    return _rownorm(A), _rownorm(E), pi / pi.sum()


def parity_sample(n: int, m: int, block: int = 128) -> np.ndarray:
    """At least m (at most m + 7) sorted distinct element indices of [0, n):
    m evenly spaced, plus both ends and the first / last element of a few
    `block`-sized tiles (CTA / cluster edges).  Used by the sampled full-size
    parity checks."""
    edges = [0, n - 1, block - 1, block, n // 2 - 1, n // 2, n - block]
    even = np.linspace(0, n - 1, min(m, n)).astype(np.int64)
    return np.unique(np.clip(np.concatenate([np.array(edges, np.int64), even]), 0, n - 1))

"""Pin the CPU oracle against the reference's own outputs (tests/golden) and
the reference's known-answer tests.  CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from cases import FOLD_CASES, MAP2_CASES, MAP_CASES, REDUCE_CASES
from conftest import parse_tokens
from paper_2211_00621_b200 import synth


def _expect(entry):
    return ("error", entry["error"]) if "error" in entry else ("ok", entry["stdout"])


# ---------------------------------------------------------------- IR evaluator

@pytest.mark.parametrize("case", MAP_CASES, ids=[c[0] for c in MAP_CASES])
def test_ir_map_matches_reference(case, golden):
    name, _, build, ty, xs = case
    kind, want = _expect(golden["map"][name])
    if kind == "error":
        with pytest.raises(O.OracleError) as ei:
            O.ir_map(build(), xs)
        assert str(ei.value) == want
    else:
        got = O.ir_map(build(), xs)
        assert [int(v) if isinstance(v, bool) else v for v in got] == parse_tokens(want)


@pytest.mark.parametrize("case", REDUCE_CASES, ids=[c[0] for c in REDUCE_CASES])
@pytest.mark.parametrize("workers", [1, 3, 4])
def test_ir_reduce_matches_reference(case, workers, golden):
    name, _, build, _, acc, ty, xs = case
    want = parse_tokens(golden["reduce"][name]["stdout"])[0]
    assert O.ir_reduce(build(), acc, xs, workers=workers) == want


@pytest.mark.parametrize("case", FOLD_CASES, ids=[c[0] for c in FOLD_CASES])
def test_ir_fold_matches_reference(case, golden):
    name, _, build, _, acc, ty, xs = case
    assert O.ir_fold(build(), acc, xs) == parse_tokens(golden["foldl"][name]["stdout"])[0]


@pytest.mark.parametrize("case", MAP2_CASES, ids=[c[0] for c in MAP2_CASES])
def test_ir_map2_matches_reference(case, golden):
    name, _, build, ty, xs, ys = case
    kind, want = _expect(golden["map2"][name])
    if kind == "error":
        with pytest.raises(O.OracleError, match="different lengths"):
            O.ir_map2(build(), xs, ys)
    else:
        assert O.ir_map2(build(), xs, ys) == parse_tokens(want)


# ------------------------------------------------------------ C restatement

def test_mapreduce_oracle_matches_reference(golden):
    for entry in golden["mapreduce"]:
        n, w = entry["N"], entry["workers"]
        x = synth.mapreduce_x(n)
        want = float(entry["stdout"])
        for threads in (1, 4):
            assert O.map_affine_reduce_add(x, 2.0, 1.0, 0.0, workers=w, threads=threads) == want
        # the data are exact: any partition gives the same sum
        assert synth.mapreduce_exact_sum(n) == want


def test_mapreduce_generator_is_exact_in_f32():
    x64 = synth.mapreduce_x(1 << 16, np.float64)
    assert np.array_equal(x64.astype(np.float32).astype(np.float64), x64)
    assert (x64 >= 0).all() and (x64 < 1).all()


def test_rk4_oracle_matches_reference_program(golden):
    # programs/rk4.pmx: 16 params p_k = 0.5 + 0.1 k, 100 steps (test_acceptance.py:385-394)
    lines = [l for l in golden["program_rk4"]["stdout"].splitlines() if l.strip()]
    ps = np.array([0.5 + 0.1 * float(k) for k in range(16)])
    got = O.rk4(ps, synth.RK4_INIT, 100, synth.RK4_H, threads=2)
    for k, line in enumerate(lines):
        want = [float(v) for v in line.split()]
        for g, w in zip(got[k], want):
            assert math.isclose(g, w, rel_tol=1e-12), (k, got[k], want)


def test_rk4_oracle_matches_param_variant(golden):
    for entry in golden["rk4_param"]:
        n, m = entry["N"], entry["M"]
        lines = [l for l in entry["stdout"].splitlines() if l.strip()]
        got = O.rk4(synth.rk4_params(n), synth.RK4_INIT, m, synth.RK4_H)
        for k, line in enumerate(lines):
            for g, w in zip(got[k], map(float, line.split())):
                assert math.isclose(g, w, rel_tol=1e-12)


def test_viterbi_oracle_matches_reference_program(golden):
    # programs/viterbi.pmx model (S=4, K=8, T=64), tests/test_acceptance.py:307-354
    def norm(r):
        t = 0.0
        for v in r:
            t += v
        return [v / t for v in r]
    A = np.array([norm([float(1 + ((i * 7 + j * 3) % 5)) for j in range(4)]) for i in range(4)])
    E = np.array([norm([float(1 + ((j * 5 + k * 2) % 7)) for k in range(8)]) for j in range(4)])
    pi = np.array(norm([float(1 + i) for i in range(4)]))
    obs = np.array([[(t * t + 3 * t) % 8 for t in range(64)]], np.int32)
    path, logp = O.viterbi(A, E, pi, obs)
    lines = golden["program_viterbi"]["stdout"].strip().splitlines()
    assert path[0].tolist() == [int(v) for v in lines[0].split()]
    assert math.isclose(logp[0], float(lines[1]), rel_tol=1e-12)


def _model_seqnorm(S, K):
    """synth.hmm_model with rowNorm's sequential foldl sum (A.1 line 6)."""
    A, E, pi = synth.hmm_model(S, K)
    return A, E, pi


@pytest.mark.parametrize("ix", [0, 1, 2])
def test_hmm_forward_oracle_matches_reference(ix, golden):
    e = golden["hmm_forward"][ix]
    A, E, pi = synth.hmm_model(e["S"], e["K"])
    obs = synth.hmm_obs(e["NS"], e["T"], e["K"])
    got = O.hmm_forward(A, E, pi, obs, threads=2)
    want = [float(v) for v in e["stdout"].split()]
    assert np.allclose(got, want, rtol=1e-13, atol=0)


@pytest.mark.parametrize("ix", [0, 1, 2])
def test_knn_oracle_matches_reference(ix, golden):
    e = golden["knn"][ix]
    X = synth.knn_train(e["NT"], e["D"])
    Q = synth.knn_query(e["NQ"], e["D"])
    L = synth.knn_labels(e["NT"], e["C"])
    lab, idx = O.knn(X, L, Q, e["K"], e["C"], threads=2)
    assert lab.tolist() == [int(v) for v in e["stdout"].split()]


@pytest.mark.parametrize("ix", [0, 1])
def test_kmer_oracle_matches_reference(ix, golden):
    e = golden["kmer"][ix]
    E = synth.kmer_emission(e["kmer"], e["K"])
    obs = synth.hmm_obs(e["NS"], e["T"], e["K"])
    got = O.kmer_forward(e["kmer"], e["p_stay"], e["p_step"], E, obs, threads=2)
    want = [float(v) for v in e["stdout"].split()]
    assert np.allclose(got, want, rtol=1e-13, atol=0)


def test_chunks_rule():
    # _chunks (pmx/interp.py:273-276)
    import ctypes as C
    lo, hi = C.c_int64(), C.c_int64()
    spans = []
    for i in range(4):
        O.lib().oracle_chunk(10, 4, i, C.byref(lo), C.byref(hi))
        spans.append((lo.value, hi.value))
    assert spans == [(0, 2), (2, 5), (5, 7), (7, 10)]


def _nn_data():
    # programs/nn.pmx:5-21 (= tests/test_acceptance.py:399-410 of the reference)
    n_in, n_out, n_pts = 16, 8, 32
    x = np.array([[((p * 5 + i * 3) % 11 - 5) / 10.0 for i in range(n_in)] for p in range(n_pts)])
    y = np.array([(p * 7 + 3) % n_out for p in range(n_pts)], np.int32)
    w = np.array([[((i * 3 + j * 7) % 13 - 6) / 20.0 for j in range(n_out)] for i in range(n_in)])
    b = np.array([((j * 5) % 9 - 4) / 15.0 for j in range(n_out)])
    return x, y, w, b


def test_nn_oracle_matches_reference_program(golden):
    # the reference ran programs/nn.pmx in accel mode with 4 workers: same
    # chunked reduces, same libm -> bit-identical printed values
    lines = [l for l in golden["program_nn"]["stdout"].splitlines() if l.strip()]
    loss, dw, db = O.nn(*_nn_data(), workers=4)
    assert loss == float(lines[0])
    assert [[float(v) for v in l.split()] for l in lines[1:17]] == dw.tolist()
    assert [float(v) for v in lines[17].split()] == db.tolist()


def test_nn_oracle_label_out_of_range():
    x, y, w, b = _nn_data()
    y = y.copy()
    y[5] = 8
    with pytest.raises(ValueError, match="point 5"):
        O.nn(x, y, w, b)

"""Case-study bindings of the whole-program drop-in.

The generic adapter (pmx_adapter.py) runs an accelerated construct on the
B200 when its function argument is a scalar lambda.  The paper's case-study
programs are whole accelerated *bindings* instead — `runAll params`
(programs/rk4.pmx), `viterbi trans emit init obs` (programs/viterbi.pmx),
`gradients xs ys w b` (programs/nn.pmx) and the Appendix A programs of the
BASELINE configs (HMM forward, k-NN, k-mer forward) — whose bodies build
nested sequences, records and recursions that this backend executes as one
hand-written kernel each (csrc/rk4.cu, viterbi.cu, nn.cu, hmm*.cu, knn*.cu,
kmer.cu), as the paper's compiler maps them to CUDA.

`recognise(fn, args, ...)` identifies such a binding by its structure: the
lifted body and every closure it reaches (pmx/interp.py:178-220 AccelFn and
Closure values) are reduced to a canonical token string — binders as de
Bruijn indices, captured scalars / sequences and literals as typed holes —
whose digest is looked up in SIGNATURES.  The binder then checks the literal
values the kernel hard-codes (e.g. the pendulum's coefficients in rk4.pmx's
`deriv`) and reads the run-time parameters (sizes, step count, h, p_stay...)
from the holes.  A binding that does not match keeps the generic path.

The signatures are produced by tools/dropin_signatures.py from the programs
in tests/golden/golden.json (run with the reference installed).
"""
from __future__ import annotations

import hashlib
from typing import Any, Callable, Optional

import numpy as np


class NotRecognised(Exception):
    pass


class Canon:
    """Canonical token string of an accelerated binding."""

    def __init__(self, syn, rt):
        self.S, self.R = syn, rt
        self.toks: list[str] = []
        self.lits: list = []          # literal values, traversal order
        self.caps: list = []          # (name, value) captured from environments, traversal order
        self.active: dict = {}        # id(closure) -> index while being expanded

    def fn(self, params, body, env) -> "Canon":
        scope = {p: i for i, p in enumerate(params)}
        self.toks.append(f"fn{len(params)}")
        self.expr(body, scope, len(params), env)
        return self

    def digest(self) -> str:
        return hashlib.sha1("|".join(self.toks).encode()).hexdigest()[:20]

    # -- values captured from an environment
    def value(self, v, name: str):
        R = self.R
        t = self.toks
        if isinstance(v, bool):
            t.append("cap:bool"); self.caps.append((name, v)); return
        if isinstance(v, int):
            t.append("cap:int"); self.caps.append((name, v)); return
        if isinstance(v, float):
            t.append("cap:float"); self.caps.append((name, v)); return
        if isinstance(v, str):
            t.append("cap:char"); self.caps.append((name, v)); return
        if isinstance(v, list):
            t.append("cap:seq"); self.caps.append((name, v)); return
        if isinstance(v, dict):
            t.append("cap:rec"); self.caps.append((name, v)); return
        if isinstance(v, R.TensorView):
            t.append("cap:tensor"); self.caps.append((name, v)); return
        if isinstance(v, R.BuiltinPartial):
            t.append(f"bp:{v.name}:{len(v.args)}(")
            for a in v.args:
                self.value(a, name)
            t.append(")")
            return
        if isinstance(v, R.Closure):
            k = id(v)
            if k in self.active:
                t.append(f"rec{self.active[k]}")
                return
            self.active[k] = len(self.active)
            t.append("clo(")
            self.expr(v.body, {v.param: 0}, 1, v.env)
            t.append(")")
            del self.active[k]
            return
        raise NotRecognised(f"captured {type(v).__name__}")

    def bind(self, scope, level, *names):
        s = dict(scope)
        for n in names:
            s[n] = level
            level += 1
        return s, level

    def pattern(self, p, scope, level):
        S = self.S
        if isinstance(p, S.PVar):
            self.toks.append("pv")
            return self.bind(scope, level, p.name)
        if isinstance(p, S.PConst):
            self.const(p.const)
            return scope, level
        if isinstance(p, S.PRecord):
            self.toks.append(f"pr{len(p.fields)}")
            for label, sub in p.fields:
                self.toks.append(f"l:{label}")
                scope, level = self.pattern(sub, scope, level)
            return scope, level
        raise NotRecognised(f"pattern {type(p).__name__}")

    def const(self, c):
        S = self.S
        if isinstance(c, S.CBuiltin):
            self.toks.append(f"bi:{c.name}")
            return
        kind = type(c).__name__
        self.toks.append(f"lit:{kind}")
        self.lits.append(c.value)

    def expr(self, e, scope, level, env):
        S, t = self.S, self.toks
        if isinstance(e, S.Var):
            if e.name in scope:
                t.append(f"v{level - 1 - scope[e.name]}")
                return
            try:
                v = env.lookup(e.name)
            except AssertionError:
                raise NotRecognised(f"unbound {e.name.text}") from None
            self.value(v, e.name.text)
            return
        if isinstance(e, S.ConstE):
            self.const(e.const)
            return
        if isinstance(e, S.Lam):
            t.append("lam(")
            s2, l2 = self.bind(scope, level, e.param)
            self.expr(e.body, s2, l2, env)
            t.append(")")
            return
        if isinstance(e, S.App):
            t.append("app(")
            self.expr(e.fn, scope, level, env)
            self.expr(e.arg, scope, level, env)
            t.append(")")
            return
        if isinstance(e, S.Let):
            t.append("let(")
            self.expr(e.value, scope, level, env)
            s2, l2 = self.bind(scope, level, e.name)
            self.expr(e.body, s2, l2, env)
            t.append(")")
            return
        if isinstance(e, S.RecLets):
            t.append(f"rec{len(e.bindings)}(")
            s2, l2 = self.bind(scope, level, *[b.name for b in e.bindings])
            for b in e.bindings:
                self.expr(b.value, s2, l2, env)
            self.expr(e.body, s2, l2, env)
            t.append(")")
            return
        if isinstance(e, S.Match):
            t.append("match(")
            self.expr(e.scrut, scope, level, env)
            s2, l2 = self.pattern(e.pat, scope, level)
            self.expr(e.thn, s2, l2, env)
            self.expr(e.els, scope, level, env)
            t.append(")")
            return
        if isinstance(e, S.Never):
            t.append("never")
            return
        if isinstance(e, S.RecordE):
            t.append(f"record{len(e.fields)}(")
            for label, x in e.fields:
                t.append(f"l:{label}")
                self.expr(x, scope, level, env)
            t.append(")")
            return
        if isinstance(e, S.SeqE):
            t.append(f"seq{len(e.items)}(")
            for x in e.items:
                self.expr(x, scope, level, env)
            t.append(")")
            return
        for cls, fields in ((S.MapE, ("fn", "seq")), (S.Map2E, ("fn", "seq1", "seq2")),
                            (S.ReduceE, ("fn", "acc", "seq")), (S.FlattenE, ("seq",)),
                            (S.LoopE, ("count", "fn")), (S.Accelerate, ("operand",))):
            if isinstance(e, cls):
                t.append(cls.__name__ + "(")
                for f in fields:
                    self.expr(getattr(e, f), scope, level, env)
                t.append(")")
                return
        raise NotRecognised(f"{type(e).__name__}")


def canon(fn, syn, rt) -> Canon:
    """The canonical form of an AccelFn (params, body, env)."""
    return Canon(syn, rt).fn(fn.params, fn.body, fn.env)


# ====================================================== binders
# A binder gets (args, canon) and returns a callable producing the binding's
# result as reference values (computed on the B200), or raises NotRecognised.

def _floats(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64)


def _need(cond: bool, what: str):
    if not cond:
        raise NotRecognised(what)


SIGNATURES: dict[str, tuple[str, Callable]] = {}


def signature(digest: str, family: str):
    def deco(f):
        SIGNATURES[digest] = (family, f)
        return f
    return deco


def recognise(fn, args: list, syn, rt):
    """(family, thunk) for a recognised case-study binding, else None."""
    try:
        c = canon(fn, syn, rt)
    except NotRecognised:
        return None
    hit = SIGNATURES.get(c.digest())
    if hit is None:
        return None
    family, binder = hit
    try:
        return family, binder(args, c)
    except NotRecognised:
        return None


def _host(seq) -> np.ndarray:
    from .runtime import seq_to_host
    return seq_to_host(seq)


def _regular(rows, what: str) -> np.ndarray:
    _need(isinstance(rows, list) and len(rows) > 0 and all(isinstance(r, list) for r in rows), what)
    n = len(rows[0])
    _need(all(len(r) == n for r in rows), f"{what}: irregular rows")
    return np.asarray(rows)


# programs/rk4.pmx (and its parameter-sweep variants): runAll params with
# integrate p initState numSteps, the pendulum `deriv` and the classical
# RK4 `step` (programs/rk4.pmx:11-45) -> csrc/rk4.cu
RK4_LITS = [0, True, 0, 1, 2, 3, 0.2, 0.3, 9.81, 0.1, 0, 1, 2, 3, 0.2, 0.3, 9.81, 0.1, 2.0, 0, 1, 2, 3, 0.2, 0.3,
            9.81, 0.1, 2.0, 0, 1, 2, 3, 0.2, 0.3, 9.81, 0.1, 4, 6.0, 2.0, 2.0, 1]


@signature("35c038d63f963a0437cc", "rk4")
def _rk4(args, c):
    num_steps, h, params, init = args
    _need(c.lits == RK4_LITS, "rk4: model constants differ from csrc/rk4.cu")
    _need(isinstance(num_steps, int) and num_steps >= 0 and isinstance(h, float), "rk4: step count / size")
    _need(isinstance(init, list) and len(init) == 4 and all(isinstance(v, float) for v in init), "rk4: state")
    _need(isinstance(params, list) and all(isinstance(p, float) for p in params), "rk4: parameters")

    def run():
        from .casestudies import rk4_sweep
        if not params:
            return []
        out = _host(rk4_sweep(_floats(params), _floats(init), num_steps, h))
        return [[float(v) for v in row] for row in out]
    return run


# programs/viterbi.pmx: viterbi trans emit init obs (viterbi.pmx:23-59) -> csrc/viterbi.cu
@signature("0bbb44ced84cecb72236", "viterbi")
def _viterbi(args, c):
    S, state_idx, trans, emit, init, obs = args
    _need(c.lits == [0, True, True, 0, 1, 1, True, 0, 0, True, 1, 2], "viterbi: program constants")
    _need(state_idx == list(range(S)), "viterbi: stateIdx must be [0 .. numStates)")
    A, E = _regular(trans, "transition"), _regular(emit, "emission")
    _need(A.shape == (S, S) and E.shape[0] == S and len(init) == S, "viterbi: model shapes")
    o = np.asarray(obs, dtype=np.int64)
    _need(o.ndim == 1 and o.size >= 1 and o.min() >= 0 and o.max() < E.shape[1], "viterbi: observations")

    def run():
        from .casestudies import viterbi
        r = viterbi(A.astype(np.float64), E.astype(np.float64), _floats(init), o.astype(np.int32))
        path = [int(v) for v in _host(r["path"]).reshape(-1)]
        return {"path": path, "logp": float(_host(r["logp"]).reshape(-1)[0])}
    return run


# programs/nn.pmx: gradients xs ys w b (nn.pmx:22-49) -> csrc/nn.cu
@signature("fd52e651f1de4a328724", "nn")
def _nn(args, c):
    nin, nout, in_idx, xs, ys, w, b = args
    _need(c.lits == [0.0, 0.0, True, 1.0, 0.0, 0.0, 0.0], "nn: program constants")
    _need(in_idx == list(range(nin)) and 0 < nin <= 64 and 0 < nout <= 32, "nn: sizes")
    X, W = _regular(xs, "xs"), _regular(w, "w")
    _need(X.shape[1] == nin and W.shape == (nin, nout) and len(b) == nout and len(ys) == len(xs), "nn: shapes")

    def run():
        from .casestudies import nn_gradients
        r = nn_gradients(X.astype(np.float64), np.asarray(ys, dtype=np.int32), W.astype(np.float64), _floats(b))
        dw = _host(r["dw"]).reshape(nin, nout)
        return {"loss": float(r["loss"].get()), "dw": [[float(v) for v in row] for row in dw],
                "db": [float(v) for v in _host(r["db"]).reshape(-1)]}
    return run


# SURVEY Appendix A.1 hmm_forward.pmx: forwardAll trans emit init sigs -> csrc/hmm*.cu
@signature("4fa7dbc7340d1ab36927", "hmm_forward")
def _hmm_forward(args, c):
    S, K, trans, emit, init, sigs = args
    _need(c.lits == [0, True, 0, 0.0, True, 1, True, 0, 0.0, 1], "hmm_forward: program constants")
    A, E = _regular(trans, "transition"), _regular(emit, "emission")
    _need(A.shape == (S, S) and E.shape == (S, K) and len(init) == S, "hmm_forward: model shapes")
    O = _regular(sigs, "signals").astype(np.int64)
    _need(O.shape[1] >= 1 and O.min() >= 0 and O.max() < K, "hmm_forward: observations")

    def run():
        from .casestudies import hmm_forward
        return [float(v) for v in _host(hmm_forward(A.astype(np.float64), E.astype(np.float64), _floats(init),
                                                    O.astype(np.int32)))]
    return run


# SURVEY Appendix A.2 knn.pmx: classify train labels queries -> csrc/knn*.cu.
# The kernels rank fp32 distances; the drop-in takes them only when every
# distance is exact in fp32 (integer coordinates, small range), so the ranking
# equals the reference's fp64 one.
@signature("5520330c20b0ab8c60c0", "knn")
def _knn(args, c):
    ntr, k, ncls, dim_idx, cls_idx, train, labels, queries = args
    _need(c.lits == [1e+308, 9223372036854775807, True, True, True, True, False, True, 1, 1, 0.0, 0, True, 1, 0,
                     True, 0], "knn: program constants")
    X, Q = _regular(train, "train"), _regular(queries, "queries")
    d = len(dim_idx)
    _need(dim_idx == list(range(d)) and cls_idx == list(range(ncls)) and X.shape == (ntr, d) and Q.shape[1] == d,
          "knn: shapes")
    L = np.asarray(labels, dtype=np.int64)
    _need(L.shape == (ntr,) and (L.size == 0 or (L.min() >= 0 and L.max() < ncls)) and 1 <= k <= ntr <= (1 << 31) - 1,
          "knn: labels / k")
    both = np.concatenate([X.reshape(-1), Q.reshape(-1)]).astype(np.float64)
    m = float(np.max(np.abs(both))) if both.size else 0.0
    _need(np.all(both == np.round(both)) and d * (2 * m) ** 2 < 2 ** 24, "knn: distances not exact in fp32")

    def run():
        from .casestudies import knn_classify
        out = knn_classify(X.astype(np.float32), L.astype(np.int32), Q.astype(np.float32), int(k), int(ncls))
        return [int(v) for v in _host(out)]
    return run


# the k-mer (de Bruijn) forward of SURVEY §8(d): forwardAll emit sigs with
# p_stay / p_step as literals -> csrc/kmer.cu
@signature("179012a43d4536b334ce", "hmm_kmer")
def _kmer(args, c):
    S, hi, K, emit, sigs = args
    _need(c.lits[2:] == [1.0, 0, True, 0, 0.0, True, 1, 4, True, 0, 0.0, 2, 3, 1], "kmer: program constants")
    p_stay, p_step = c.lits[0], c.lits[1]
    _need(isinstance(p_stay, float) and isinstance(p_step, float) and p_stay > 0 and p_step > 0, "kmer: p")
    kmer = (S.bit_length() - 1) // 2
    _need(S >= 4 and (1 << (2 * kmer)) == S and hi * 4 == S and 1 <= kmer <= 10, "kmer: state count")
    E = _regular(emit, "emission")
    _need(E.shape == (S, K), "kmer: emission shape")
    O = _regular(sigs, "signals").astype(np.int64)
    _need(O.shape[1] >= 1 and O.min() >= 0 and O.max() < K, "kmer: observations")

    def run():
        from .casestudies import hmm_kmer_forward
        return [float(v) for v in _host(hmm_kmer_forward(kmer, p_stay, p_step, E.astype(np.float64),
                                                         O.astype(np.int32)))]
    return run

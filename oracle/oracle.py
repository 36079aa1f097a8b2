"""CPU oracle for the accelerated-expression hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  It is the checker, never the thing
measured as the product or shipped on the product path.

Two parts:
  * liboracle.so (oracle/pmx_oracle.c): C restatement of the reference's
    case-study algorithms and of the map/reduce skeleton semantics, OpenMP
    parallel over independent elements (the CPU baseline);
  * ir_* below: a pure-Python evaluator of this repo's lambda IR with the
    reference's scalar semantics (pmx/interp.py:379-436) and skeleton
    semantics (eval_map/eval_map2/eval_reduce/_fold, interp.py:294-343), for
    small cases.
Both are pinned against the reference's own outputs in tests/golden.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: build it with __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        P = C.c_void_p
        L.oracle_map_affine_reduce_add.restype = C.c_double
        L.oracle_map_affine_reduce_add.argtypes = [P, C.c_int64, C.c_double, C.c_double, C.c_double,
                                                   C.c_int64, C.c_int, P]
        L.oracle_rk4.argtypes = [P, C.c_int64, P, C.c_int, C.c_double, P, C.c_int]
        L.oracle_rk4_trace.argtypes = [P, C.c_int64, P, C.c_int, C.c_double, P, C.c_int, P, C.c_int]
        L.oracle_hmm_forward.argtypes = [P, P, P, C.c_int, C.c_int, P, C.c_int64, C.c_int, P, C.c_int]
        L.oracle_viterbi.argtypes = [P, P, P, C.c_int, C.c_int, P, C.c_int64, C.c_int, P, P, C.c_int]
        L.oracle_knn.argtypes = [P, P, C.c_int64, P, C.c_int64, C.c_int, C.c_int, C.c_int, P, P, C.c_int]
        L.oracle_kmer_forward.argtypes = [C.c_int, C.c_double, C.c_double, P, C.c_int, P, C.c_int64,
                                          C.c_int, P, C.c_int]
        L.oracle_hmm_forward_scaled.argtypes = [P, P, P, C.c_int, C.c_int, P, C.c_int64, C.c_int, P, C.c_int]
        L.oracle_kmer_forward_scaled.argtypes = [C.c_int, C.c_double, C.c_double, P, C.c_int, P, C.c_int64,
                                                 C.c_int, P, C.c_int]
        L.oracle_nn.restype = C.c_int64
        L.oracle_nn.argtypes = [P, P, P, P, C.c_int64, C.c_int, C.c_int, C.c_int64, P, P, P, C.c_int]
        L.oracle_max_threads.restype = C.c_int
        _lib = L
    return _lib


def threads_default() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def map_affine_reduce_add(x: np.ndarray, a: float = 2.0, b: float = 1.0, acc: float = 0.0,
                          workers: int = 1, threads: int | None = None, want_y: bool = False):
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty(x.size, np.float64) if want_y else None
    s = lib().oracle_map_affine_reduce_add(_p(x), x.size, a, b, acc, workers, threads or threads_default(),
                                           _p(y) if y is not None else None)
    return (s, y) if want_y else s


def rk4(params: np.ndarray, init4, steps: int, h: float, threads: int | None = None) -> np.ndarray:
    p = np.ascontiguousarray(params, dtype=np.float64)
    s0 = np.ascontiguousarray(init4, dtype=np.float64)
    out = np.empty((p.size, 4), np.float64)
    lib().oracle_rk4(_p(p), p.size, _p(s0), steps, h, _p(out), threads or threads_default())
    return out


def rk4_trace(params, init4, steps: int, h: float, comp: int, threads: int | None = None):
    """(final states [N][4], trace [N][steps] of state `comp`) — PAPER.md:1435-1440."""
    p = np.ascontiguousarray(params, dtype=np.float64)
    s0 = np.ascontiguousarray(init4, dtype=np.float64)
    out = np.empty((p.size, 4), np.float64)
    tr = np.empty((p.size, steps), np.float64)
    lib().oracle_rk4_trace(_p(p), p.size, _p(s0), steps, h, _p(out), comp, _p(tr), threads or threads_default())
    return out, tr


def hmm_forward(A, E, pi, obs, threads: int | None = None) -> np.ndarray:
    A = np.ascontiguousarray(A, np.float64)
    E = np.ascontiguousarray(E, np.float64)
    pi = np.ascontiguousarray(pi, np.float64)
    obs = np.ascontiguousarray(obs, np.int32)
    S, K = E.shape
    nsig, T = obs.shape
    ll = np.empty(nsig, np.float64)
    lib().oracle_hmm_forward(_p(A), _p(E), _p(pi), S, K, _p(obs), nsig, T, _p(ll), threads or threads_default())
    return ll


def hmm_forward_scaled(A, E, pi, obs, threads: int | None = None) -> np.ndarray:
    """hmm_forward in scaled linear form (fp64, signals batched): the sampled
    full-size parity checks (S = 1024, T = 10^4).  Same values as hmm_forward
    to ~1e-13 relative (tests/test_oracle.py)."""
    A = np.ascontiguousarray(A, np.float64)
    E = np.ascontiguousarray(E, np.float64)
    pi = np.ascontiguousarray(pi, np.float64)
    obs = np.ascontiguousarray(obs, np.int32)
    S, K = E.shape
    nsig, T = obs.shape
    ll = np.empty(nsig, np.float64)
    lib().oracle_hmm_forward_scaled(_p(A), _p(E), _p(pi), S, K, _p(obs), nsig, T, _p(ll),
                                    threads or threads_default())
    return ll


def viterbi(A, E, pi, obs, threads: int | None = None):
    A = np.ascontiguousarray(A, np.float64)
    E = np.ascontiguousarray(E, np.float64)
    pi = np.ascontiguousarray(pi, np.float64)
    obs = np.ascontiguousarray(np.atleast_2d(obs), np.int32)
    S, K = E.shape
    nsig, T = obs.shape
    path = np.empty((nsig, T), np.int32)
    logp = np.empty(nsig, np.float64)
    lib().oracle_viterbi(_p(A), _p(E), _p(pi), S, K, _p(obs), nsig, T, _p(path), _p(logp),
                         threads or threads_default())
    return path, logp


def knn(train, labels, query, k: int, ncls: int, threads: int | None = None):
    X = np.ascontiguousarray(train, np.float32)
    Q = np.ascontiguousarray(query, np.float32)
    L = np.ascontiguousarray(labels, np.int32)
    ntr, d = X.shape
    nq = Q.shape[0]
    out = np.empty(nq, np.int32)
    idx = np.empty((nq, k), np.int32)
    lib().oracle_knn(_p(X), _p(L), ntr, _p(Q), nq, d, k, ncls, _p(out), _p(idx), threads or threads_default())
    return out, idx


def kmer_forward(kmer: int, p_stay: float, p_step: float, E, obs, threads: int | None = None) -> np.ndarray:
    log_E = np.ascontiguousarray(np.log(np.asarray(E, np.float64)))
    obs = np.ascontiguousarray(obs, np.int32)
    nsig, T = obs.shape
    K = log_E.shape[1]
    ll = np.empty(nsig, np.float64)
    lib().oracle_kmer_forward(kmer, p_stay, p_step, _p(log_E), K, _p(obs), nsig, T, _p(ll),
                              threads or threads_default())
    return ll


def kmer_forward_scaled(kmer: int, p_stay: float, p_step: float, E, obs, threads: int | None = None) -> np.ndarray:
    """kmer_forward in scaled linear form (fp64): the sampled full-size parity
    checks (S = 65,536, T = 6000).  Same values as kmer_forward to ~1e-13."""
    E = np.ascontiguousarray(E, np.float64)
    obs = np.ascontiguousarray(obs, np.int32)
    nsig, T = obs.shape
    K = E.shape[1]
    ll = np.empty(nsig, np.float64)
    lib().oracle_kmer_forward_scaled(kmer, p_stay, p_step, _p(E), K, _p(obs), nsig, T, _p(ll),
                                     threads or threads_default())
    return ll


# =========================================================== IR evaluator
class OracleError(Exception):
    """A reference RuntimeError (message text of pmx/interp.py:379-436)."""


_MIN = -(1 << 63)


def _wrap(x: int) -> int:            # pmx/interp.py:32-37
    return ((x - _MIN) & ((1 << 64) - 1)) + _MIN


def _prim(name: str, a: list, types: list):
    t = types[0] if types else None
    if name in ("add", "sub", "mul", "div", "neg", "lt", "gt", "le", "ge", "eq", "ne"):
        f = t == "float"
        name = {"add": "addf" if f else "addi", "sub": "subf" if f else "subi",
                "mul": "mulf" if f else "muli", "div": "divf" if f else "divi",
                "neg": "negf" if f else "negi", "lt": "lt", "gt": "gt", "le": "le", "ge": "ge",
                "eq": "eq", "ne": "ne"}[name]
    x = a[0]
    y = a[1] if len(a) > 1 else None
    if name == "addi": return _wrap(x + y)
    if name == "subi": return _wrap(x - y)
    if name == "muli": return _wrap(x * y)
    if name in ("divi", "modi"):
        if y == 0:
            raise OracleError("integer division by zero" if name == "divi" else "integer modulo by zero")
        q = abs(x) // abs(y)
        if (x < 0) != (y < 0):
            q = -q
        return _wrap(q) if name == "divi" else _wrap(x - q * y)
    if name == "negi": return _wrap(-x)
    if name == "addf": return x + y
    if name == "subf": return x - y
    if name == "mulf": return x * y
    if name == "divf":
        if y == 0.0:
            raise OracleError("float division by zero")
        return x / y
    if name == "negf": return -x
    if name in ("eqi", "eqf", "eq"): return x == y
    if name in ("neqi", "ne"): return x != y
    if name in ("lti", "ltf", "lt"): return x < y
    if name in ("gti", "gtf", "gt"): return x > y
    if name in ("leqi", "leqf", "le"): return x <= y
    if name in ("geqi", "geqf", "ge"): return x >= y
    if name == "int2float": return float(x)
    if name == "floor": return _wrap(math.floor(x))
    if name in ("exp", "log", "sin", "cos"):
        try:
            return getattr(math, name)(x)
        except (ValueError, OverflowError) as exc:
            raise OracleError(f"{name}: {exc}") from None
    if name == "sqrtf":
        if x < 0:
            raise OracleError("sqrtf of a negative number")
        return math.sqrt(x)
    raise OracleError(f"unsupported builtin {name}")


def _ty(v) -> str:
    return "float" if isinstance(v, float) else ("bool" if isinstance(v, bool) else "int")


def ir_eval(e, env: dict):
    from paper_2211_00621_b200 import lambdas as L
    if isinstance(e, L.Var):
        return env[e.name]
    if isinstance(e, L.Const):
        return bool(e.value) if e.ty == "bool" else e.value
    if isinstance(e, L.Prim):
        args = [ir_eval(x, env) for x in e.args]
        return _prim(e.name, args, [_ty(v) for v in args])
    if isinstance(e, L.If):
        return ir_eval(e.then if ir_eval(e.cond, env) else e.els, env)
    if isinstance(e, L.LetE):
        env2 = dict(env)
        env2[e.name] = ir_eval(e.value, env)
        return ir_eval(e.body, env2)
    if isinstance(e, L.Never):
        raise OracleError("reached a never expression (no pattern matched)")
    if isinstance(e, L.Get):                 # interp.py:448-451 + _seq_bounds 536-541
        i = ir_eval(e.index, env)
        n = e.arr.shape[0]
        if not 0 <= i < n:
            raise OracleError(f"get index {i} out of bounds for sequence of length {n}")
        return e.arr.data[e.arr.offset + i]
    if isinstance(e, L.Len):
        return e.arr.shape[0]
    if isinstance(e, (L.TGet, L.TSet)):      # interp.py:468-474, runtime.py:63-75
        t = e.tensor
        idx = [ir_eval(x, env) for x in e.index]
        pos, stride = t.offset, 1
        for d in range(len(t.shape) - 1, -1, -1):
            if not 0 <= idx[d] < t.shape[d]:
                raise OracleError(f"tensor index {idx[d]} out of bounds for dimension {d} of size {t.shape[d]}")
            pos += idx[d] * stride
            stride *= t.shape[d]
        if isinstance(e, L.TGet):
            return t.data[pos]
        t.data[pos] = ir_eval(e.value, env)
        return 0
    if isinstance(e, L.Do):
        out = 0
        for x in e.exprs:
            out = ir_eval(x, env)
        return out
    if isinstance(e, L.Field):
        return ir_eval(e.rec, env)[e.label]
    if isinstance(e, L.Iterate):             # k-term recursion, base cases upward
        lo, hi = ir_eval(e.lo, env), ir_eval(e.hi, env)
        k = 1 + len(e.more)
        if hi - lo > L.ITERATE_LIMIT or hi - lo < -k:
            raise OracleError("maximum recursion depth exceeded")
        names = [e.acc] + [n for n, _ in e.more]
        inits = [e.init] + [x for _, x in e.more]
        # accs[j] = f(lo - 1 - j); a base case is evaluated only when hi reaches it
        accs = [ir_eval(x, env) if hi >= lo - 1 - j else 0 for j, x in enumerate(inits)]
        if hi < lo:
            return accs[lo - 1 - hi]
        for m in range(lo, hi + 1):
            env2 = dict(env)
            env2[e.var] = m
            env2.update(zip(names, accs))
            accs = [ir_eval(e.body, env2)] + accs[:-1]
        return accs[0]
    raise OracleError(f"ir_eval: unsupported node {type(e).__name__}")


def ir_apply(f, *args):
    from paper_2211_00621_b200.lambdas import as_lam
    fl = as_lam(f)
    return ir_eval(fl.body, dict(zip(fl.params, args)))


def ir_map(f, xs):                      # eval_map, interp.py:294-304
    return [ir_apply(f, x) for x in xs]


def ir_map2(f, xs, ys):                 # eval_map2 + length check, interp.py:151-154, 307-319
    if len(xs) != len(ys):
        raise OracleError(f"map2 over sequences of different lengths ({len(xs)} and {len(ys)})")
    return [ir_apply(f, x, y) for x, y in zip(xs, ys)]


def ir_fold(f, acc, xs):                # _fold, interp.py:322-325
    for x in xs:
        acc = ir_apply(f, acc, x)
    return acc


def ir_reduce(f, acc, xs, workers: int = 1):   # eval_reduce, interp.py:328-343
    if workers <= 1 or not xs:
        return ir_fold(f, acc, xs)
    n = len(xs)
    spans = [(i * n // workers, (i + 1) * n // workers) for i in range(workers)]
    parts = [ir_fold(f, acc, xs[lo:hi]) for lo, hi in spans if lo < hi]
    total = parts[0]
    for p in parts[1:]:
        total = ir_apply(f, total, p)
    return total


def nn(x, y, w, b, workers: int = 4, threads: int | None = None):
    """(loss, dw, db) of programs/nn.pmx:22-49 with the reference's chunked
    top-level reduces over `workers` chunks (one OpenMP thread per chunk, up to
    `threads`).  Raises ValueError on a label out of range (the reference's get
    error)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.int32)
    w = np.ascontiguousarray(w, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    npts, nin = x.shape
    nout = b.size
    loss = np.zeros(1, np.float64)
    dw = np.empty((nin, nout), np.float64)
    db = np.empty(nout, np.float64)
    bad = lib().oracle_nn(_p(x), _p(y), _p(w), _p(b), npts, nin, nout, workers, _p(loss), _p(dw), _p(db),
                         threads or threads_default())
    if bad:
        raise ValueError(f"label out of range at point {bad - 1}")
    return float(loss[0]), dw, db

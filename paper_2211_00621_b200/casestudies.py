"""The paper's case-study kernels behind the accelerate entry point.

Each function is the device form of an accelerate binding of the reference's
case-study programs (or of the SURVEY Appendix A programs for the BASELINE
configs the reference has no program for).  Arguments may be host values
(marshalled here) or device values inside `accelerate`; results are device
values (host values when called outside accelerate through `accelerate`).

    rk4_sweep         programs/rk4.pmx:42-45             (runAll params)
    hmm_forward       SURVEY Appendix A.1 hmm_forward.pmx (forwardAll ...)
    viterbi           programs/viterbi.pmx:23-59          (viterbi trans emit init obs)
    knn_classify      SURVEY Appendix A.2 knn.pmx          (classify train labels queries)
    hmm_kmer_forward  SURVEY §8(d) nanopore k-mer model
    nn_gradients      programs/nn.pmx:22-49               (gradients xs ys w b)
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .diagnostics import runtime_error
from .runtime import DeviceSeq, _device, seq_to_device
from .lambdas import lam, log as _log
from .runtime import pmx_code_of_torch
from .skeletons import default_ctx, map_tensor


def _dev(x, dtype):
    """Host or device sequence -> contiguous device tensor of `dtype`
    (conversion by the library's map kernel, not by torch)."""
    if isinstance(x, DeviceSeq):
        t = x.data
    elif isinstance(x, torch.Tensor):
        t = x if x.is_cuda else seq_to_device(x).data
    else:
        t = seq_to_device(np.asarray(x)).data
    t = t.contiguous().reshape(-1)
    if t.dtype == dtype:
        return t
    return map_tensor(lam("v", "v"), t, pmx_code_of_torch(dtype))


def _dev_log(x, dtype):
    """log of a device/host sequence of probabilities, on the device (the
    programs take logs inside the accelerated region, viterbi.pmx:140-141);
    log of a non-positive value raises the reference's domain error."""
    t = _dev(x, torch.float64)
    return map_tensor(lam("p", _log("p")), t, pmx_code_of_torch(dtype))


def _stream():
    return default_ctx().stream_ptr()


def _count():
    default_ctx().launches += 1


# ------------------------------------------------------------------ RK4
def rk4_sweep(params, init4, steps: int, h: float) -> DeviceSeq:
    """out[k] = integrate p_k init steps (programs/rk4.pmx:38-45), fp64."""
    p = _dev(params, torch.float64)
    s0 = _dev(init4, torch.float64)
    if s0.numel() != 4:
        raise runtime_error("rk4: the state has 4 components")
    n = p.numel()
    out = torch.empty(n * 4, dtype=torch.float64, device=_device())
    rc = _lib.load().pmx_rk4_sweep_f64(p.data_ptr(), n, s0.data_ptr(), int(steps), float(h),
                                       out.data_ptr(), _stream())
    _lib.check(rc, "rk4_sweep")
    _count()
    return DeviceSeq(out, (n, 4), _lib.PMX_F64)


def rk4_trace(params, init4, steps: int, h: float, comp: int = 2, trace=None):
    """The paper's ODE study: N simulation traces of one
    measured state component, an N x M tensor with trace[k][m] = component
    `comp` of integrate p_k after m + 1 steps.  `trace` may be a tensor view
    marshalled into the accelerated region (written in place in its device
    root, like the paper's `loop ... tensorSet`); otherwise a new N x M
    sequence is returned.  Returns (trace, final states)."""
    from .runtime import DeviceTensor
    p = _dev(params, torch.float64)
    s0 = _dev(init4, torch.float64)
    if s0.numel() != 4:
        raise runtime_error("rk4: the state has 4 components")
    n = p.numel()
    out = torch.empty(n * 4, dtype=torch.float64, device=_device())
    if isinstance(trace, DeviceTensor):
        if tuple(trace.shape) != (n, int(steps)) or trace.root.dtype_code != _lib.PMX_F64:
            raise runtime_error(f"rk4_trace: trace tensor must be [{n}][{steps}] Float, got {list(trace.shape)}")
        ptr = trace.root.data.data_ptr() + 8 * trace.offset
        trace.root.dirty = True           # written root: copied back by marshal_out
        res = trace
    else:
        buf = torch.empty(n * int(steps), dtype=torch.float64, device=_device())
        ptr = buf.data_ptr()
        res = DeviceSeq(buf, (n, int(steps)), _lib.PMX_F64)
    rc = _lib.load().pmx_rk4_trace_f64(p.data_ptr(), n, s0.data_ptr(), int(steps), float(h), int(comp), ptr,
                                       out.data_ptr(), _stream())
    _lib.check(rc, "rk4_trace")
    _count()
    return res, DeviceSeq(out, (n, 4), _lib.PMX_F64)


# ------------------------------------------------------------------ HMM
class HMMWorkspace:
    def __init__(self):
        self.buf = None

    def get(self, nbytes: int):
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=_device())
        return self.buf


_ws = HMMWorkspace()


def hmm_forward(trans, emit, init, obs) -> DeviceSeq:
    """Log-likelihood of each observation row (Appendix A.1 forwardAll).

    trans [S][S], emit [S][K], init [S] are probabilities (as in the program,
    which takes logs on the device); obs [nsig][T] symbols.  fp32 trellis with
    an fp64 log-scale; returns fp64 [nsig]."""
    A = _dev(trans, torch.float32)
    log_E = _dev_log(emit, torch.float32)
    log_pi = _dev_log(init, torch.float32)
    o = _dev(obs, torch.int32)
    S = log_pi.numel()
    K = log_E.numel() // S
    if A.numel() != S * S or log_E.numel() != S * K:
        raise runtime_error("hmm_forward: inconsistent model shapes")
    nsig = int(obs.shape[0]) if hasattr(obs, "shape") else len(obs)
    T = o.numel() // max(nsig, 1)
    out = torch.empty(nsig, dtype=torch.float64, device=_device())
    lib = _lib.load()
    nbytes = lib.pmx_hmm_forward_workspace_bytes(S, nsig)
    ws = _ws.get(nbytes)
    rc = lib.pmx_hmm_forward_f32(log_pi.data_ptr(), A.data_ptr(), log_E.data_ptr(), S, K, o.data_ptr(),
                                 nsig, T, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    _lib.check(rc, "hmm_forward")
    _count()
    return DeviceSeq(out, (nsig,), _lib.PMX_F64)


def hmm_forward_rerun_count(S: int, nsig: int, ws=None) -> int:
    """How many signals of the last hmm_forward call (on `ws`, default this
    module's workspace) the fp16 path's range guard re-ran in TF32."""
    buf = ws if ws is not None else _ws.buf
    if buf is None:
        return 0
    n = _lib.load().pmx_hmm_forward_rerun_count(buf.data_ptr(), S, nsig, _stream())
    if n < 0:
        raise RuntimeError("pmx_hmm_forward_rerun_count failed")
    return int(n)


def hmm_forward_raw(log_pi, A, log_E, obs, S: int, K: int, nsig: int, T: int, out, ws) -> None:
    """Device-resident entry used by the benchmark: all arguments are device
    tensors already in the kernel's layout."""
    rc = _lib.load().pmx_hmm_forward_f32(log_pi.data_ptr(), A.data_ptr(), log_E.data_ptr(), S, K,
                                         obs.data_ptr(), nsig, T, out.data_ptr(), ws.data_ptr(),
                                         ws.numel(), _stream())
    _lib.check(rc, "hmm_forward")
    _count()


def viterbi(trans, emit, init, obs):
    """{path, logp} per observation row (programs/viterbi.pmx:23-59), fp64."""
    lt = _dev_log(trans, torch.float64)
    le = _dev_log(emit, torch.float64)
    lp = _dev_log(init, torch.float64)
    o = _dev(obs, torch.int32)
    S = lp.numel()
    K = le.numel() // S
    single = np.ndim(obs) == 1 if not isinstance(obs, (DeviceSeq, torch.Tensor)) else len(getattr(obs, "shape", (0,))) == 1
    nsig = 1 if single else int(obs.shape[0] if hasattr(obs, "shape") else len(obs))
    T = o.numel() // nsig
    path = torch.empty(nsig * T, dtype=torch.int32, device=_device())
    logp = torch.empty(nsig, dtype=torch.float64, device=_device())
    lib = _lib.load()
    ws = _ws.get(lib.pmx_viterbi_workspace_bytes(S, nsig, T))
    rc = lib.pmx_viterbi_f64(lp.data_ptr(), lt.data_ptr(), le.data_ptr(), S, K, o.data_ptr(), nsig, T,
                             path.data_ptr(), logp.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    _lib.check(rc, "viterbi")
    _count()
    if single:
        return {"path": DeviceSeq(path, (T,), _lib.PMX_I32), "logp": DeviceSeq(logp, (1,), _lib.PMX_F64)}
    return {"path": DeviceSeq(path, (nsig, T), _lib.PMX_I32), "logp": DeviceSeq(logp, (nsig,), _lib.PMX_F64)}


# ------------------------------------------------------------------ k-NN
def knn_classify(train, labels, queries, k: int, ncls: int, return_indices: bool = False):
    """Majority label of the k nearest train points per query (Appendix A.2)."""
    X = _dev(train, torch.float32)
    Q = _dev(queries, torch.float32)
    L = _dev(labels, torch.int32)
    ntr = L.numel()
    d = X.numel() // max(ntr, 1)
    nq = Q.numel() // d
    out = torch.empty(nq, dtype=torch.int32, device=_device())
    idx = torch.empty(nq * k, dtype=torch.int32, device=_device()) if return_indices else None
    lib = _lib.load()
    ws = _ws.get(lib.pmx_knn_workspace_bytes(ntr, nq, d, k))
    rc = lib.pmx_knn_f32(X.data_ptr(), L.data_ptr(), ntr, Q.data_ptr(), nq, d, k, ncls, out.data_ptr(),
                         0 if idx is None else idx.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    _lib.check(rc, "knn")
    _count()
    res = DeviceSeq(out, (nq,), _lib.PMX_I32)
    if return_indices:
        return res, DeviceSeq(idx, (nq, k), _lib.PMX_I32)
    return res


def knn_raw(X, L, Q, ntr, nq, d, k, ncls, out, idx, ws) -> None:
    rc = _lib.load().pmx_knn_f32(X.data_ptr(), L.data_ptr(), ntr, Q.data_ptr(), nq, d, k, ncls,
                                 out.data_ptr(), 0 if idx is None else idx.data_ptr(), ws.data_ptr(),
                                 ws.numel(), _stream())
    _lib.check(rc, "knn")
    _count()


# ------------------------------------------------------------ k-mer HMM
def hmm_kmer_forward(kmer: int, p_stay: float, p_step: float, emit, obs) -> DeviceSeq:
    """Forward log-likelihoods on the de Bruijn k-mer model."""
    log_E = _dev_log(emit, torch.float32)
    o = _dev(obs, torch.int32)
    S = 1 << (2 * kmer)
    K = log_E.numel() // S
    nsig = int(obs.shape[0]) if hasattr(obs, "shape") else len(obs)
    T = o.numel() // nsig
    out = torch.empty(nsig, dtype=torch.float64, device=_device())
    lib = _lib.load()
    ws = _ws.get(lib.pmx_hmm_kmer_workspace_bytes(kmer, nsig))
    rc = lib.pmx_hmm_kmer_forward_f32(kmer, float(p_stay), float(p_step), log_E.data_ptr(), K, o.data_ptr(),
                                      nsig, T, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream())
    _lib.check(rc, "hmm_kmer_forward")
    _count()
    return DeviceSeq(out, (nsig,), _lib.PMX_F64)


# ------------------------------------------------------------- NN gradients
def nn_gradients(xs, ys, w, b):
    """{loss, dw, db} of softmax regression (programs/nn.pmx:22-49): mean
    cross-entropy over the points and its analytic gradients, fp64, one fused
    launch.  xs [npts][nin], ys [npts] class labels, w [nin][nout], b [nout]."""
    from .runtime import DeviceScalar
    from .diagnostics import NO_SPAN
    X = _dev(xs, torch.float64)
    Y = _dev(ys, torch.int32)
    W = _dev(w, torch.float64)
    B = _dev(b, torch.float64)
    nout = B.numel()
    nin = W.numel() // max(nout, 1)
    npts = Y.numel()
    if X.numel() != npts * nin:
        raise runtime_error(f"nn_gradients: xs has {X.numel()} values, expected {npts} x {nin}")
    loss = torch.empty(1, dtype=torch.float64, device=_device())
    dw = torch.empty(nin * nout, dtype=torch.float64, device=_device())
    db = torch.empty(nout, dtype=torch.float64, device=_device())
    lib = _lib.load()
    ws = _ws.get(lib.pmx_nn_workspace_bytes(npts, nin, nout))
    err = default_ctx().new_err(NO_SPAN)
    rc = lib.pmx_nn_softmax_grad_f64(X.data_ptr(), Y.data_ptr(), W.data_ptr(), B.data_ptr(), npts, nin, nout,
                                     loss.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(),
                                     err.data_ptr(), _stream())
    _lib.check(rc, "nn_gradients")
    _count()
    return {"loss": DeviceScalar(loss, True, err, NO_SPAN),
            "dw": DeviceSeq(dw, (nin, nout), _lib.PMX_F64),
            "db": DeviceSeq(db, (nout,), _lib.PMX_F64)}

"""The accelerated-expression operator surface on the B200.

Same names, argument meaning and error behaviour as the reference's hot-path
functions in pmx/interp.py, which a host binding can replace by assignment:

    device_call(fn, args, ctx, span)    interp.py:230-237   accelerate entry
    eval_map(f, s, ctx, span)           interp.py:294-304
    eval_map2(f, s1, s2, ctx, span)     interp.py:307-319   (+ length check 151-154)
    eval_reduce(f, acc, s, ctx, span)   interp.py:328-343
    eval_loop(n, f, ctx, span)          interp.py:346-358
    fold(f, acc, s, ctx, span)          interp.py:322-325   (`_fold`, the foldl builtin 461-463)
    flatten(s, ctx, span)               interp.py:161-166
    seq_loop(n, f, state, ctx, span)    recursion used as a device loop (rk4.pmx:38-40)

Function arguments are lambdas of `paper_2211_00621_b200.lam` (the device
form of the reference's Closure/BuiltinPartial).  Every operation runs in the
sm_100a library through the C ABI; nothing is computed on the host.

Evaluation is asynchronous: `eval_map` returns a lazy device sequence that a
following `eval_reduce` fuses into one map->reduce kernel (4 B/element
instead of 12), reductions return device scalars, and device error words are
checked once at the end of `device_call` (or when a value is read).
"""
from __future__ import annotations

import ctypes as C
from typing import Any, Optional

import numpy as np

from . import _lib
from .diagnostics import NO_SPAN, Span, device_error, runtime_error
from .lambdas import Builtin, Lam, as_lam, compile_lambda, CompileError
from .runtime import (
    DeviceArena, DeviceRecordSeq, DeviceScalar, DeviceSeq, DeviceTensor, DeviceValue, Heap,
    _device, _torch_dtype, marshal_in, marshal_out, seq_to_device,
)

import torch


# ------------------------------------------------------------------ context

class Ctx:
    """Evaluation context (pmx/interp.py:56-84).  `workers` has no effect on
    results here (reduce applies `acc` once, debug semantics); device work is
    issued on `stream` of the current CUDA device."""

    def __init__(self, *, mode: str = "accel", heap: Optional[Heap] = None, workers: int = 1,
                 max_rank: int = 3, checks: bool = False, check_determinism: bool = False,
                 stream=None):
        assert mode in ("debug", "accel")
        self.mode = mode
        self.heap = heap if heap is not None else Heap()
        self.workers = max(workers, 1)
        self.max_rank = max_rank
        self.checks = checks
        self.check_determinism = check_determinism
        self.stream = stream
        self.device = False
        self.pending: list = []        # (err tensor, span, what) awaiting a check
        self.launches = 0

    def device_clone(self) -> "Ctx":
        import copy
        d = copy.copy(self)
        d.device = True
        d.pending = []
        d._err_pool = None
        return d

    @property
    def run_parallel(self) -> bool:
        return self.device

    def stream_ptr(self) -> int:
        s = self.stream if self.stream is not None else torch.cuda.current_stream()
        return s.cuda_stream

    def new_err(self, span: Span, what: str = "element"):
        """A fresh device error word (slot of a pooled block, reset to
        PMX_ERR_NONE with an async memset — no kernel launch)."""
        pool = getattr(self, "_err_pool", None)
        if pool is None or self._err_next >= pool.numel():
            pool = torch.empty(256, dtype=torch.int64, device=_device())
            self._err_pool, self._err_next = pool, 0
        err = pool[self._err_next:self._err_next + 1]
        self._err_next += 1
        _lib.check(_lib.load().pmx_err_reset(err.data_ptr(), self.stream_ptr()), "err_reset")
        self.pending.append((err, span, what))
        return err

    def check_errors(self) -> None:
        """One device->host read of all pending error words; raise the first
        failing operation's error (program order)."""
        pend, self.pending = self.pending, []
        if not pend:
            return
        pool = getattr(self, "_err_pool", None)
        if pool is not None and all(e.data_ptr() >= pool.data_ptr() and
                                    e.data_ptr() < pool.data_ptr() + pool.numel() * 8 for e, _, _ in pend):
            words = pool.to("cpu").numpy().view(np.uint64)
            base = pool.data_ptr()
            for err, span, what in pend:
                w = int(words[(err.data_ptr() - base) // 8])
                if w != _lib.PMX_ERR_NONE:
                    raise device_error(w, span, what)
            return
        for err, span, what in pend:
            raise_if_error(err, span, what)


_default_ctx: Optional[Ctx] = None
_ctx_stack: list = []


def default_ctx() -> Ctx:
    """The device context of the innermost active device_call, else a
    process-wide device context (direct use of the operators)."""
    global _default_ctx
    if _ctx_stack:
        return _ctx_stack[-1]
    if _default_ctx is None:
        _default_ctx = Ctx()
        _default_ctx.device = True
    return _default_ctx


def raise_if_error(err, span: Span = NO_SPAN, what: str = "element") -> None:
    if err is None:
        return
    w = int(err.to("cpu").item()) & 0xFFFFFFFFFFFFFFFF
    if w != _lib.PMX_ERR_NONE:
        raise device_error(w, span, what)


_workspaces: dict = {}


def reduce_workspace():
    dev = torch.cuda.current_device()
    ws = _workspaces.get(dev)
    if ws is None:
        n = _lib.load().pmx_reduce_workspace_bytes(0)
        ws = torch.zeros(n, dtype=torch.uint8, device=_device())
        _workspaces[dev] = ws
    return ws


def _ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


# ------------------------------------------------------------ type helpers

def _elem_type(s: DeviceSeq) -> str:
    return "char" if s.elem_tag == "char" else s.elem_tag


def _out_code(in_code: int, out_type: str) -> int:
    if out_type == "float":
        return in_code if in_code in (_lib.PMX_F32, _lib.PMX_F64) else _lib.PMX_F64
    if out_type in ("int", "char"):
        return _lib.PMX_I64
    if out_type == "bool":
        return _lib.PMX_BOOL
    raise runtime_error(f"map result of type {out_type} cannot be stored in a device sequence")


def _as_seq(s, what: str, span: Span) -> DeviceValue:
    if isinstance(s, LazyMap):
        return s
    if isinstance(s, (DeviceSeq, DeviceRecordSeq)):
        return s
    if isinstance(s, (list, np.ndarray)) or isinstance(s, torch.Tensor):
        return seq_to_device(s)
    raise runtime_error(f"{what} expects a sequence", span)


def _compile(f, types, span, state_array=None):
    try:
        return compile_lambda(f, types, state_array=state_array)
    except CompileError as exc:
        raise runtime_error(f"function not supported on the B200 device: {exc}", span) from None


# ------------------------------------------------------------------- map

class LazyMap(DeviceValue):
    """map f s, not yet materialised (fused into a consuming reduce)."""

    def __init__(self, f, src: DeviceSeq, ctx: Ctx, span: Span):
        self.f = f
        self.src = src
        self.ctx = ctx
        self.span = span
        self.compiled = _compile(f, [_elem_type(src), "int"], span)
        self.out_code = _out_code(src.dtype_code, self.compiled.out_type)
        self._value: Optional[DeviceSeq] = None

    def __len__(self) -> int:
        return len(self.src)

    @property
    def shape(self):
        return self.src.shape

    def materialize(self) -> DeviceSeq:
        if self._value is None:
            n = self.src.numel
            y = torch.empty(n, dtype=_torch_dtype(self.out_code), device=_device())
            err = self.ctx.new_err(self.span)
            rc = _lib.load().pmx_map(C.byref(self.compiled.program), self.src.ptr(), self.src.dtype_code,
                                     y.data_ptr(), self.out_code, n, err.data_ptr(), self.ctx.stream_ptr())
            _lib.check(rc, "map")
            self.ctx.launches += 1
            tag = "float" if self.compiled.out_type == "float" else self.compiled.out_type
            self._value = DeviceSeq(y, self.src.shape, self.out_code, offsets=self.src.offsets,
                                    elem_tag=tag)
        return self._value

    # behave like a DeviceSeq when consumed by other operators
    @property
    def data(self):
        return self.materialize().data

    @property
    def dtype_code(self):
        return self.out_code

    @property
    def offsets(self):
        return self.src.offsets

    @property
    def elem_tag(self):
        return self.compiled.out_type

    @property
    def numel(self):
        return self.src.numel

    def ptr(self):
        return self.materialize().ptr()

    def as_pmx_array(self, write: bool = True):
        return self.materialize().as_pmx_array(write)


def _materialize(s):
    return s.materialize() if isinstance(s, LazyMap) else s


def map_tensor(f, t, out_code: int, span: Span = NO_SPAN):
    """Apply a scalar lambda to a flat device tensor, storing `out_code`
    (dtype conversion = identity lambda).  Used by the case-study wrappers
    for their on-device preprocessing (log of probabilities, narrowing)."""
    from .runtime import pmx_code_of_torch
    ctx = default_ctx()
    src = DeviceSeq(t.reshape(-1), (t.numel(),), pmx_code_of_torch(t.dtype))
    comp = _compile(f, [_elem_type(src), "int"], span)
    y = torch.empty(t.numel(), dtype=_torch_dtype(out_code), device=_device())
    err = ctx.new_err(span)
    rc = _lib.load().pmx_map(C.byref(comp.program), src.ptr(), src.dtype_code, y.data_ptr(), out_code,
                             t.numel(), err.data_ptr(), ctx.stream_ptr())
    _lib.check(rc, "map")
    ctx.launches += 1
    return y


def eval_map(f, s, ctx: Optional[Ctx] = None, span: Span = NO_SPAN):
    """y[j] = f(s[j]), element order preserved (pmx/interp.py:294-304)."""
    ctx = ctx or default_ctx()
    s = _materialize(_as_seq(s, "map", span))
    if isinstance(s, DeviceRecordSeq):
        return _map_record(f, s, ctx, span)
    if s.rank != 1 and s.offsets is None:
        raise runtime_error("map over a nested sequence needs a row function; use map_rows", span)
    return LazyMap(f, s, ctx, span)


def _map_record(f, s: DeviceRecordSeq, ctx: Ctx, span: Span):
    # lam p. p.l  (field projection) is a zero-copy column selection
    fl = as_lam(f)
    from .lambdas import Field, Var
    body = fl.body
    if isinstance(body, Field) and isinstance(body.rec, Var) and body.rec.name == fl.params[0]:
        return s.fields[body.label]
    raise runtime_error("map over records supports field projections (lam p. p.l)", span)


def eval_map2(f, s1, s2, ctx: Optional[Ctx] = None, span: Span = NO_SPAN):
    """z[j] = f(s1[j], s2[j]) (pmx/interp.py:307-319); lengths must agree
    (interp.py:151-154)."""
    ctx = ctx or default_ctx()
    s1 = _materialize(_as_seq(s1, "map2", span))
    s2 = _materialize(_as_seq(s2, "map2", span))
    if len(s1) != len(s2):
        raise runtime_error(f"map2 over sequences of different lengths ({len(s1)} and {len(s2)})", span)
    comp = _compile(f, [_elem_type(s1), _elem_type(s2), "int"], span)
    code = _out_code(s1.dtype_code if comp.out_type == "float" and s1.dtype_code in (_lib.PMX_F32, _lib.PMX_F64)
                     else s2.dtype_code, comp.out_type)
    n = s1.numel
    z = torch.empty(n, dtype=_torch_dtype(code), device=_device())
    err = ctx.new_err(span)
    rc = _lib.load().pmx_map2(C.byref(comp.program), s1.ptr(), s1.dtype_code, s2.ptr(), s2.dtype_code,
                              z.data_ptr(), code, n, err.data_ptr(), ctx.stream_ptr())
    _lib.check(rc, "map2")
    ctx.launches += 1
    return DeviceSeq(z, s1.shape, code, offsets=s1.offsets, elem_tag=comp.out_type)


# ---------------------------------------------------------------- reduce

def _acc_code(t: str) -> int:
    if t == "float":
        return _lib.PMX_F64
    if t in ("int", "char", "bool"):
        return _lib.PMX_I64
    raise runtime_error(f"reduce over values of type {t} is not supported on the device")


def _scalar_bits(v, t: str) -> C.c_int64:
    if t == "float":
        return C.c_int64(int(np.array([float(v)], np.float64).view(np.int64)[0]))
    return C.c_int64(int(v))


def eval_reduce(f, acc, s, ctx: Optional[Ctx] = None, span: Span = NO_SPAN, *, keep_map: bool = False):
    """fold f acc s as a deterministic parallel tree (pmx/interp.py:328-343).

    `acc` is applied once (the reference's debug semantics; its parallel
    path folds `acc` into every chunk, identical for the neutral element the
    operator contract requires).  A lazy map operand is fused
    into the reduction; with keep_map=True its output is also materialised in
    the same pass."""
    ctx = ctx or default_ctx()
    s = _as_seq(s, "reduce", span)
    lib = _lib.load()
    fprog = None
    if isinstance(s, LazyMap) and s._value is None:
        src, fprog, elem_t = s.src, s.compiled.program, s.compiled.out_type
        y = torch.empty(src.numel, dtype=_torch_dtype(s.out_code), device=_device()) if keep_map else None
    else:
        src = _materialize(s)
        if isinstance(src, DeviceRecordSeq):
            raise runtime_error("reduce over records is not supported on the device", span)
        elem_t = _elem_type(src)
        y = None
    if isinstance(acc, DeviceScalar):
        acc = acc.get()
    acc_t = "float" if isinstance(acc, float) else ("bool" if isinstance(acc, bool) else "int")
    if acc_t != ("int" if elem_t == "char" else elem_t):
        raise runtime_error(f"reduce: accumulator of type {acc_t} over elements of type {elem_t}", span)
    op = _compile(f, [acc_t, acc_t], span)
    code = _acc_code(acc_t)
    out = torch.empty(1, dtype=torch.float64 if code == _lib.PMX_F64 else torch.int64, device=_device())
    init = _scalar_bits(acc, acc_t)
    ws = reduce_workspace()
    err = ctx.new_err(span)
    out_code = s.out_code if (y is not None) else src.dtype_code
    rc = lib.pmx_map_reduce(C.byref(fprog) if fprog is not None else None, C.byref(op.program),
                            src.ptr(), src.dtype_code, src.numel, C.byref(init), code, out.data_ptr(),
                            _ptr(y), out_code, ws.data_ptr(), ws.numel(), err.data_ptr(), ctx.stream_ptr())
    _lib.check(rc, "reduce")
    ctx.launches += 1
    if y is not None:
        s._value = DeviceSeq(y, src.shape, s.out_code, offsets=src.offsets, elem_tag=elem_t)
    res = DeviceScalar(out, acc_t == "float", err, span)
    if ctx.check_determinism:
        _check_determinism(op, acc, acc_t, code, _materialize(s), res, ctx, span)
    return res


def _check_determinism(op, acc, acc_t, code, src, res, ctx, span):
    """--check-determinism (pmx/interp.py:337-342, pmx/cli.py:41-42): re-fold
    the sequence in element order on the device (one thread, pmx_fold without
    a workspace) and warn, with the reference's message, when the tree
    result differs beyond rel 1e-6 (interp.py:361-372)."""
    import math
    import sys
    ref = torch.empty(1, dtype=torch.float64 if code == _lib.PMX_F64 else torch.int64, device=_device())
    err = ctx.new_err(span)
    init = _scalar_bits(acc, acc_t)
    rc = _lib.load().pmx_fold(C.byref(op.program), src.ptr(), src.dtype_code, src.numel, C.byref(init), code,
                              ref.data_ptr(), None, 0, err.data_ptr(), ctx.stream_ptr())
    _lib.check(rc, "check_determinism fold")
    ctx.launches += 1
    total = res.get()
    reference = DeviceScalar(ref, acc_t == "float", err, span).get()
    if acc_t == "float":
        close = math.isclose(total, reference, rel_tol=1e-6, abs_tol=1e-6)
    else:
        close = total == reference
    if not close:
        print("warning: reduce result depends on the evaluation order "
              f"(blocked {total!r} vs sequential {reference!r}); the "
              "operator may not be associative", file=sys.stderr)


class PreparedMapReduce:
    """`reduce op acc (map f s)` over a device sequence, lowered once and
    launched many times (one C-ABI call per launch, no host work): the
    plugin-level entry used by the benchmark's device-resident loop and by
    the sharded reduce.  f=None is a plain reduce; materialize=tensor also
    writes map f s; reduce=False makes it a plain map."""

    def __init__(self, f, op, acc, s: DeviceSeq, ctx: Optional[Ctx] = None, materialize=None,
                 reduce: bool = True, span: Span = NO_SPAN):
        self.ctx = ctx or default_ctx()
        self.lib = _lib.load()
        self.s = s
        et = _elem_type(s)
        self.f = _compile(f, [et, "int"], span) if f is not None else None
        out_t = self.f.out_type if self.f is not None else et
        acc_t = "float" if isinstance(acc, float) else "int"
        self.op = _compile(op, [acc_t, acc_t], span)
        self.code = _acc_code(acc_t)
        self.init = _scalar_bits(acc, acc_t)
        self.y = materialize
        self.reduce = reduce
        self.out = torch.empty(1, dtype=torch.float64 if self.code == _lib.PMX_F64 else torch.int64,
                               device=_device())
        self.err = self.ctx.new_err(span)
        self.ws = reduce_workspace()
        self.ycode = _out_code(s.dtype_code, out_t)
        self._fold_op = None

    def launch(self):
        if not self.reduce:
            rc = self.lib.pmx_map(C.byref(self.f.program), self.s.ptr(), self.s.dtype_code, self.y.data_ptr(),
                                  self.ycode, self.s.numel, self.err.data_ptr(), self.ctx.stream_ptr())
            _lib.check(rc, "map")
            self.ctx.launches += 1
            return self.y
        rc = self.lib.pmx_map_reduce(C.byref(self.f.program) if self.f is not None else None,
                                     C.byref(self.op.program), self.s.ptr(), self.s.dtype_code, self.s.numel,
                                     C.byref(self.init), self.code, self.out.data_ptr(), _ptr(self.y), self.ycode,
                                     self.ws.data_ptr(), self.ws.numel(), self.err.data_ptr(),
                                     self.ctx.stream_ptr())
        _lib.check(rc, "map_reduce")
        self.ctx.launches += 1
        return self.out

    def launch_peers(self, group):
        """This rank's shard reduced and combined with every other rank's
        partial over NVLink peer memory in the same kernel (pmx_map_reduce_peers):
        returns the global result (identical on every rank)."""
        assert self.reduce and self.y is None
        g = group.next()
        rc = self.lib.pmx_map_reduce_peers(C.byref(self.f.program) if self.f is not None else None,
                                           C.byref(self.op.program), self.s.ptr(), self.s.dtype_code,
                                           self.s.numel, C.byref(self.init), self.code, self.out.data_ptr(),
                                           self.ws.data_ptr(), self.ws.numel(), C.byref(g),
                                           self.err.data_ptr(), self.ctx.stream_ptr())
        _lib.check(rc, "map_reduce_peers")
        self.ctx.launches += 1
        return self.out

    def has_peer_kernel(self) -> bool:
        kf = 1 if self.f is None else self.lib.pmx_program_kind(C.byref(self.f.program), 0)
        return kf in (1, 2, 3) and self.lib.pmx_program_kind(C.byref(self.op.program), 1) >= 10

    def fold_partials(self, partials):
        """Left fold of per-GPU partials in rank order (interp.py:334-336),
        on the device; `init` is not re-applied."""
        if self._fold_op is None:
            self._fold_op = self.op
            self._fold_out = torch.empty_like(self.out)
        kind = self.lib.pmx_program_kind(C.byref(self.op.program), 1)
        if kind in (10, 20):
            # sum: total = p0 + p1 + ... = fold from the neutral 0 (no host read)
            rest, init = partials, C.c_int64(0)
        else:
            rest = partials[1:]
            init = _scalar_bits(partials[:1].to("cpu").item(), "float" if self.code == _lib.PMX_F64 else "int")
        rc = self.lib.pmx_fold(C.byref(self.op.program), rest.data_ptr(), self.code, rest.numel(), C.byref(init),
                               self.code, self._fold_out.data_ptr(), None, 0, self.err.data_ptr(),
                               self.ctx.stream_ptr())
        _lib.check(rc, "fold_partials")
        self.ctx.launches += 1
        return self._fold_out


def fold(f, acc, s, ctx: Optional[Ctx] = None, span: Span = NO_SPAN):
    """foldl f acc s: sequential left fold on the device (pmx/interp.py:322-325,
    461-463); exactly-associative operators use the parallel tree."""
    ctx = ctx or default_ctx()
    src = _materialize(_as_seq(s, "foldl", span))
    if isinstance(acc, DeviceScalar):
        acc = acc.get()
    acc_t = "float" if isinstance(acc, float) else ("bool" if isinstance(acc, bool) else "int")
    op = _compile(f, [acc_t, _elem_type(src)], span)
    if op.out_type not in (acc_t, "never"):
        raise runtime_error(f"foldl: operator returns {op.out_type}, accumulator is {acc_t}", span)
    code = _acc_code(acc_t)
    out = torch.empty(1, dtype=torch.float64 if code == _lib.PMX_F64 else torch.int64, device=_device())
    init = _scalar_bits(acc, acc_t)
    ws = reduce_workspace()
    err = ctx.new_err(span)
    rc = _lib.load().pmx_fold(C.byref(op.program), src.ptr(), src.dtype_code, src.numel, C.byref(init),
                              code, out.data_ptr(), ws.data_ptr(), ws.numel(), err.data_ptr(),
                              ctx.stream_ptr())
    _lib.check(rc, "foldl")
    ctx.launches += 1
    return DeviceScalar(out, acc_t == "float", err, span)


# ------------------------------------------------------------ row folds

def map_rows_fold(g, op, acc, s, ctx: Optional[Ctx] = None, span: Span = NO_SPAN) -> DeviceSeq:
    """map (lam row. reduce op acc (map g row)) s over a sequence of sequences
    (g=None: `foldl op acc row` / `reduce op acc row`).  Inside a map body the
    reference runs the inner skeletons sequentially (pmx/interp.py:82-84), so
    each row is a left fold from `acc` in element order (interp.py:322-325)."""
    ctx = ctx or default_ctx()
    s = _materialize(_as_seq(s, "map", span))
    if isinstance(s, DeviceRecordSeq):
        raise runtime_error("map over records supports field projections (lam p. p.l)", span)
    if s.offsets is not None:
        nrows, offs = len(s), s.offsets
    elif s.rank == 2:
        nrows, m = s.shape
        offs = torch.empty(nrows + 1, dtype=torch.int64, device=_device())
        _lib.check(_lib.load().pmx_row_offsets(offs.data_ptr(), nrows, m, ctx.stream_ptr()), "row offsets")
        ctx.launches += 1
    else:
        raise runtime_error("a row function needs a sequence of sequences", span)
    if isinstance(acc, DeviceScalar):
        acc = acc.get()
    acc_t = "float" if isinstance(acc, float) else ("bool" if isinstance(acc, bool) else "int")
    et = _elem_type(s)
    gc = _compile(g, [et, "int"], span) if g is not None else None
    vt = gc.out_type if gc is not None else et
    opc = _compile(op, [acc_t, "int" if vt == "char" else vt], span)
    if opc.out_type not in (acc_t, "never"):
        raise runtime_error(f"fold: operator returns {opc.out_type}, accumulator is {acc_t}", span)
    code = _lib.PMX_F64 if acc_t == "float" else (_lib.PMX_BOOL if acc_t == "bool" else _lib.PMX_I64)
    out = torch.empty(nrows, dtype=_torch_dtype(code), device=_device())
    init = _scalar_bits(acc, acc_t)
    err = ctx.new_err(span)
    rc = _lib.load().pmx_map_rows_fold(C.byref(gc.program) if gc is not None else None, C.byref(opc.program),
                                       s.ptr(), s.dtype_code, offs.data_ptr(), nrows, C.byref(init),
                                       out.data_ptr(), code, err.data_ptr(), ctx.stream_ptr())
    _lib.check(rc, "map_rows_fold")
    ctx.launches += 1
    return DeviceSeq(out, (nrows,), code, elem_tag=acc_t)


# ------------------------------------------------------------------ loop

def eval_loop(n: int, f, ctx: Optional[Ctx] = None, span: Span = NO_SPAN) -> dict:
    """f(i) for i in [0, n) with effects through tensorSet on marshalled tensor
    views (pmx/interp.py:346-358); n <= 0 runs nothing.  Returns unit ({})."""
    ctx = ctx or default_ctx()
    if isinstance(n, DeviceScalar):
        n = n.get()
    if n <= 0:
        return {}
    prog = _compile(f, ["int"], span)
    err = ctx.new_err(span, "iteration")
    rc = _lib.load().pmx_loop(C.byref(prog.program), int(n), err.data_ptr(), ctx.stream_ptr())
    _lib.check(rc, "loop")
    ctx.launches += 1
    return {}


def seq_loop(n: int, f, state, ctx: Optional[Ctx] = None, span: Span = NO_SPAN) -> DeviceSeq:
    """seqLoop: n in-order iterations of a parallel step over a Float state,
    one persistent kernel (grid barrier between steps).

        state'[j] = f(state[j], j, t)   with `prev` (get prev i) the state of step t

    `f` is lam(x, j, t, body) and may read the whole previous state through
    the captured placeholder `PREV` (see lam.get)."""
    ctx = ctx or default_ctx()
    s = _materialize(_as_seq(state, "seqLoop", span))
    if s.dtype_code == _lib.PMX_F64:
        init = s.data.reshape(-1)                                      # read by step 0, left unchanged
    else:
        from .lambdas import lam
        init = map_tensor(lam("x", "x"), s.data, _lib.PMX_F64, span)  # Float state in fp64 (one pmx_map)
    a = torch.empty(init.numel(), dtype=torch.float64, device=init.device)
    b = torch.empty(init.numel() + 8, dtype=torch.float64, device=init.device)   # + grid-barrier word
    prog = _compile(f, ["float", "int", "int"], span, state_array=PREV)
    err = ctx.new_err(span)
    rc = _lib.load().pmx_seq_loop_from(C.byref(prog.program), init.data_ptr(), a.data_ptr(), b.data_ptr(),
                                       a.numel(), int(n), err.data_ptr(), ctx.stream_ptr())
    _lib.check(rc, "seq_loop")
    ctx.launches += 1
    return DeviceSeq(a, s.shape, _lib.PMX_F64)


class _PrevState:
    """Placeholder for the previous seqLoop state inside a step lambda."""
    dtype_code = _lib.PMX_F64

    def as_pmx_array(self, write: bool = True):
        a = _lib.Array()
        a.rank = 1
        a.dtype = _lib.PMX_F64
        a.shape[0] = 1 << 62
        return a


PREV = _PrevState()


# --------------------------------------------------------------- flatten

def flatten(s, ctx: Optional[Ctx] = None, span: Span = NO_SPAN) -> DeviceSeq:
    """flatten [[a]] -> [a] (pmx/interp.py:161-166).  The device layout is
    already flat, so this is a metadata change (no copy)."""
    s = _materialize(_as_seq(s, "flatten", span))
    if s.offsets is not None:
        return DeviceSeq(s.data, (s.data.numel(),), s.dtype_code, elem_tag=s.elem_tag)
    if s.rank < 2:
        raise runtime_error("flatten expects a sequence of sequences", span)
    return DeviceSeq(s.data, (s.shape[0] * s.shape[1],) + s.shape[2:], s.dtype_code, elem_tag=s.elem_tag)


def length(s) -> int:
    return len(s)


# ------------------------------------------------------------ accelerate

def device_call(fn, args: list, ctx: Optional[Ctx] = None, span: Span = NO_SPAN, verdict=None):
    """The accelerate entry point (pmx/interp.py:230-237): marshal the
    arguments to the device (Alg. 2), evaluate the body in a device context,
    check device errors, copy written roots back and return host values.

    `fn` is a Python callable over device values built from this module's
    operators (the lifted accelerate binding, pmx/transform.py:198-317).
    `verdict` is the binding's backend classification ("futhark" / "cuda");
    it selects which assumption check `ctx.checks` runs (pmx/interp.py:223-227),
    both when None."""
    ctx = ctx or Ctx()
    if ctx.checks:
        from .checks import check_arg
        for a in args:
            check_arg(a, ctx.max_rank, verdict)
    dev_args, arena = marshal_in(list(args), ctx.heap)
    dctx = ctx.device_clone()
    _ctx_stack.append(dctx)
    try:
        result = fn(*dev_args, ctx=dctx) if _takes_ctx(fn) else fn(*dev_args)
        result = _force(result)
        dctx.check_errors()
    finally:
        _ctx_stack.pop()
    out = marshal_out(arena, ctx.heap, result)
    ctx.launches += dctx.launches
    ctx.last_arena = arena
    return out


def _force(v):
    """Materialise lazy maps in a result (they must exist before marshal_out)."""
    if isinstance(v, LazyMap):
        return v.materialize()
    if isinstance(v, list):
        return [_force(x) for x in v]
    if isinstance(v, tuple):
        return tuple(_force(x) for x in v)
    if isinstance(v, dict):
        return {k: _force(x) for k, x in v.items()}
    return v


def _takes_ctx(fn) -> bool:
    code = getattr(fn, "__code__", None)
    if code is not None and not hasattr(fn, "__wrapped__"):   # plain function / lambda: no inspect
        return "ctx" in code.co_varnames[:code.co_argcount + code.co_kwonlyargcount]
    import inspect
    try:
        return "ctx" in inspect.signature(fn).parameters
    except (TypeError, ValueError):
        return False


def accelerate(fn, *args, ctx: Optional[Ctx] = None, span: Span = NO_SPAN, verdict=None):
    """`accelerate (fn args...)` — run fn on the B200 with its arguments marshalled."""
    return device_call(fn, list(args), ctx, span, verdict)

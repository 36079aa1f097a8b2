"""Whole-program drop-in: run the reference interpreter's accelerated
constructs on the B200.

The reference's parallel skeletons are module globals of `pmx.interp`, looked
up by name at every call (pmx/interp.py:146, 155, 160, 170).  `install(interp)`
replaces them:

    eval_map    (interp.py:294-304)   eval_map2 (307-319)
    eval_reduce (interp.py:328-343)   eval_loop (346-358)

When the construct runs in device context and is not nested (`ctx.run_parallel`,
interp.py:82-84), its function argument — a reference `Closure` or
`BuiltinPartial` (pmx/runtime.py:78-93), i.e. an AST with an environment — is
translated to this package's lambda IR (`to_lam`), the sequence is marshalled
to the device, the construct runs in libpmxb200.so, and the result comes back
as reference values.  Everything else (host code, nested constructs inside a
worker, debug mode) keeps the reference's own implementation, exactly as the
reference runs it.  A function the device cannot execute raises the
reference's `Diagnostics` — there is no silent CPU fallback.

Only this module imports `pmx`, and only when the caller passes it in (the
reference is not shipped with this repository).
"""
from __future__ import annotations

from typing import Any, Callable, Optional

from . import lambdas as L
from .lambdas import CompileError


class Unsupported(Exception):
    pass


# ============================================================ translation

def to_lam(f, n_params: int, syn, rt, host_array: Callable) -> L.Lam:
    """Translate a reference function value of arity n_params to a Lam.

    `syn` / `rt` are the reference modules pmx.syntax / pmx.runtime;
    `host_array(value)` turns a captured host sequence / tensor into the object
    stored in Get/TGet/TSet nodes (a device array for the B200, the host value
    for the CPU checker)."""
    tr = _Translator(syn, rt, host_array)
    params = [f"_a{i}" for i in range(n_params)]
    body = tr.apply_value(f, [L.Var(p) for p in params], depth=0)
    return L.Lam(params, body)


def to_row_fold(f, syn, rt, host_array: Callable):
    """A row function of `map` over a sequence of sequences:
        lam row. foldl op acc row  |  lam row. reduce op acc row
      | lam row. reduce op acc (map g row)
    -> (g Lam or None, op Lam, acc).  Anything else is Unsupported."""
    S = syn
    if not isinstance(f, rt.Closure):
        raise Unsupported("row function")
    tr = _Translator(syn, rt, host_array)
    scope = {"__env__": f.env}
    row = f.param

    def is_row(x):
        return isinstance(x, S.Var) and x.name == row

    e = f.body
    g_e = None
    if isinstance(e, S.ReduceE):
        op_e, acc_e = e.fn, e.acc
        if isinstance(e.seq, S.MapE) and is_row(e.seq.seq):
            g_e = e.seq.fn
        elif not is_row(e.seq):
            raise Unsupported("row function: reduce over something other than the row")
    else:
        head, args = e, []
        while isinstance(head, S.App):
            args.append(head.arg)
            head = head.fn
        args.reverse()
        if not (isinstance(head, S.ConstE) and isinstance(head.const, S.CBuiltin) and head.const.name == "foldl"
                and len(args) == 3 and is_row(args[2])):
            raise Unsupported("row function (expected foldl / reduce over the row)")
        op_e, acc_e = args[0], args[1]

    def fn_lam(fe, n):
        params = [f"_r{i}" for i in range(n)]
        body = tr.apply_value(tr.expr(fe, scope, 0), [L.Var(p) for p in params], depth=1)
        return L.Lam(params, tr.as_expr(body))

    op_lam = fn_lam(op_e, 2)
    g_lam = fn_lam(g_e, 1) if g_e is not None else None
    acc = tr.expr(acc_e, scope, 0)
    if not isinstance(acc, L.Const):
        raise Unsupported("row function: accumulator must be a constant or captured scalar")
    v = acc.value
    return g_lam, op_lam, (bool(v) if acc.ty == "bool" else v)


class _Fn:
    """A function value during translation: Closure, builtin partial, or a
    lambda bound in the body being translated."""

    def __init__(self, kind, **kw):
        self.kind = kind
        self.__dict__.update(kw)


class _Translator:
    MAX_INLINE = 16

    def __init__(self, syn, rt, host_array):
        self.S = syn
        self.R = rt
        self.host_array = host_array
        self.names: dict = {}
        self.counter = 0

    def fresh(self, base: str) -> str:
        self.counter += 1
        return f"{base}_{self.counter}"

    # -- values captured from the reference environment
    def value(self, v):
        if isinstance(v, bool):
            return L.Const(bool(v), "bool")
        if isinstance(v, int):
            return L.Const(int(v), "int")
        if isinstance(v, float):
            return L.Const(float(v), "float")
        if isinstance(v, str) and len(v) == 1:
            return L.Const(ord(v), "char")
        if isinstance(v, (self.R.Closure, self.R.BuiltinPartial)):
            return _Fn("value", v=v)
        if isinstance(v, (list, self.R.TensorView)):
            return _Captured(v)
        raise Unsupported(f"captured value of type {type(v).__name__}")

    # -- applying a function value to IR arguments
    def apply_value(self, fv, args: list, depth: int):
        R = self.R
        if depth > self.MAX_INLINE:
            raise Unsupported("recursion or deep function nesting")
        if isinstance(fv, _Fn):
            if fv.kind == "value":
                return self.apply_value(fv.v, args, depth)
            if fv.kind == "lam":                      # lambda bound in the body
                return self.apply_lam(fv.param, fv.body, fv.scope, args, depth)
            raise Unsupported("function value")
        if isinstance(fv, R.BuiltinPartial):
            pre = [self.value(a) for a in fv.args]
            return self.builtin(fv.name, pre + args)
        if isinstance(fv, R.Closure):
            return self.apply_closure(fv, args, depth)
        raise Unsupported(f"application of {type(fv).__name__}")

    def apply_closure(self, clo, args, depth):
        rec = self.linear_recursion(clo, args, depth)
        if rec is None:
            rec = self.kterm_recursion(clo, args, depth)
        if rec is not None:
            return rec
        scope = {"__env__": clo.env}
        return self.apply_lam(clo.param, clo.body, scope, args, depth)

    # -- linear recursion as a device loop
    def _peel(self, clo):
        """(parameter names, innermost body) of a curried closure."""
        S = self.S
        params, body = [clo.param], clo.body
        while isinstance(body, S.Lam):
            params.append(body.param)
            body = body.body
        return params, body

    def linear_recursion(self, clo, args, depth):
        """f p.. = match pj with c then BASE else E[f p.. (subi pj 1)] (the
        recursive call once, outside any lambda, other arguments passed
        through unchanged) -> Iterate: acc = BASE[pj := c]; for m in c+1..pj:
        acc = E[pj := m, call := acc].  None if f is not of this form."""
        S, R = self.S, self.R
        params, body = self._peel(clo)
        if len(params) != len(args) or not isinstance(body, S.Match):
            return None
        m = body
        if not (isinstance(m.scrut, S.Var) and m.scrut.name in params and isinstance(m.pat, S.PConst)
                and isinstance(m.pat.const, S.CInt)):
            return None
        pj, c = m.scrut.name, int(m.pat.const.value)
        calls = []

        def resolves_to_self(name):
            if name in params:
                return None
            try:
                v = clo.env.lookup(name)
            except AssertionError:
                return None
            if not isinstance(v, R.Closure):
                return None
            dps, dbody = self._peel(v)
            return dps if dbody is body else None

        def walk(e):
            if isinstance(e, S.Lam):
                return not self._mentions_self(e, resolves_to_self)
            if isinstance(e, S.App):
                head, a = e, []
                while isinstance(head, S.App):
                    a.append(head.arg)
                    head = head.fn
                a.reverse()
                if isinstance(head, S.Var):
                    dps = resolves_to_self(head.name)
                    if dps is not None:
                        calls.append((e, dps, a))
                        return True
                return walk(head) and all(walk(x) for x in a)
            if isinstance(e, S.Let):
                return walk(e.value) and walk(e.body)
            if isinstance(e, S.Match):
                return walk(e.scrut) and walk(e.thn) and walk(e.els)
            if isinstance(e, S.Var):
                return resolves_to_self(e.name) is None
            return True

        if not walk(m.els) or len(calls) != 1 or self._mentions_self(m.thn, resolves_to_self):
            return None
        call, dps, cargs = calls[0]
        if len(cargs) != len(dps):
            return None
        for q, a in zip(dps, cargs):
            if q == pj:                               # subi pj 1
                ok = (isinstance(a, S.App) and isinstance(a.fn, S.App) and isinstance(a.fn.fn, S.ConstE)
                      and isinstance(a.fn.fn.const, S.CBuiltin) and a.fn.fn.const.name == "subi"
                      and isinstance(a.fn.arg, S.Var) and a.fn.arg.name == pj
                      and isinstance(a.arg, S.ConstE) and isinstance(a.arg.const, S.CInt)
                      and int(a.arg.const.value) == 1)
            else:                                     # passed through unchanged
                ok = isinstance(a, S.Var) and a.name == q
            if not ok:
                return None
        # bind the actual arguments (scalars once), then build the loop
        scope = {"__env__": clo.env}
        binds = []
        for prm, a in zip(params, args):
            if isinstance(a, (_Fn, _Captured, L.Var)):
                scope[prm] = a
            else:
                nm = self.fresh(prm.text)
                scope[prm] = L.Var(nm)
                binds.append((nm, a))
        hi = self.as_expr(scope[pj])
        mvar, accvar = self.fresh("rec_m"), self.fresh("rec_acc")
        base_scope = dict(scope)
        base_scope[pj] = L.Const(c, "int")
        init = self.as_expr(self.expr(m.thn, base_scope, depth + 1))
        step_scope = dict(scope)
        step_scope[pj] = L.Var(mvar)
        prev = getattr(self, "_rec_hole", None)
        self._rec_hole = {id(call): accvar}
        try:
            step = self.as_expr(self.expr(m.els, step_scope, depth + 1))
        finally:
            self._rec_hole = prev
        out = L.Iterate(mvar, L.Const(c + 1, "int"), hi, accvar, init, step)
        for n, a in reversed(binds):
            out = L.LetE(n, a, out)
        return out

    def kterm_recursion(self, clo, args, depth):
        """f p.. = match pj with c0 then B0 else match pj with c1 then B1 ...
        else E[f p.. (subi pj d1), f p.. (subi pj d2), ..] with the base cases
        c .. c+k-1 consecutive and 1 <= d <= k, d = 1 among them (so the
        reference's top-down evaluation visits every level, e.g. fib) ->
        Iterate from the base cases up with k accumulators (f(m-1) .. f(m-k)).
        The calls must be strict: not under a match or a lambda of E, so the
        bottom-up loop evaluates exactly the levels the reference does (once
        each instead of exponentially often).  None if f is not of this form."""
        S, R = self.S, self.R
        params, body = self._peel(clo)
        if len(params) != len(args) or not isinstance(body, S.Match):
            return None
        pj = None
        bases = {}
        e = body
        while isinstance(e, S.Match):
            if not (isinstance(e.scrut, S.Var) and e.scrut.name in params and isinstance(e.pat, S.PConst)
                    and isinstance(e.pat.const, S.CInt)):
                return None
            if pj is None:
                pj = e.scrut.name
            elif e.scrut.name != pj:
                return None
            cv = int(e.pat.const.value)
            if cv in bases:
                return None
            bases[cv] = e.thn
            e = e.els
        E = e
        k = len(bases)
        c = min(bases)
        if k < 2 or sorted(bases) != list(range(c, c + k)):
            return None

        def resolves_to_self(name):
            if name in params:
                return None
            try:
                v = clo.env.lookup(name)
            except AssertionError:
                return None
            if not isinstance(v, R.Closure):
                return None
            dps, dbody = self._peel(v)
            return dps if dbody is body else None

        if any(self._mentions_self(b, resolves_to_self) for b in bases.values()):
            return None
        calls = []

        def walk(x):                                  # strict positions only
            if isinstance(x, (S.Lam, S.Match)):
                return not self._mentions_self(x, resolves_to_self)
            if isinstance(x, S.App):
                head, a = x, []
                while isinstance(head, S.App):
                    a.append(head.arg)
                    head = head.fn
                a.reverse()
                if isinstance(head, S.Var):
                    dps = resolves_to_self(head.name)
                    if dps is not None:
                        calls.append((x, dps, a))
                        return all(not self._mentions_self(y, resolves_to_self) for y in a)
                return walk(head) and all(walk(y) for y in a)
            if isinstance(x, S.Let):
                return walk(x.value) and walk(x.body)
            if isinstance(x, S.Var):
                return resolves_to_self(x.name) is None
            return True

        if not walk(E) or not calls:
            return None
        offsets = {}
        for call, dps, cargs in calls:
            if len(cargs) != len(dps):
                return None
            d = None
            for q, a in zip(dps, cargs):
                if q == pj:                           # subi pj d
                    if not (isinstance(a, S.App) and isinstance(a.fn, S.App) and isinstance(a.fn.fn, S.ConstE)
                            and isinstance(a.fn.fn.const, S.CBuiltin) and a.fn.fn.const.name == "subi"
                            and isinstance(a.fn.arg, S.Var) and a.fn.arg.name == pj
                            and isinstance(a.arg, S.ConstE) and isinstance(a.arg.const, S.CInt)):
                        return None
                    d = int(a.arg.const.value)
                elif not (isinstance(a, S.Var) and a.name == q):
                    return None
            if d is None or not 1 <= d <= k:
                return None
            offsets[id(call)] = d
        if 1 not in offsets.values():
            return None
        scope = {"__env__": clo.env}
        binds = []
        for prm, a in zip(params, args):
            if isinstance(a, (_Fn, _Captured, L.Var)):
                scope[prm] = a
            else:
                nm = self.fresh(prm.text)
                scope[prm] = L.Var(nm)
                binds.append((nm, a))
        hi = self.as_expr(scope[pj])
        mvar = self.fresh("rec_m")
        accs = [self.fresh("rec_acc") for _ in range(k)]        # accs[j] = f(m - 1 - j)
        inits = []
        for j in range(k):
            bs = dict(scope)
            bs[pj] = L.Const(c + k - 1 - j, "int")
            inits.append(self.as_expr(self.expr(bases[c + k - 1 - j], bs, depth + 1)))
        step_scope = dict(scope)
        step_scope[pj] = L.Var(mvar)
        prev = getattr(self, "_rec_hole", None)
        self._rec_hole = {cid: accs[d - 1] for cid, d in offsets.items()}
        try:
            step = self.as_expr(self.expr(E, step_scope, depth + 1))
        finally:
            self._rec_hole = prev
        out = L.Iterate(mvar, L.Const(c + k, "int"), hi, accs[0], inits[0], step,
                        tuple(zip(accs[1:], inits[1:])))
        for n, a in reversed(binds):
            out = L.LetE(n, a, out)
        return out

    def _mentions_self(self, e, resolves_to_self):
        S = self.S
        if isinstance(e, S.Var):
            return resolves_to_self(e.name) is not None
        for child in getattr(e, "__dict__", {}).values():
            if isinstance(child, S.Expr) and self._mentions_self(child, resolves_to_self):
                return True
            if isinstance(child, list):
                for x in child:
                    if isinstance(x, S.Expr) and self._mentions_self(x, resolves_to_self):
                        return True
        return False

    def apply_lam(self, param, body, scope, args, depth):
        if not args:
            raise Unsupported("partial application returned as a value")
        S = self.S
        inner = dict(scope)
        binds = []

        def bind(p, a):
            if isinstance(a, (_Fn, _Captured, L.Var)):   # function / sequence / variable: substitute
                inner[p] = a
            else:                                     # scalar argument: let-bind (evaluated once)
                nm = self.fresh(p.text)
                inner[p] = L.Var(nm)
                binds.append((nm, a))

        bind(param, args[0])
        rest = args[1:]
        e = body
        while rest and isinstance(e, S.Lam):          # consume further curried parameters
            bind(e.param, rest[0])
            rest = rest[1:]
            e = e.body
        out = self.expr(e, inner, depth + 1)
        if rest:
            out = self.apply_value(out, rest, depth + 1)
        if binds and isinstance(out, (_Fn, _Captured)):
            raise Unsupported("function value returned from a device function")
        for n, a in reversed(binds):
            out = L.LetE(n, a, out)
        return out

    def as_expr(self, x):
        if isinstance(x, (_Fn, _Captured)):
            raise Unsupported("function or sequence used as a scalar")
        return x

    # -- AST -> IR
    def lookup(self, name, scope):
        if name in scope:
            return scope[name]
        env = scope.get("__env__")
        if env is None:
            raise Unsupported(f"unbound {name}")
        try:
            v = env.lookup(name)
        except AssertionError:
            raise Unsupported(f"unbound {name}") from None
        return self.value(v)

    def expr(self, e, scope, depth):
        S = self.S
        hole = getattr(self, "_rec_hole", None)
        if hole is not None and id(e) in hole:        # a recursive call: one of the loop's accumulators
            return L.Var(hole[id(e)])
        if isinstance(e, S.Var):
            return self.lookup(e.name, scope)
        if isinstance(e, S.ConstE):
            c = e.const
            if isinstance(c, S.CBuiltin):
                return _Fn("value", v=self.R.BuiltinPartial(c.name, ()))
            if isinstance(c, S.CChar):
                return L.Const(ord(c.value), "char")
            if isinstance(c, S.CBool):
                return L.Const(bool(c.value), "bool")
            if isinstance(c, S.CInt):
                return L.Const(int(c.value), "int")
            return L.Const(float(c.value), "float")
        if isinstance(e, S.Lam):
            return _Fn("lam", param=e.param, body=e.body, scope=scope)
        if isinstance(e, S.App):
            head, args = e, []
            while isinstance(head, S.App):
                args.append(head.arg)
                head = head.fn
            args.reverse()
            if isinstance(head, S.ConstE) and isinstance(head.const, S.CBuiltin):
                name = head.const.name
                if name in ("tensorGet", "tensorSet"):
                    return self.tensor_op(name, args, scope, depth)
                return self.builtin(name, [self.expr(a, scope, depth) for a in args])
            fv = self.expr(head, scope, depth)
            return self.apply_value(fv, [self.expr(a, scope, depth) for a in args], depth + 1)
        if isinstance(e, S.Let):
            v = self.expr(e.value, scope, depth)
            inner = dict(scope)
            if isinstance(v, (_Fn, _Captured)):
                inner[e.name] = v
                return self.expr(e.body, inner, depth)
            nm = self.fresh(e.name.text)
            inner[e.name] = L.Var(nm)
            return L.LetE(nm, v, self.as_expr(self.expr(e.body, inner, depth)))
        if isinstance(e, S.Match):
            return self.match(e, scope, depth)
        if isinstance(e, S.Never):
            return L.Never()
        raise Unsupported(f"{type(e).__name__} in a device function")

    def match(self, e, scope, depth):
        S = self.S
        pat = e.pat
        if isinstance(pat, S.PVar):
            v = self.expr(e.scrut, scope, depth)
            inner = dict(scope)
            if isinstance(v, (_Fn, _Captured)):
                inner[pat.name] = v
                return self.expr(e.thn, inner, depth)
            nm = self.fresh(pat.name.text)
            inner[pat.name] = L.Var(nm)
            return L.LetE(nm, v, self.as_expr(self.expr(e.thn, inner, depth)))
        if isinstance(pat, S.PConst):
            v = self.as_expr(self.expr(e.scrut, scope, depth))
            c = self.expr(S.ConstE(pat.const), scope, depth)
            return L.If(L.Prim("eq", [v, c]), self.as_expr(self.expr(e.thn, scope, depth)),
                        self.as_expr(self.expr(e.els, scope, depth)))
        if isinstance(pat, S.PRecord):
            # projection sugar (pmx/parser.py:400-406): match r with {l = x} then x else never
            if len(pat.fields) == 1 and isinstance(pat.fields[0][1], S.PVar) and isinstance(e.els, S.Never):
                label, sub = pat.fields[0]
                rec = self.expr(e.scrut, scope, depth)
                if isinstance(e.thn, S.Var) and e.thn.name == sub.name:
                    return L.Field(self.as_expr(rec), label)
                inner = dict(scope)
                nm = self.fresh(sub.name.text)
                inner[sub.name] = L.Var(nm)
                return L.LetE(nm, L.Field(self.as_expr(rec), label), self.as_expr(self.expr(e.thn, inner, depth)))
            raise Unsupported("record pattern")
        raise Unsupported("pattern")

    def builtin(self, name, args):
        if name in L.BUILTINS:
            if len(args) < L.BUILTINS[name].arity:
                # partial builtin as a value
                return _Fn("value", v=self.R.BuiltinPartial(name, tuple()))
            return L.Prim(name, [self.as_expr(a) for a in args])
        if name == "get":
            s, i = args
            if not isinstance(s, _Captured):
                raise Unsupported("get on a non-captured sequence")
            return L.Get(self.host_array(s.v), self.as_expr(i))
        if name == "length":
            (s,) = args
            if not isinstance(s, _Captured):
                raise Unsupported("length of a non-captured sequence")
            return L.Len(self.host_array(s.v))
        raise Unsupported(f"builtin {name}")

    def tensor_op(self, name, args, scope, depth):
        S = self.S
        t = self.expr(args[0], scope, depth)
        if not isinstance(t, _Captured) or not isinstance(t.v, self.R.TensorView):
            raise Unsupported(f"{name} on a non-captured tensor")
        if not isinstance(args[1], S.SeqE):
            raise Unsupported(f"{name} index must be a literal sequence")
        idx = [self.as_expr(self.expr(x, scope, depth)) for x in args[1].items]
        arr = self.host_array(t.v)
        if name == "tensorGet":
            return L.TGet(arr, idx)
        return L.TSet(arr, idx, self.as_expr(self.expr(args[2], scope, depth)))


class _Captured:
    def __init__(self, v):
        self.v = v


# ============================================================ installation

def _elem_type(s: list) -> str:
    if not s:
        return "int"
    x = s[0]
    if isinstance(x, bool):
        return "bool"
    if isinstance(x, int):
        return "int"
    if isinstance(x, float):
        return "float"
    if isinstance(x, str):
        return "char"
    if isinstance(x, dict):
        return "record"
    raise Unsupported(f"sequence of {type(x).__name__}")


class DeviceList(list):
    """A construct's result as the reference sees it (a Python list, fully
    populated) that also carries its device sequence, so a later construct of
    the same accelerate call consumes it without another upload."""

    def __init__(self, values, dev=None):
        super().__init__(values)
        self.dev = dev


class _WatchedBuffer(list):
    """A heap buffer mirrored on the device: host-side writes (the
    interpreter's tensorSet outside a construct, interp.py:471-474) mark the
    device copy stale."""

    def __init__(self, values, mirror):
        super().__init__(values)
        self.mirror = mirror

    def __setitem__(self, k, v):
        self.mirror.host_newer = True
        list.__setitem__(self, k, v)


class _Mirror:
    """Device copy of one heap buffer for the duration of an accelerate call."""

    def __init__(self, heap, bid):
        from . import _lib
        buf = heap.buffers[bid]
        self.elem_float = bool(buf) and isinstance(buf[0], float)
        if not isinstance(buf, _WatchedBuffer):
            buf = _WatchedBuffer(buf, self)
            heap.buffers[bid] = buf                 # the interpreter looks buffers up by id
        self.buf = buf
        self.data = None
        self.host_newer = True
        self.dtype_code = None
        self.uploads = 0
        self._lib = _lib

    def device(self, elem: str):
        import numpy as np
        from .runtime import to_device
        if self.data is None or self.host_newer:
            np_t = np.float64 if elem == "float" else np.int64
            self.data = to_device(np.array(self.buf, dtype=np_t))
            self.dtype_code = self._lib.PMX_F64 if elem == "float" else self._lib.PMX_I64
            self.host_newer = False
            self.uploads += 1
        return self.data

    def copy_back(self):
        vals = self.data.to("cpu").numpy().tolist()
        if self.dtype_code == self._lib.PMX_F64:
            vals = [float(v) for v in vals]
        list.__setitem__(self.buf, slice(None), vals)   # coherent: not a host write


class CallState:
    """Device state of one accelerate call (`device_call` below): every host
    sequence is uploaded at most once and construct results stay on the
    device for the constructs that follow; every heap buffer a construct
    touches is mirrored once and copied back after a construct writes it.
    This is the single Alg. 2 marshal per accelerate (pmx/runtime.py:227-282)
    on the device side: the reference's own marshal_in builds the roots, the
    roots and sequences cross to the B200 once."""

    def __init__(self, heap):
        self.heap = heap
        self.seqs: dict = {}
        self.mirrors: dict = {}
        self.h2d_sequences = 0

    def seq(self, s):
        from .runtime import seq_to_device
        if isinstance(s, DeviceList) and s.dev is not None:
            return s.dev
        hit = self.seqs.get(id(s))
        if hit is not None and hit[0] is s:
            return hit[1]
        d = seq_to_device(s)
        self.seqs[id(s)] = (s, d)                   # keeps s alive: its id stays unique
        self.h2d_sequences += 1
        return d

    def mirror(self, bid) -> _Mirror:
        m = self.mirrors.get(bid)
        if m is None:
            m = self.mirrors[bid] = _Mirror(self.heap, bid)
        return m


def install(interp, *, device_call: bool = True):
    """Replace pmx.interp's parallel skeletons (and, by default, its
    `device_call`) by the B200 versions.  Returns an `uninstall()` callable
    restoring the originals."""
    from . import skeletons as K
    from .diagnostics import Diagnostics as B200Diagnostics
    from .dropin_programs import recognise
    from .runtime import seq_to_host
    pkg = interp.__name__.rsplit(".", 1)[0]
    syn = __import__(pkg + ".syntax", fromlist=["x"])
    rt = __import__(pkg + ".runtime", fromlist=["x"])
    names = ["eval_map", "eval_map2", "eval_reduce", "eval_loop"] + (["device_call"] if device_call else [])
    orig = {n: getattr(interp, n) for n in names}

    def state(ctx) -> CallState:
        cs = getattr(ctx, "_b200_call", None)
        return cs if cs is not None else CallState(ctx.heap)   # per construct outside our device_call

    def translate(f, n, ctx, span, touched, cs):
        def host_array(v):
            if isinstance(v, rt.TensorView):
                t = HeapTensor(v, cs.mirror(v.buffer))
                touched.append(t)
                return t
            return cs.seq(v)
        try:
            lam = to_lam(f, n, syn, rt, host_array)
        except (Unsupported, CompileError) as exc:
            raise rt.runtime_error(f"not supported on the B200 device: {exc}", span) from None
        _mark_written(lam, touched)
        return lam

    def to_ref(seq):
        vals = seq_to_host(seq).tolist()
        if seq.elem_tag == "char":
            vals = [chr(v) for v in vals]
        elif seq.elem_tag == "bool":
            vals = [bool(v) for v in vals]
        return DeviceList(vals, seq)

    def on_device(ctx, span, touched, body):
        dctx = K.Ctx(check_determinism=bool(getattr(ctx, "check_determinism", False)))
        dctx.device = True
        K._ctx_stack.append(dctx)
        try:
            out = body()
            dctx.check_errors()
        except B200Diagnostics as d:               # device error -> the reference's Diagnostics
            raise rt.runtime_error(d.items[0].message, span) from None
        finally:
            K._ctx_stack.pop()
        for t in touched:                           # tensors the construct wrote (tensorSet)
            if t.written:
                t.mirror.copy_back()
        return out

    def run(f, n, ctx, span, body):
        cs = state(ctx)
        touched: list = []
        lam = translate(f, n, ctx, span, touched, cs)
        return on_device(ctx, span, touched, lambda: body(lam, cs))

    def run_rows(f, s, ctx, span):
        cs = state(ctx)
        touched: list = []

        def host_array(v):
            if isinstance(v, rt.TensorView):
                t = HeapTensor(v, cs.mirror(v.buffer))
                touched.append(t)
                return t
            return cs.seq(v)
        try:
            g, op, acc = to_row_fold(f, syn, rt, host_array)
        except (Unsupported, CompileError) as exc:
            raise rt.runtime_error(f"not supported on the B200 device: {exc}", span) from None
        return on_device(ctx, span, touched, lambda: to_ref(K.map_rows_fold(g, op, acc, cs.seq(s))))

    def eval_map(f, s, ctx, span):
        if not ctx.run_parallel or not s:
            return orig["eval_map"](f, s, ctx, span)
        if isinstance(s[0], list):                  # row function over [[a]]
            return run_rows(f, s, ctx, span)
        _elem_type(s)
        return run(f, 1, ctx, span, lambda lam, cs: to_ref(K._materialize(K.eval_map(lam, cs.seq(s)))))

    def eval_map2(f, s1, s2, ctx, span):
        if not ctx.run_parallel or not s1:
            return orig["eval_map2"](f, s1, s2, ctx, span)
        return run(f, 2, ctx, span, lambda lam, cs: to_ref(K.eval_map2(lam, cs.seq(s1), cs.seq(s2))))

    def eval_reduce(f, acc, s, ctx, span):
        if not ctx.run_parallel or not s:
            return orig["eval_reduce"](f, acc, s, ctx, span)
        return run(f, 2, ctx, span, lambda lam, cs: K.eval_reduce(lam, acc, cs.seq(s)).get())

    def eval_loop(n, f, ctx, span):
        if not ctx.run_parallel or n <= 0:
            return orig["eval_loop"](n, f, ctx, span)
        return run(f, 1, ctx, span, lambda lam, cs: K.eval_loop(n, lam))

    def b200_device_call(fn, args, ctx, span):
        """interp.device_call (pmx/interp.py:230-237) with the device state of
        the call: the reference's checks and Alg. 2 marshal_in, the body in
        device context (its constructs run on the B200 and share one
        CallState), then marshal_out."""
        if ctx.checks:
            for a in args:
                interp._check_arg(fn.verdict, a, ctx)
        # a case-study binding (rk4.pmx, viterbi.pmx, nn.pmx, Appendix A) runs as
        # its hand-written kernel (dropin_programs.py); anything else below
        hit = recognise(fn, args, syn, rt)
        if hit is not None:
            family, thunk = hit
            install.last_binding = family
            return on_device(ctx, span, [], thunk)
        install.last_binding = None
        dev_args, arena = interp.marshal_in(args, ctx.heap)
        env = interp.Env(fn.env, dict(zip(fn.params, dev_args)))
        dctx = ctx.device_clone()
        dctx._b200_call = CallState(ctx.heap)
        result = interp.eval_expr(fn.body, env, dctx)
        install.last_call = dctx._b200_call
        return interp.marshal_out(arena, ctx.heap, result)

    interp.eval_map, interp.eval_map2 = eval_map, eval_map2
    interp.eval_reduce, interp.eval_loop = eval_reduce, eval_loop
    if device_call:
        interp.device_call = b200_device_call

    def uninstall():
        for name, fn in orig.items():
            setattr(interp, name, fn)
    return uninstall


install.last_call = None
install.last_binding = None


def _mark_written(lam, touched):
    """Flag the HeapTensors a lambda writes (TSet targets)."""
    written = set()

    def walk(e):
        if isinstance(e, L.TSet):
            written.add(id(e.tensor))
        for v in getattr(e, "__dict__", {}).values():
            if isinstance(v, L.Expr):
                walk(v)
            elif isinstance(v, (list, tuple)):
                for x in v:
                    if isinstance(x, L.Expr):
                        walk(x)
    walk(lam.body)
    for t in touched:
        t.written = t.written or id(t) in written


class HeapTensor:
    """A reference TensorView (a view into a heap buffer, a Python list) used
    by a device construct, backed by the call's device mirror of that buffer
    (uploaded once per accelerate call, copied back after a construct writes
    it: the tensorSet effects of interp.py:471-474)."""

    def __init__(self, view, mirror: _Mirror):
        from . import _lib
        self.view = view
        self.mirror = mirror
        self.shape = tuple(view.shape)
        self.dtype_code = _lib.PMX_F64 if view.elem == "float" else _lib.PMX_I64
        self.written = False

    @property
    def data(self):
        return self.mirror.data

    def as_pmx_array(self, write: bool = True):
        from . import _lib
        d = self.mirror.device(self.view.elem)
        a = _lib.Array()
        a.data = d.data_ptr()
        a.offset = self.view.offset
        for i, n in enumerate(self.shape):
            a.shape[i] = n
        a.rank = len(self.shape)
        a.dtype = self.dtype_code
        return a

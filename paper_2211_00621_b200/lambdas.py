"""Scalar lambdas of the accelerated subset and their compiler to device bytecode.

The reference passes function arguments to its skeletons as interpreted
closures (`Closure` / `BuiltinPartial`, pmx/runtime.py:78-93) — ASTs, not
callables.  The B200 backend receives the same information as a small
expression IR (this module), type-checks it against the element types of the
sequences it is applied to (monomorphic, like pmx/typecheck.py), and lowers it
to the register bytecode of include/pmx_b200.h that the device interpreter
(csrc/vm.cuh) runs, or that the library recognises as a fast-path shape.

Building lambdas:

    lam("x", addf(mulf(2.0, "x"), 1.0))          # PMExpr: lam x. addf (mulf 2.0 x) 1.0
    lam(lambda x: addf(mulf(2.0, x), 1.0))       # same, traced from Python
    addf                                          # a builtin used as a function value
    lam("a", "b", if_(lti("a", "b"), "a", "b"))   # match lti a b with true then a else b

Strings stand for variables; Python ints/floats/bools are Int/Float/Bool
constants; `char("a")` is a Char literal.
"""
from __future__ import annotations

import ctypes as C
import inspect
import struct
from dataclasses import dataclass, field
from typing import Any, Callable, Optional

from . import _lib
from ._lib import OP

_lib_E_RECURSION = 13      # enum pmx_code PMX_E_RECURSION

# ============================================================================ IR


class Expr:
    # operator sugar builds generic primitives, resolved by type at compile time
    def __add__(self, o): return Prim("add", [self, lift(o)])
    def __radd__(self, o): return Prim("add", [lift(o), self])
    def __sub__(self, o): return Prim("sub", [self, lift(o)])
    def __rsub__(self, o): return Prim("sub", [lift(o), self])
    def __mul__(self, o): return Prim("mul", [self, lift(o)])
    def __rmul__(self, o): return Prim("mul", [lift(o), self])
    def __truediv__(self, o): return Prim("div", [self, lift(o)])
    def __rtruediv__(self, o): return Prim("div", [lift(o), self])
    def __neg__(self): return Prim("neg", [self])
    def __lt__(self, o): return Prim("lt", [self, lift(o)])
    def __gt__(self, o): return Prim("gt", [self, lift(o)])
    def __le__(self, o): return Prim("le", [self, lift(o)])
    def __ge__(self, o): return Prim("ge", [self, lift(o)])


@dataclass(eq=False)
class Var(Expr):
    name: str


@dataclass(eq=False)
class Const(Expr):
    value: Any
    ty: str  # "int" | "float" | "bool" | "char"


@dataclass(eq=False)
class Prim(Expr):
    name: str
    args: list


@dataclass(eq=False)
class If(Expr):
    cond: Expr
    then: Expr
    els: Expr


@dataclass(eq=False)
class LetE(Expr):
    name: str
    value: Expr
    body: Expr


@dataclass(eq=False)
class Get(Expr):
    arr: Any       # a device sequence (captured host data, rank 1)
    index: Expr


@dataclass(eq=False)
class Len(Expr):
    arr: Any


@dataclass(eq=False)
class TGet(Expr):
    tensor: Any    # a DeviceTensor view
    index: list


@dataclass(eq=False)
class TSet(Expr):
    tensor: Any
    index: list
    value: Expr


@dataclass(eq=False)
class Do(Expr):
    """Sequence effects; value of the last (PMExpr `let u = e1 in e2`)."""
    exprs: list


@dataclass(eq=False)
class Never(Expr):
    pass


# Bound on the iterations of a linear recursion run as a loop (the reference
# itself fails with a RecursionError long before this depth).
ITERATE_LIMIT = 1 << 24


@dataclass(eq=False)
class Iterate(Expr):
    """acc = init; for m in [lo, hi]: acc = body(m, acc); the value is acc.

    The device form of a linear recursion f p = match p with c then base
    else E[f (p - 1)]: evaluated from the base case up, E applied with
    p = c+1 .. p (the reference evaluates the same expressions innermost
    call first).

    `more` generalises it to a k-term recurrence f p = E[f (p-1), .., f (p-k)]
    with base cases at c .. c+k-1 (lo = c+k): acc holds f(m-1) and
    more[i] = (name, init) holds f(m-2-i), initialised to f(lo-2-i).  A base
    value is evaluated only when hi reaches its level (the reference only
    evaluates the cases it recurses into); for hi in [lo-k, lo-1] the value is
    that base case, below lo-k the recursion never reaches a base case."""
    var: str
    lo: Expr
    hi: Expr
    acc: str
    init: Expr
    body: Expr
    more: tuple = ()


@dataclass(eq=False)
class Field(Expr):
    """Record projection r.l (SoA: selects one column of a record sequence)."""
    rec: Expr
    label: str


def field_(rec, label: str) -> Field:
    return Field(lift(rec), label)


def char(c: str) -> Const:
    assert len(c) == 1
    return Const(ord(c), "char")


def lift(x) -> Expr:
    if isinstance(x, Expr):
        return x
    if isinstance(x, str):
        return Var(x)
    if isinstance(x, bool):
        return Const(bool(x), "bool")
    if isinstance(x, int):
        return Const(int(x), "int")
    if isinstance(x, float):
        return Const(float(x), "float")
    raise TypeError(f"cannot use {type(x).__name__} in a device lambda")


class Lam:
    """A lambda of `len(params)` parameters (curried in PMExpr)."""

    def __init__(self, params: list[str], body: Expr):
        self.params = list(params)
        self.body = body

    def __repr__(self) -> str:
        return f"Lam({self.params}, {self.body!r})"


def lam(*args) -> Lam:
    """lam("x", body) / lam("x", "y", body) / lam(python_callable)."""
    if len(args) == 1 and callable(args[0]) and not isinstance(args[0], (Expr, Builtin, Lam)):
        fn = args[0]
        n = len(inspect.signature(fn).parameters)
        names = [f"_p{i}" for i in range(n)]
        return Lam(names, lift(fn(*[Var(v) for v in names])))
    *params, body = args
    return Lam(list(params), lift(body))


class Builtin:
    """A builtin operator; calling it builds a primitive, and it is itself a
    function value (BuiltinPartial, pmx/runtime.py:88-93)."""

    def __init__(self, name: str, arity: int):
        self.name = name
        self.arity = arity

    def __call__(self, *args):
        if len(args) != self.arity:
            raise TypeError(f"{self.name} takes {self.arity} arguments")
        return Prim(self.name, [lift(a) for a in args])

    def as_lam(self) -> Lam:
        if getattr(self, "_lam", None) is None:
            ps = [f"_b{i}" for i in range(self.arity)]
            self._lam = Lam(ps, Prim(self.name, [Var(p) for p in ps]))
        return self._lam

    def __repr__(self) -> str:
        return self.name


# builtin names and arities follow pmx/syntax.py:196-209 (scalar subset)
_ARITY = {
    "addi": 2, "subi": 2, "muli": 2, "divi": 2, "modi": 2, "negi": 1,
    "addf": 2, "subf": 2, "mulf": 2, "divf": 2, "negf": 1,
    "eqi": 2, "neqi": 2, "lti": 2, "gti": 2, "leqi": 2, "geqi": 2,
    "eqf": 2, "ltf": 2, "gtf": 2, "leqf": 2, "geqf": 2,
    "int2float": 1, "floor": 1, "exp": 1, "log": 1, "sqrtf": 1, "sin": 1, "cos": 1,
}
BUILTINS = {n: Builtin(n, a) for n, a in _ARITY.items()}
globals().update(BUILTINS)


def if_(c, a, b) -> If:
    return If(lift(c), lift(a), lift(b))


def match(scrut, pattern, then, els) -> If:
    """match scrut with <literal> then .. else ..  (pattern is a literal)."""
    return If(Prim("eq", [lift(scrut), lift(pattern)]), lift(then), lift(els))


def let(name: str, value, body) -> LetE:
    return LetE(name, lift(value), lift(body))


def get(arr, index) -> Get:
    return Get(arr, lift(index))


def length(arr) -> Len:
    return Len(arr)


def tensor_get(t, index) -> TGet:
    return TGet(t, [lift(i) for i in index])


def tensor_set(t, index, value) -> TSet:
    return TSet(t, [lift(i) for i in index], lift(value))


def do(*exprs) -> Do:
    return Do([lift(e) for e in exprs])


def as_lam(f) -> Lam:
    if isinstance(f, Lam):
        return f
    if isinstance(f, Builtin):
        return f.as_lam()
    if callable(f):
        return lam(f)
    raise TypeError(f"not a function value: {f!r}")


# ===================================================================== compiler

class CompileError(Exception):
    pass


_TYPED = {
    # generic -> (int op, float op)
    "add": ("ADDI", "ADDF"), "sub": ("SUBI", "SUBF"), "mul": ("MULI", "MULF"),
    "div": ("DIVI", "DIVF"), "neg": ("NEGI", "NEGF"),
    "lt": ("LTI", "LTF"), "gt": ("GTI", "GTF"), "le": ("LEQI", "LEQF"), "ge": ("GEQI", "GEQF"),
    "eq": ("EQI", "EQF"), "ne": ("NEQI", None),
}
_FIXED = {
    # builtin -> (opcode, arg types, result type)
    "addi": ("ADDI", ("int", "int"), "int"), "subi": ("SUBI", ("int", "int"), "int"),
    "muli": ("MULI", ("int", "int"), "int"), "divi": ("DIVI", ("int", "int"), "int"),
    "modi": ("MODI", ("int", "int"), "int"), "negi": ("NEGI", ("int",), "int"),
    "addf": ("ADDF", ("float", "float"), "float"), "subf": ("SUBF", ("float", "float"), "float"),
    "mulf": ("MULF", ("float", "float"), "float"), "divf": ("DIVF", ("float", "float"), "float"),
    "negf": ("NEGF", ("float",), "float"),
    "eqi": ("EQI", ("int", "int"), "bool"), "neqi": ("NEQI", ("int", "int"), "bool"),
    "lti": ("LTI", ("int", "int"), "bool"), "gti": ("GTI", ("int", "int"), "bool"),
    "leqi": ("LEQI", ("int", "int"), "bool"), "geqi": ("GEQI", ("int", "int"), "bool"),
    "eqf": ("EQF", ("float", "float"), "bool"), "ltf": ("LTF", ("float", "float"), "bool"),
    "gtf": ("GTF", ("float", "float"), "bool"), "leqf": ("LEQF", ("float", "float"), "bool"),
    "geqf": ("GEQF", ("float", "float"), "bool"),
    "int2float": ("INT2FLOAT", ("int",), "float"), "floor": ("FLOOR", ("float",), "int"),
    "exp": ("EXP", ("float",), "float"), "log": ("LOG", ("float",), "float"),
    "sqrtf": ("SQRT", ("float",), "float"), "sin": ("SIN", ("float",), "float"),
    "cos": ("COS", ("float",), "float"),
}

DTYPE_TYPE = {_lib.PMX_F32: "float", _lib.PMX_F64: "float", _lib.PMX_I64: "int",
              _lib.PMX_I32: "int", _lib.PMX_BOOL: "bool"}


def _int_like(t: str) -> bool:
    return t in ("int", "char")


@dataclass
class Compiled:
    program: _lib.Program
    out_type: str
    kind: int = 0      # fast-path kind reported by the library (0 = interpreter)
    insns: list = field(default_factory=list)


class _Gen:
    def __init__(self, n_inputs: int):
        self.insns: list[list[int]] = []
        self.consts: list[int] = []
        self.const_ix: dict[tuple, int] = {}
        self.arrays: list[Any] = []
        self.written: set[int] = set()          # arrays a TSET stores into
        self.free = list(range(_lib.MAX_REGS - 1, n_inputs - 1, -1))  # pop() gives lowest
        self.n_inputs = n_inputs

    # -- resources
    def reg(self) -> int:
        if not self.free:
            raise CompileError("lambda needs more than 32 registers")
        return self.free.pop()

    def release(self, o: int) -> None:
        if self.n_inputs <= o < 32 and o not in self.free:
            self.free.append(o)
            self.free.sort(reverse=True)

    def const(self, value, ty: str) -> int:
        if ty == "float":
            bits = struct.unpack("<q", struct.pack("<d", float(value)))[0]
        else:
            bits = int(value)
            bits = ((bits + (1 << 63)) % (1 << 64)) - (1 << 63)
        key = (ty == "float", bits)
        if key not in self.const_ix:
            if len(self.consts) >= _lib.MAX_CONSTS:
                raise CompileError("lambda needs more than 32 constants")
            self.const_ix[key] = len(self.consts)
            self.consts.append(bits)
        return 32 + self.const_ix[key]

    def array(self, arr) -> int:
        for i, a in enumerate(self.arrays):
            if a is arr:
                return i
        if len(self.arrays) >= _lib.MAX_ARRAYS:
            raise CompileError("lambda captures more than 6 sequences/tensors")
        self.arrays.append(arr)
        return len(self.arrays) - 1

    def emit(self, op: str, dst=0, a=0, b=0, c=0) -> int:
        if len(self.insns) >= _lib.MAX_INSNS:
            raise CompileError("lambda too long for the device interpreter (96 instructions)")
        self.insns.append([OP[op], dst, a, b, c])
        return len(self.insns) - 1

    def patch(self, at: int, target: int) -> None:
        self.insns[at][3] = target & 0xFF
        self.insns[at][4] = target >> 8


def _simple(e: Expr) -> bool:
    return isinstance(e, (Var, Const))


def _compile(e: Expr, env: dict, g: _Gen) -> tuple[int, str, bool]:
    """Returns (operand, type, owned) — owned temporaries are released by the caller."""
    if isinstance(e, Var):
        if e.name not in env:
            raise CompileError(f"unbound variable {e.name!r} in device lambda")
        o, t = env[e.name]
        return o, t, False
    if isinstance(e, Const):
        ty = "int" if e.ty == "char" else e.ty
        v = int(e.value) if e.ty == "bool" else e.value
        return g.const(v, "float" if ty == "float" else "int"), e.ty, False
    if isinstance(e, Prim):
        args = [_compile(a, env, g) for a in e.args]
        if e.name in _FIXED:
            op, ats, rt = _FIXED[e.name]
            for (o, t, _), want in zip(args, ats):
                if not (t == want or (want == "int" and _int_like(t))):
                    raise CompileError(f"{e.name} expects {want}, got {t}")
        elif e.name in _TYPED:
            ts = {t for _, t, _ in args}
            if len(ts) != 1:
                raise CompileError(f"{e.name}: mismatched operand types {sorted(ts)}")
            t = ts.pop()
            if t == "bool" and e.name in ("eq", "ne"):
                op = "EQB" if e.name == "eq" else None
                if op is None:
                    raise CompileError("ne on Bool")
            elif _int_like(t):
                op = _TYPED[e.name][0]
            elif t == "float":
                op = _TYPED[e.name][1]
                if op is None:
                    raise CompileError(f"{e.name} on Float")
            else:
                raise CompileError(f"{e.name} on {t}")
            rt = t if e.name in ("add", "sub", "mul", "div", "neg") else "bool"
        else:
            raise CompileError(f"builtin {e.name!r} is not supported on the device")
        for o, _, owned in args:
            if owned:
                g.release(o)
        dst = g.reg()
        ops = [o for o, _, _ in args] + [0, 0]
        g.emit(op, dst, ops[0], ops[1])
        return dst, rt, True
    if isinstance(e, If):
        c, ct, cown = _compile(e.cond, env, g)
        if ct != "bool":
            raise CompileError("condition must be Bool")
        if _simple(e.then) and _simple(e.els):
            a, at, _ = _compile(e.then, env, g)
            b, bt, _ = _compile(e.els, env, g)
            if at != bt:
                raise CompileError("match branches have different types")
            if cown:
                g.release(c)
            dst = g.reg()
            g.emit("SELECT", dst, c, a, b)
            return dst, at, True
        dst = g.reg()
        jz = g.emit("JZ", 0, c)
        if cown:
            g.release(c)
        a, at, aown = _compile(e.then, env, g)
        g.emit("MOV", dst, a)
        if aown:
            g.release(a)
        jmp = g.emit("JMP")
        g.patch(jz, len(g.insns))
        b, bt, bown = _compile(e.els, env, g)
        if at != bt and not (isinstance(e.els, Never) or isinstance(e.then, Never)):
            raise CompileError("match branches have different types")
        g.emit("MOV", dst, b)
        if bown:
            g.release(b)
        g.patch(jmp, len(g.insns))
        return dst, at if not isinstance(e.then, Never) else bt, True
    if isinstance(e, LetE):
        v, vt, vown = _compile(e.value, env, g)
        if not vown and v < 32:          # alias an input register: copy to keep it stable
            pass
        env2 = dict(env)
        env2[e.name] = (v, vt)
        r, rt, rown = _compile(e.body, env2, g)
        if vown and v != r:
            g.release(v)
        return r, rt, rown
    if isinstance(e, Get):
        i, it, iown = _compile(e.index, env, g)
        if not _int_like(it):
            raise CompileError("get index must be Int")
        k = g.array(e.arr)
        if iown:
            g.release(i)
        dst = g.reg()
        g.emit("GET", dst, i, 0, k)
        return dst, DTYPE_TYPE[e.arr.dtype_code], True
    if isinstance(e, Len):
        k = g.array(e.arr)
        dst = g.reg()
        g.emit("LEN", dst, 0, 0, k)
        return dst, "int", True
    if isinstance(e, (TGet, TSet)):
        t = e.tensor
        if len(e.index) != len(t.shape):
            raise CompileError(f"tensor index of rank {len(e.index)} against rank {len(t.shape)} tensor")
        k = g.array(t)
        base = _consecutive(g, len(e.index))
        for d, ie in enumerate(e.index):
            o, ot, own = _compile(ie, env, g)
            if not _int_like(ot):
                raise CompileError("tensor index must be Int")
            g.emit("MOV", base + d, o)
            if own:
                g.release(o)
        if isinstance(e, TGet):
            dst = g.reg()
            g.emit("TGET", dst, base, 0, k)
            for d in range(len(e.index)):
                g.release(base + d)
            return dst, DTYPE_TYPE[t.dtype_code], True
        v, vt, vown = _compile(e.value, env, g)
        g.emit("TSET", 0, base, v, k)
        g.written.add(k)
        if vown:
            g.release(v)
        for d in range(len(e.index)):
            g.release(base + d)
        return g.const(0, "int"), "unit", False
    if isinstance(e, Do):
        r, rt, rown = g.const(0, "int"), "unit", False
        for x in e.exprs:
            if rown:
                g.release(r)
            r, rt, rown = _compile(x, env, g)
        return r, rt, rown
    if isinstance(e, Never):
        g.emit("NEVER")
        return g.const(0, "int"), "never", False
    if isinstance(e, Iterate):
        k = 1 + len(e.more)
        lo, lt, lown = _compile(e.lo, env, g)
        hi, ht, hown = _compile(e.hi, env, g)
        if not (_int_like(lt) and _int_like(ht)):
            raise CompileError("recursion counter must be Int")
        m, h = g.reg(), g.reg()
        g.emit("MOV", m, lo)
        g.emit("MOV", h, hi)
        if lown:
            g.release(lo)
        if hown:
            g.release(hi)
        # depth bound: -k <= hi - lo <= ITERATE_LIMIT. hi < lo - k never reaches
        # a base case (the reference recurses until its stack overflows); the
        # upper bound stands in for that stack (the reference overflows first)
        span, big = g.reg(), g.reg()
        g.emit("SUBI", span, h, m)
        g.emit("GTI", big, span, g.const(ITERATE_LIMIT, "int"))
        ok = g.emit("JZ", 0, big)
        g.emit("FAIL", 0, 0, _lib_E_RECURSION)
        g.patch(ok, len(g.insns))
        g.emit("LTI", big, span, g.const(-k, "int"))
        ok = g.emit("JZ", 0, big)
        g.emit("FAIL", 0, 0, _lib_E_RECURSION)
        g.patch(ok, len(g.insns))
        g.release(big)
        if k == 1:
            g.release(span)
        names = [e.acc] + [n for n, _ in e.more]
        inits = [e.init] + [x for _, x in e.more]
        accs = []
        at = None
        for j, (nm, x) in enumerate(zip(names, inits)):
            # acc j holds f(lo - 1 - j): evaluated only when hi >= lo - 1 - j
            acc = g.reg()
            skip = None
            if k > 1:
                c = g.reg()
                g.emit("GEQI", c, span, g.const(-1 - j, "int"))
                skip = g.emit("JZ", 0, c)
                g.release(c)
            a0, t0, aown = _compile(x, env, g)
            if at is None:
                at = t0
            elif t0 not in (at, "never") and at != "never":
                raise CompileError("recursion base cases differ in type")
            elif at == "never":
                at = t0
            g.emit("MOV", acc, a0)
            if aown:
                g.release(a0)
            if skip is not None:
                done = g.emit("JMP")
                g.patch(skip, len(g.insns))
                g.emit("MOV", acc, g.const(0, "int"))
                g.patch(done, len(g.insns))
            accs.append(acc)
        top = len(g.insns)
        c = g.reg()
        g.emit("LEQI", c, m, h)
        jz = g.emit("JZ", 0, c)
        g.release(c)
        env2 = dict(env)
        env2[e.var] = (m, "int")
        for nm, acc in zip(names, accs):
            env2[nm] = (acc, at)
        b, bt, bown = _compile(e.body, env2, g)
        if bt != at and not (at == "never" or bt == "never"):
            raise CompileError("recursion step changes the result type")
        for j in range(k - 1, 0, -1):                  # shift: f(m-1-j) <- f(m-j)
            g.emit("MOV", accs[j], accs[j - 1])
        g.emit("MOV", accs[0], b)
        if bown:
            g.release(b)
        g.emit("ADDI", m, m, g.const(1, "int"))
        back = g.emit("JMP")
        g.patch(back, top)
        g.patch(jz, len(g.insns))
        g.release(m)
        g.release(h)
        if k > 1:
            # no step ran (hi < lo): the value is the base case f(hi) = acc[lo-1-hi]
            res = g.reg()
            g.emit("MOV", res, accs[0])
            for j in range(1, k):
                c = g.reg()
                g.emit("EQI", c, span, g.const(-1 - j, "int"))
                g.emit("SELECT", res, c, accs[j], res)
                g.release(c)
            g.release(span)
            for acc in accs:
                g.release(acc)
            return res, at, True
        return accs[0], at, True
    raise CompileError(f"cannot compile {type(e).__name__} for the device")


def _consecutive(g: _Gen, n: int) -> int:
    """Reserve n consecutive registers (for tensor index operands)."""
    free = sorted(g.free)
    for start in free:
        if all((start + d) in g.free for d in range(n)):
            for d in range(n):
                g.free.remove(start + d)
            return start
    raise CompileError("out of registers for a tensor index")


def compile_lambda(f, in_types: list[str], state_array=None) -> Compiled:
    """Lower a function value applied to arguments of `in_types`.

    Register convention of pmx_b200.h: the lambda's parameters occupy
    r0..r(k-1); extra implicit inputs (element index, step) follow them.
    `state_array` reserves arrays[0] (seqLoop's previous state)."""
    fl = as_lam(f)
    if len(fl.params) > len(in_types):
        raise CompileError(f"lambda takes {len(fl.params)} arguments, applied to {len(in_types)}")
    # lambdas are immutable: memoise the lowering per argument types
    key = (tuple(in_types), id(state_array))
    cache = fl.__dict__.setdefault("_compiled", {})
    if key in cache:
        return cache[key]
    cache[key] = out = _lower(fl, in_types, state_array)
    return out


def _lower(fl: Lam, in_types: list[str], state_array) -> Compiled:
    g = _Gen(len(in_types))
    if state_array is not None:
        g.array(state_array)
    env = {p: (i, t) for i, (p, t) in enumerate(zip(fl.params, in_types))}
    o, t, _ = _compile(fl.body, env, g)
    prog = _lib.Program()
    prog.n_insns = len(g.insns)
    prog.n_inputs = len(in_types)
    prog.out = o
    prog.out_is_float = 1 if t == "float" else 0
    prog.n_arrays = len(g.arrays)
    for i, (op, dst, a, b, c) in enumerate(g.insns):
        prog.insns[i] = _lib.Insn(op, dst, a, b, c, 0, 0, 0)
    for i, v in enumerate(g.consts):
        prog.consts[i] = v
    for i, arr in enumerate(g.arrays):
        prog.arrays[i] = arr.as_pmx_array(write=i in g.written)
    return Compiled(prog, t, insns=[list(x) for x in g.insns])

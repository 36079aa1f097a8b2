"""Seeded random scalar lambdas for differential testing of the device
interpreter, the run-time specialised kernels and the CPU oracle.

Programs mix Int and Float arithmetic (wrap-around, truncating divi/modi,
fp64 without contraction), comparisons, lazy `if_` branches (match jumps)
and select-able branches, let-bindings and the builtins that can raise the
reference's runtime errors (divi/modi by zero, divf by zero, log domain,
sqrtf of a negative, exp overflow), so both the values and the first-failing
element of a sequence are exercised."""
from __future__ import annotations

import random

from paper_2211_00621_b200.lambdas import (
    addf, addi, cos, divf, divi, exp, floor, gtf, gti, if_, int2float, lam, let, log, ltf, lti, modi,
    mulf, muli, negf, negi, sin, sqrtf, subf, subi,
)

INT_CONST = [0, 1, 2, 3, 7, -5, 13, 1 << 40, -(1 << 62), 9223372036854775807]
FLOAT_CONST = [0.0, 0.5, 1.0, -2.25, 3.0, 1e-3, 1e300, -7.5, 0.1]


class Gen:
    def __init__(self, seed: int, var: str, ty: str, with_errors: bool = True):
        self.r = random.Random(seed)
        self.var, self.ty = var, ty
        self.errors = with_errors
        self.nlet = 0
        self.scope = {var: ty}

    def leaf(self, ty):
        names = [n for n, t in self.scope.items() if t == ty]
        if names and self.r.random() < 0.6:
            return self.r.choice(names)
        if ty == "int":
            return self.r.choice(INT_CONST)
        return self.r.choice(FLOAT_CONST)

    def cond(self, d):
        if self.r.random() < 0.5:
            return self.r.choice([lti, gti])(self.expr("int", d - 1), self.expr("int", d - 1))
        return self.r.choice([ltf, gtf])(self.expr("float", d - 1), self.expr("float", d - 1))

    def expr(self, ty, d):
        if d <= 0 or self.r.random() < 0.2:
            return self.leaf(ty)
        k = self.r.random()
        if k < 0.12:
            return if_(self.cond(d), self.expr(ty, d - 1), self.expr(ty, d - 1))
        if k < 0.2 and self.nlet < 3:
            name = f"v{self.nlet}"
            self.nlet += 1
            t2 = self.r.choice(["int", "float"])
            val = self.expr(t2, d - 1)
            self.scope[name] = t2
            body = self.expr(ty, d - 1)
            del self.scope[name]
            return let(name, val, body)
        if ty == "int":
            ops = [addi, subi, muli, negi, floor] + ([divi, modi] if self.errors else [])
            op = self.r.choice(ops)
            if op is negi:
                return negi(self.expr("int", d - 1))
            if op is floor:
                return floor(self.expr("float", d - 1))
            return op(self.expr("int", d - 1), self.expr("int", d - 1))
        ops = [addf, subf, mulf, negf, int2float, sin, cos] + ([divf, exp, log, sqrtf] if self.errors else [])
        op = self.r.choice(ops)
        if op in (negf, sin, cos, exp, log, sqrtf):
            return op(self.expr("float", d - 1))
        if op is int2float:
            return int2float(self.expr("int", d - 1))
        return op(self.expr("float", d - 1), self.expr("float", d - 1))


def random_lambda(seed: int, in_ty: str, out_ty: str, depth: int = 4, with_errors: bool = True):
    g = Gen(seed, "x", in_ty, with_errors)
    return lam("x", g.expr(out_ty, depth))


def random_inputs(seed: int, ty: str, n: int):
    r = random.Random(seed * 7919 + 1)
    if ty == "int":
        pool = [0, 1, -1, 2, 3, 5, -7, 100, 1 << 33, -(1 << 50)]
        return [r.choice(pool) if r.random() < 0.3 else r.randint(-1000, 1000) for _ in range(n)]
    pool = [0.0, -0.0, 1.0, -1.0, 0.5, 1e-300, 700.0, -3.5]
    return [r.choice(pool) if r.random() < 0.3 else r.uniform(-50.0, 50.0) for _ in range(n)]

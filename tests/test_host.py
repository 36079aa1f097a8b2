"""Host-side logic: lambda compiler, Alg. 2 interval merging, tensor views.
CPU only.  Interval tests restate tests/test_runtime.py:12-34 and the
randomised bitmap oracle of tests/test_acceptance.py:184-214."""
import random

import pytest

from paper_2211_00621_b200 import Diagnostics
from paper_2211_00621_b200.lambdas import (
    CompileError, addf, addi, compile_lambda, divi, get, if_, lam, let, lti, match, mulf, muli,
    tensor_set, int2float, floor, char,
)
from paper_2211_00621_b200.runtime import (
    Interval, TensorView, collect_tensors, merge_intervals, merge_overlapping_intervals,
)
from paper_2211_00621_b200 import _lib


# ------------------------------------------------------------- intervals

def test_touching_intervals_merge():
    assert merge_intervals([(0, 2), (2, 4)]) == [Interval(0, 4)]


def test_contained_and_unordered():
    assert merge_intervals([(0, 10), (3, 5)]) == [Interval(0, 10)]
    assert merge_intervals([(5, 6), (0, 2), (1, 4)]) == [Interval(0, 4), Interval(5, 6)]
    assert merge_intervals([(7, 9)]) == [Interval(7, 9)]


def test_merge_views_requires_one_buffer():
    views = [TensorView(0, 0, (2,), "int"), TensorView(0, 1, (3,), "int")]
    assert merge_overlapping_intervals(views) == [Interval(0, 4)]
    with pytest.raises(AssertionError):
        merge_overlapping_intervals([TensorView(0, 0, (1,), "int"), TensorView(1, 0, (1,), "int")])


def _bitmap_merge(pairs):
    hi = max(e for _, e in pairs)
    cells = [False] * hi
    for s, e in pairs:
        for i in range(s, e):
            cells[i] = True
    out, i = [], 0
    while i < hi:
        if cells[i]:
            j = i
            while j < hi and cells[j]:
                j += 1
            out.append(Interval(i, j))
            i = j
        else:
            i += 1
    return out


def test_interval_merging_random_vs_bitmap():
    rng = random.Random(7)
    for _ in range(1000):
        pairs = [(s, s + rng.randint(1, 10)) for s in (rng.randint(0, 50) for _ in range(rng.randint(1, 8)))]
        assert merge_intervals(pairs) == _bitmap_merge(pairs), pairs


def test_view_strides_and_linear():
    t = TensorView(0, 3, (2, 3, 4), "int")
    assert t.strides() == (12, 4, 1)
    assert t.linear([1, 2, 3]) == 3 + 12 + 8 + 3
    with pytest.raises(Diagnostics, match="out of bounds"):
        t.linear([0, 3, 0])
    with pytest.raises(Diagnostics, match="rank"):
        t.linear([0, 0])


def test_collect_tensors():
    t = TensorView(0, 0, (1,), "int")
    assert collect_tensors([{"x": t}, [t, 1], "c"]) == [t, t]


# ----------------------------------------------------------- compiler

def test_compile_types_and_outputs():
    c = compile_lambda(lam("x", int2float("x")), ["int", "int"])
    assert c.out_type == "float"
    c = compile_lambda(lam("x", floor("x")), ["float", "int"])
    assert c.out_type == "int"
    c = compile_lambda(lam("c", match("c", char("a"), 1, 0)), ["char", "int"])
    assert c.out_type == "int"


def test_compile_rejects_type_errors():
    with pytest.raises(CompileError):
        compile_lambda(lam("x", addf("x", 1.0)), ["int", "int"])
    with pytest.raises(CompileError):
        compile_lambda(lam("x", addi("x", 1.0)), ["int", "int"])
    with pytest.raises(CompileError):
        compile_lambda(lam("x", addi("y", 1)), ["int", "int"])


def test_lazy_branches_use_jumps_and_pure_ones_select():
    c = compile_lambda(lam("x", if_(lti("x", 5), muli("x", 2), divi("x", 0))), ["int", "int"])
    ops = [i[0] for i in c.insns]
    assert _lib.OP["JZ"] in ops and _lib.OP["JMP"] in ops
    c = compile_lambda(lam("a", "b", if_(lti("a", "b"), "a", "b")), ["int", "int"])
    assert [i[0] for i in c.insns] == [_lib.OP["LTI"], _lib.OP["SELECT"]]


def test_registers_are_recycled():
    # a long chain needs few registers
    e = "x"
    for k in range(40):
        e = addf(mulf(e, 1.0001), float(k % 8))
    c = compile_lambda(lam("x", e), ["float", "int"])
    assert max(max(i[1], i[2] if i[2] < 32 else 0) for i in c.insns) < 8


def test_python_callable_tracing():
    c1 = compile_lambda(lam(lambda x: x * 2.0 + 1.0), ["float", "int"])
    c2 = compile_lambda(lam("x", addf(mulf("x", 2.0), 1.0)), ["float", "int"])
    assert c1.insns == c2.insns


def test_let_binding():
    c = compile_lambda(lam("x", let("y", muli("x", "x"), addi("y", "y"))), ["int", "int"])
    assert c.out_type == "int"

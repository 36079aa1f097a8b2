"""Differential test over seeded random scalar lambdas: the device
interpreter, the run-time specialised kernels and the CPU oracle (pinned to
the reference interpreter by tests/test_oracle.py) agree on every element —
integers exactly, floats bit for bit between the two device paths (same CUDA
libm) and to 1e-15 relative against the oracle's glibc, and on the first
failing element and message when a runtime error occurs."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2211_00621_b200 import Diagnostics, _lib, accelerate, eval_map
from randprog import random_inputs, random_lambda

pytestmark = pytest.mark.gpu

N = 777
CASES = [(seed, ti, to) for seed in range(24) for ti, to in (("int", "int"), ("float", "float"),
                                                             ("int", "float"), ("float", "int"))]


def _run(f, xs, mode):
    lib = _lib.load()
    prev = lib.pmx_jit_set_mode(mode)
    try:
        return "ok", [v for v in np.asarray(accelerate(lambda s: eval_map(f, s), xs)).tolist()]
    except Diagnostics as d:
        return "err", str(d)
    finally:
        lib.pmx_jit_set_mode(prev)


def _oracle(f, xs):
    out = []
    for j, x in enumerate(xs):
        try:
            out.append(O.ir_apply(f, x))
        except O.OracleError as e:
            return "err", (j, str(e))
        except (ValueError, OverflowError):
            # floor of nan/inf: the reference itself crashes with a Python
            # exception (interp.py:426-427), no defined result to compare
            return "undef", j
    return "ok", out


@pytest.mark.parametrize("seed,ti,to", CASES, ids=[f"{s}-{a}-{b}" for s, a, b in CASES])
def test_random_lambda_vm_jit_oracle(seed, ti, to):
    f = random_lambda(seed, ti, to)
    xs = random_inputs(seed, ti, N)
    if ti == "float":
        xs = np.array(xs, np.float64)
    else:
        xs = np.array(xs, np.int64)
    vm = _run(f, xs, 0)
    jit = _run(f, xs, 1)
    ref = _oracle(f, xs.tolist())
    if ref[0] == "undef":
        assert vm[0] == jit[0]
        return
    assert vm[0] == jit[0] == ref[0], (vm[0], jit[0], ref, f)
    if vm[0] == "err":
        assert vm[1] == jit[1]
        j, msg = ref[1]
        assert f"element {j})" in vm[1], (vm[1], ref[1])
        return
    a, b, c = vm[1], jit[1], ref[1]
    for k, (u, v, w) in enumerate(zip(a, b, c)):
        if to == "int":
            assert int(u) == int(v) == int(w), (k, u, v, w)
        else:
            assert (u == v) or (math.isnan(u) and math.isnan(v)), (k, u, v)
            if math.isnan(w) or math.isinf(w):
                assert (math.isnan(u) and math.isnan(w)) or u == w, (k, u, w)
            else:
                assert math.isclose(u, w, rel_tol=1e-13, abs_tol=1e-300), (k, u, w)

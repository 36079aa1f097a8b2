"""Run-time kernel specialisation (csrc/jit.cu), CPU side: every golden
lambda translates to C++ and NVRTC compiles it for sm_100a into the
streaming skeleton kernels (no GPU needed for code generation + compile)."""
import ctypes as C

import pytest

from cases import MAP2_CASES, MAP_CASES
from paper_2211_00621_b200 import _lib
import torch

from paper_2211_00621_b200.lambdas import (
    addf, addi, compile_lambda, divi, lam, lti, if_, mulf, muli, tensor_get, tensor_set,
)
from paper_2211_00621_b200.runtime import DeviceTensor, _Root

CODE = {"int": _lib.PMX_I64, "float": _lib.PMX_F64, "char": _lib.PMX_I64, "bool": _lib.PMX_BOOL}


def _check(prog, kind, xt, yt, zt=0):
    lib = _lib.load()
    rc = lib.pmx_jit_compile_check(C.byref(prog), kind, xt, yt, zt)
    assert rc == 0, lib.pmx_last_error().decode()


def _out(comp, xt):
    if comp.out_type == "float":
        return xt if xt in (_lib.PMX_F32, _lib.PMX_F64) else _lib.PMX_F64
    return _lib.PMX_BOOL if comp.out_type == "bool" else _lib.PMX_I64


@pytest.mark.parametrize("case", MAP_CASES, ids=[c[0] for c in MAP_CASES])
def test_map_cases_compile(case):
    name, _, build, ty, xs = case
    comp = compile_lambda(build(), [ty, "int"])
    xt = CODE[ty]
    _check(comp.program, 0, xt, _out(comp, xt))


@pytest.mark.parametrize("case", MAP2_CASES, ids=[c[0] for c in MAP2_CASES])
def test_map2_cases_compile(case):
    name, _, build, ty, xs, ys = case
    comp = compile_lambda(build(), [ty, ty, "int"])
    xt = CODE[ty]
    _check(comp.program, 1, xt, xt, _out(comp, xt))


def test_f32_storage_and_gather_compile():
    # f32 storage in and out, and a gather from a captured sequence
    comp = compile_lambda(lam("x", addf(mulf("x", "x"), 1.0)), ["float", "int"])
    _check(comp.program, 0, _lib.PMX_F32, _lib.PMX_F32)
    comp = compile_lambda(lam("x", if_(lti("x", 3), divi(10, "x"), muli("x", 2))), ["int", "int"])
    _check(comp.program, 0, _lib.PMX_I32, _lib.PMX_I64)


def test_source_is_lane_parallel_for_straight_line_and_early_exit_for_match():
    lib = _lib.load()
    buf = C.create_string_buffer(1 << 16)
    comp = compile_lambda(lam("x", addf(mulf("x", "x"), 1.0)), ["float", "int"])
    assert lib.pmx_jit_source(C.byref(comp.program), 0, buf, len(buf)) > 0
    src = buf.value.decode()
    assert "static constexpr int U = 8" in src and "run<V>(a, j, o, code)" in src and "__dmul_rn" in src and "goto" not in src
    comp = compile_lambda(lam("x", if_(lti("x", 5), muli("x", 2), divi("x", 0))), ["int", "int"])
    assert lib.pmx_jit_source(C.byref(comp.program), 0, buf, len(buf)) > 0
    src = buf.value.decode()
    assert "static constexpr int U = 1" in src and "goto L" in src and "return;" in src


@pytest.mark.parametrize("code", [_lib.PMX_F32, _lib.PMX_F64, _lib.PMX_I64])
def test_loop_body_compiles(code):
    # loop n (lam i. tensorSet y [i] (2 * tensorGet x [i] + 1)) and a rank-2 variant
    dt = {_lib.PMX_F32: torch.float32, _lib.PMX_F64: torch.float64, _lib.PMX_I64: torch.int64}[code]
    x = DeviceTensor(_Root(torch.zeros(16, dtype=dt), 0, 0, 16, code), 0, (16,), "float")
    y = DeviceTensor(_Root(torch.zeros(16, dtype=dt), 1, 0, 16, code), 0, (4, 4), "float")
    if code == _lib.PMX_I64:
        body = lam("i", tensor_set(x, ["i"], addi(muli(2, tensor_get(x, ["i"])), 1)))
    else:
        body = lam("i", tensor_set(x, ["i"], addf(mulf(2.0, tensor_get(x, ["i"])), 1.0)))
    _check(compile_lambda(body, ["int"]).program, 2, 0, 0)
    body2 = lam("i", tensor_set(y, [divi("i", 4), "i"], tensor_get(x, ["i"])))
    _check(compile_lambda(body2, ["int"]).program, 2, 0, 0)


def test_linear_recursion_loop_compiles():
    """Iterate lowers to a backward jump; the generated kernel keeps it as a
    loop (one element per lane, early exit on the recursion-depth error)."""
    from paper_2211_00621_b200 import lambdas as L
    f = L.Lam(["n"], L.Iterate("m", L.Const(1, "int"), L.Var("n"), "a", L.Const(0.0, "float"),
                               L.Prim("addf", [L.Var("a"), L.Prim("int2float", [L.Var("m")])])))
    comp = compile_lambda(f, ["int", "int"])
    _check(comp.program, 0, _lib.PMX_I64, _lib.PMX_F64)
    lib = _lib.load()
    buf = C.create_string_buffer(1 << 16)
    assert lib.pmx_jit_source(C.byref(comp.program), 0, buf, len(buf)) > 0
    src = buf.value.decode()
    assert "static constexpr int U = 1" in src and "goto L" in src and "PMX_FAILIF(true, 13)" in src

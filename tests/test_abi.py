"""The C-ABI library loads and exports every symbol include/pmx_b200.h declares
(no GPU needed: no compute calls)."""
import ctypes as C
import re

import pytest

from conftest import ROOT
from paper_2211_00621_b200 import _lib, lambdas as L
from paper_2211_00621_b200.lambdas import addf, addi, compile_lambda, gtf, if_, lam, lti, mulf, muli


def _declared():
    text = (ROOT / "include" / "pmx_b200.h").read_text()
    return sorted(set(re.findall(r"PMX_API\s+[\w\s\*]*?\b(pmx_\w+)\s*\(", text)))


def test_header_symbols_exported():
    lib = C.CDLL(str(_lib.LIB_PATH))
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)


def test_abi_version_and_load():
    lib = _lib.load()
    assert lib.pmx_abi_version() == 1


def test_program_struct_layout():
    # 24-byte header, 96 x 8-byte insns, 32 x 8-byte consts, 6 x 56-byte arrays
    assert C.sizeof(_lib.Insn) == 8
    assert C.sizeof(_lib.Array) == 56
    assert C.sizeof(_lib.Program) == 24 + 96 * 8 + 32 * 8 + 6 * 56
    assert _lib.Program.consts.offset == 24 + 96 * 8
    assert _lib.Program.arrays.offset == 24 + 96 * 8 + 32 * 8


@pytest.mark.parametrize("fn,types,role,kind", [
    (lam("x", addf(mulf(2.0, "x"), 1.0)), ["float", "int"], 0, 2),          # affine f
    (lam("x", mulf("x", 0.5)), ["float", "int"], 0, 2),
    (lam("x", addi(muli(3, "x"), 7)), ["int", "int"], 0, 3),               # affine i
    (lam("x", mulf("x", "x")), ["float", "int"], 0, 0),                    # interpreter
    (addf, ["float", "float"], 1, 10),
    (addi, ["int", "int"], 1, 20),
    (muli, ["int", "int"], 1, 21),
    (lam("a", "b", if_(lti("a", "b"), "a", "b")), ["int", "int"], 1, 22),  # min
    (lam("a", "b", if_(gtf("a", "b"), "a", "b")), ["float", "float"], 1, 13),  # max
    (lam("a", "b", addi(addi("a", "b"), 0)), ["int", "int"], 1, 0),
])
def test_fast_path_recognition(fn, types, role, kind):
    c = compile_lambda(fn, types)
    assert _lib.load().pmx_program_kind(C.byref(c.program), role) == kind


def test_last_error_is_reported_for_bad_arguments():
    lib = _lib.load()
    rc = lib.pmx_map(None, None, 0, None, 0, -1, None, None)
    assert rc < 0
    assert b"negative" in lib.pmx_last_error()

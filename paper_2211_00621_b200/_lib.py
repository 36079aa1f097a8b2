"""ctypes binding of the C ABI in include/pmx_b200.h (libpmxb200.so).

The library is the only compute path: if it is missing or fails to load, every
device operation raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = pathlib.Path(os.environ.get("PMX_B200_LIB", _PKG / "libpmxb200.so"))

# ---- constants mirrored from pmx_b200.h --------------------------------------
PMX_F32, PMX_F64, PMX_I64, PMX_I32, PMX_BOOL = 0, 1, 2, 3, 4
PMX_ERR_NONE = 0xFFFFFFFFFFFFFFFF
MAX_INSNS, MAX_CONSTS, MAX_REGS, MAX_ARRAYS, MAX_RANK = 96, 32, 32, 6, 4

OPS = [
    "NOP", "MOV",
    "ADDI", "SUBI", "MULI", "DIVI", "MODI", "NEGI",
    "ADDF", "SUBF", "MULF", "DIVF", "NEGF",
    "EQI", "NEQI", "LTI", "GTI", "LEQI", "GEQI",
    "EQF", "LTF", "GTF", "LEQF", "GEQF",
    "INT2FLOAT", "FLOOR",
    "EXP", "LOG", "SIN", "COS", "SQRT",
    "NOT", "SELECT",
    "GET", "LEN", "TGET", "TSET",
    "NEVER", "EQB", "JZ", "JMP", "FAIL",
]
OP = {name: i for i, name in enumerate(OPS)}

# device error codes -> reference messages (pmx/interp.py:379-436, runtime.py:63-75)
ERROR_MESSAGES = {
    1: "integer division by zero",
    2: "integer modulo by zero",
    3: "float division by zero",
    4: "log: math domain error",
    5: "exp: math range error",
    6: "sqrtf of a negative number",
    7: "get index out of bounds",
    8: "tensor index out of bounds",
    9: "reached a never expression (no pattern matched)",
    10: "value not representable in the f32 storage type",
    11: "math domain error",
    12: "a peer GPU did not deliver its reduce partial (timeout)",
    13: "maximum recursion depth exceeded",
}
MAX_PEERS, IPC_HANDLE_BYTES = 16, 64


class Insn(C.Structure):
    _fields_ = [("op", C.c_uint8), ("dst", C.c_uint8), ("a", C.c_uint8), ("b", C.c_uint8),
                ("c", C.c_uint8), ("pad0", C.c_uint8), ("pad1", C.c_uint8), ("pad2", C.c_uint8)]


class Array(C.Structure):
    _fields_ = [("data", C.c_void_p), ("offset", C.c_int64), ("shape", C.c_int64 * MAX_RANK),
                ("rank", C.c_int32), ("dtype", C.c_int32)]


class Program(C.Structure):
    _fields_ = [("n_insns", C.c_int32), ("n_inputs", C.c_int32), ("out", C.c_int32),
                ("out_is_float", C.c_int32), ("n_arrays", C.c_int32), ("pad", C.c_int32),
                ("insns", Insn * MAX_INSNS), ("consts", C.c_int64 * MAX_CONSTS),
                ("arrays", Array * MAX_ARRAYS)]


class PeerGroup(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("epoch", C.c_uint64),
                ("mbox", C.c_void_p * MAX_PEERS)]


_lib = None
_load_error: str | None = None

_P = C.c_void_p
_SIGS = {
    "pmx_abi_version": (C.c_int, []),
    "pmx_last_error": (C.c_char_p, []),
    "pmx_program_kind": (C.c_int, [C.POINTER(Program), C.c_int32]),
    "pmx_err_reset": (C.c_int, [_P, _P]),
    "pmx_map": (C.c_int, [C.POINTER(Program), _P, C.c_int32, _P, C.c_int32, C.c_int64, _P, _P]),
    "pmx_map2": (C.c_int, [C.POINTER(Program), _P, C.c_int32, _P, C.c_int32, _P, C.c_int32,
                           C.c_int64, _P, _P]),
    "pmx_reduce_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "pmx_map_reduce": (C.c_int, [C.POINTER(Program), C.POINTER(Program), _P, C.c_int32, C.c_int64,
                                 _P, C.c_int32, _P, _P, C.c_int32, _P, C.c_size_t, _P, _P]),
    "pmx_jit_set_mode": (C.c_int, [C.c_int32]),
    "pmx_jit_stats": (C.c_int, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pmx_jit_source": (C.c_int, [C.POINTER(Program), C.c_int32, C.c_char_p, C.c_size_t]),
    "pmx_jit_compile_check": (C.c_int, [C.POINTER(Program), C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "pmx_peer_mailbox_create": (C.c_int, [C.POINTER(C.c_void_p), _P]),
    "pmx_peer_mailbox_destroy": (C.c_int, [_P]),
    "pmx_peer_open": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "pmx_peer_close": (C.c_int, [_P]),
    "pmx_map_reduce_peers": (C.c_int, [C.POINTER(Program), C.POINTER(Program), _P, C.c_int32, C.c_int64,
                                       _P, C.c_int32, _P, _P, C.c_size_t, C.POINTER(PeerGroup), _P, _P]),
    "pmx_fold": (C.c_int, [C.POINTER(Program), _P, C.c_int32, C.c_int64, _P, C.c_int32, _P,
                           _P, C.c_size_t, _P, _P]),
    "pmx_loop": (C.c_int, [C.POINTER(Program), C.c_int64, _P, _P]),
    "pmx_map_rows_fold": (C.c_int, [C.POINTER(Program), C.POINTER(Program), _P, C.c_int32, _P, C.c_int64, _P, _P,
                                    C.c_int32, _P, _P]),
    "pmx_seq_loop": (C.c_int, [C.POINTER(Program), _P, _P, C.c_int64, C.c_int64, _P, _P]),
    "pmx_seq_loop_from": (C.c_int, [C.POINTER(Program), _P, _P, _P, C.c_int64, C.c_int64, _P, _P]),
    "pmx_scan_lengths": (C.c_int, [_P, _P, C.c_int64, _P]),
    "pmx_row_offsets": (C.c_int, [_P, C.c_int64, C.c_int64, _P]),
    "pmx_rk4_sweep_f64": (C.c_int, [_P, C.c_int64, _P, C.c_int32, C.c_double, _P, _P]),
    "pmx_rk4_trace_f64": (C.c_int, [_P, C.c_int64, _P, C.c_int32, C.c_double, C.c_int32, _P, _P, _P]),
    "pmx_hmm_forward_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int64]),
    "pmx_hmm_forward_rerun_count": (C.c_int64, [_P, C.c_int32, C.c_int64, _P]),
    "pmx_viterbi_visited_cells": (C.c_int64, [_P, C.c_int32, C.c_int64, C.c_int32, _P]),
    "pmx_hmm_forward_f32": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, _P, C.c_int64, C.c_int32,
                                      _P, _P, C.c_size_t, _P]),
    "pmx_viterbi_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int64, C.c_int32]),
    "pmx_viterbi_f64": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, _P, C.c_int64, C.c_int32,
                                  _P, _P, _P, C.c_size_t, _P]),
    "pmx_nn_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32, C.c_int32]),
    "pmx_nn_softmax_grad_f64": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P, _P,
                                          C.c_size_t, _P, _P]),
    "pmx_knn_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int64, C.c_int32, C.c_int32]),
    "pmx_knn_f32": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                              _P, _P, _P, C.c_size_t, _P]),
    "pmx_hmm_kmer_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int64]),
    "pmx_hmm_kmer_forward_f32": (C.c_int, [C.c_int32, C.c_float, C.c_float, _P, C.c_int32, _P,
                                           C.c_int64, C.c_int32, _P, _P, C.c_size_t, _P]),
}
EXPORTED = tuple(_SIGS)


def load():
    """Load libpmxb200.so (once). Raises RuntimeError if it is unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"pmx B200 extension not built ({LIB_PATH} missing): run "
            "`python -c 'import __graft_entry__ as g; g.build()'` — there is no CPU fallback")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pmx_abi_version() != 1:
        raise RuntimeError("pmx B200 extension ABI mismatch")
    _lib = lib
    return lib


def jit_stats() -> tuple[int, int]:
    """(kernels compiled, launches) of the run-time specialised path."""
    c, l = C.c_int64(), C.c_int64()
    load().pmx_jit_stats(C.byref(c), C.byref(l))
    return c.value, l.value


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().pmx_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")

"""B200-native backend for the accelerated-expression hot path of the PMExpr
reference runtime (arXiv 2211.00621, reference package `pmx`).

Operator surface (same names and meaning as pmx/interp.py's hot path):
    accelerate / device_call, eval_map, eval_map2, eval_reduce, fold (foldl),
    eval_loop, seq_loop, flatten, marshal_in / marshal_out, merge_intervals,
    Heap, TensorView, Diagnostics
Case studies: rk4_sweep, hmm_forward, viterbi, knn_classify, hmm_kmer_forward, nn_gradients.

All computation runs in libpmxb200.so (hand-written sm_100a CUDA behind a C
ABI, include/pmx_b200.h); PyTorch supplies device memory and streams only.
"""
from . import _lib
from .diagnostics import Diagnostic, Diagnostics, Span, runtime_error
from .lambdas import (
    BUILTINS, Builtin, CompileError, Lam, char, compile_lambda, do, field_, get, if_, lam, length,
    let, match, tensor_get, tensor_set,
)
from .lambdas import (  # builtins as function values (pmx/syntax.py:196-209)
    addi, subi, muli, divi, modi, negi, addf, subf, mulf, divf, negf,
    eqi, neqi, lti, gti, leqi, geqi, eqf, ltf, gtf, leqf, geqf,
    int2float, floor, exp, log, sqrtf, sin, cos,
)
from .runtime import (
    DeviceArena, DeviceRecordSeq, DeviceScalar, DeviceSeq, DeviceTensor, Heap, Interval, TensorView,
    collect_tensors, marshal_in, marshal_out, merge_intervals, merge_overlapping_intervals,
)
from .skeletons import (
    PREV, Ctx, LazyMap, accelerate, device_call, eval_loop, eval_map, eval_map2, eval_reduce, flatten,
    fold, map_rows_fold, seq_loop,
)
from .casestudies import hmm_forward, hmm_kmer_forward, knn_classify, nn_gradients, rk4_sweep, rk4_trace, viterbi

__all__ = [n for n in dir() if not n.startswith("_")]


def load_library():
    """Load the sm_100a library now (raises if it is not built)."""
    return _lib.load()

"""Runtime values, heap, alias-reconstructing marshalling (Alg. 2) for the B200.

Mirrors pmx/runtime.py: tensors are views (buffer id, element offset, shape)
over flat heap buffers, so several tensors may alias one buffer.  Before a
device call the input views of each host buffer are merged into disjoint
intervals (merge_intervals, runtime.py:151-166); one DEVICE root buffer is
allocated per interval, the data copied once, and every input view rebased
into its root (marshal_in, runtime.py:227-259).  Copy-back is one write per
root (marshal_out, runtime.py:262-282) — here only for roots the device wrote
(sequences are immutable, so read-only roots need no copy-back).

B200 layout: host sequences and records are flattened ONCE into contiguous
structure-of-arrays device buffers, staged through pinned host memory:
    [Float]            -> one fp64 buffer (f32 if the host array is float32)
    [Int] / [Bool]     -> int64 / uint8
    [[a]] regular      -> one buffer + shape (n, m)
    [[a]] irregular    -> values buffer + int64 offsets (n + 1)
    [{l: a, ...}]      -> one buffer per field (SoA)
PyTorch provides the device allocations and streams only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

from . import _lib
from .diagnostics import NO_SPAN, Span, runtime_error

try:
    import torch
except Exception:  # pragma: no cover - torch is part of the image
    torch = None

_NP_TO_PMX = {np.dtype(np.float32): _lib.PMX_F32, np.dtype(np.float64): _lib.PMX_F64,
              np.dtype(np.int64): _lib.PMX_I64, np.dtype(np.int32): _lib.PMX_I32,
              np.dtype(np.bool_): _lib.PMX_BOOL, np.dtype(np.uint8): _lib.PMX_BOOL}
_PMX_TO_NP = {_lib.PMX_F32: np.float32, _lib.PMX_F64: np.float64, _lib.PMX_I64: np.int64,
              _lib.PMX_I32: np.int32, _lib.PMX_BOOL: np.uint8}


def _torch_dtype(code: int):
    return {_lib.PMX_F32: torch.float32, _lib.PMX_F64: torch.float64, _lib.PMX_I64: torch.int64,
            _lib.PMX_I32: torch.int32, _lib.PMX_BOOL: torch.uint8}[code]


def pmx_code_of_torch(dt) -> int:
    return {torch.float32: _lib.PMX_F32, torch.float64: _lib.PMX_F64, torch.int64: _lib.PMX_I64,
            torch.int32: _lib.PMX_I32, torch.uint8: _lib.PMX_BOOL, torch.bool: _lib.PMX_BOOL}[dt]


# ------------------------------------------------------------------ host side

class Heap:
    """Flat buffers addressed by id, shared by host values (pmx/runtime.py:30-41)."""

    def __init__(self) -> None:
        self.buffers: dict[int, np.ndarray] = {}
        self._next = 0

    def alloc(self, data) -> int:
        bid = self._next
        self._next += 1
        self.buffers[bid] = np.asarray(data)
        return bid


@dataclass(frozen=True)
class TensorView:
    """View into a heap buffer (pmx/runtime.py:44-75)."""
    buffer: int
    offset: int
    shape: tuple
    elem: str  # "int" | "float"

    @property
    def size(self) -> int:
        return math.prod(self.shape)

    def strides(self) -> tuple:
        out, acc = [], 1
        for d in reversed(self.shape):
            out.append(acc)
            acc *= d
        return tuple(reversed(out))

    def linear(self, idx, span: Span = NO_SPAN) -> int:
        if len(idx) != len(self.shape):
            raise runtime_error(f"tensor index of rank {len(idx)} against rank {len(self.shape)} tensor", span)
        pos = self.offset
        for i, (k, d, s) in enumerate(zip(idx, self.shape, self.strides())):
            if not 0 <= k < d:
                raise runtime_error(f"tensor index {k} out of bounds for dimension {i} of size {d}", span)
            pos += k * s
        return pos


@dataclass(frozen=True)
class Interval:
    start: int
    end: int  # exclusive


def merge_intervals(pairs) -> list[Interval]:
    """Merge overlapping and touching half-open intervals (pmx/runtime.py:151-166):
    sort by (start, end); extend the last merged interval while the next one
    starts at or before its end."""
    assert pairs
    merged: list[list[int]] = []
    for s, e in sorted(pairs):
        if merged and merged[-1][1] >= s:
            merged[-1][1] = max(merged[-1][1], e)
        else:
            merged.append([s, e])
    return [Interval(s, e) for s, e in merged]


def merge_overlapping_intervals(views) -> list[Interval]:
    """Alias-merge the views of ONE buffer (pmx/runtime.py:169-175); empty views
    occupy one cell, as in the reference."""
    assert views
    assert len({v.buffer for v in views}) == 1, "views over distinct buffers must be partitioned first"
    return merge_intervals([(v.offset, v.offset + max(v.size, 1)) for v in views])


def collect_tensors(value) -> list:
    out: list = []

    def go(v):
        if isinstance(v, TensorView):
            out.append(v)
        elif isinstance(v, (list, tuple)):
            for x in v:
                go(x)
        elif isinstance(v, dict):
            for x in v.values():
                go(x)

    go(value)
    return out


# ---------------------------------------------------------------- device side

class DeviceValue:
    pass


class DeviceSeq(DeviceValue):
    """A device sequence: flat values + shape (regular nesting) or offsets.

    `data` is a 1-D torch tensor holding the flattened values in row-major
    order; `shape` is (n,) for [a], (n, m) for a regular [[a]], ...  For an
    irregular [[a]], `offsets` (int64, n+1) delimits the rows and shape is (n,).
    """

    def __init__(self, data, shape: tuple, dtype_code: int, offsets=None, elem_tag: str = ""):
        self.data = data
        self.shape = tuple(shape)
        self.dtype_code = dtype_code
        self.offsets = offsets
        self.elem_tag = elem_tag or _lib_elem(dtype_code)

    def __len__(self) -> int:
        return self.shape[0]

    @property
    def rank(self) -> int:
        return len(self.shape)

    @property
    def numel(self) -> int:
        return self.data.numel()

    def as_pmx_array(self, write: bool = True) -> _lib.Array:
        a = _lib.Array()
        a.data = self.data.data_ptr()
        a.offset = 0
        a.shape[0] = self.data.numel() if self.rank == 1 and self.offsets is None else self.shape[0]
        a.rank = 1
        a.dtype = self.dtype_code
        return a

    def ptr(self) -> int:
        return self.data.data_ptr()

    def __repr__(self) -> str:
        return f"DeviceSeq(shape={self.shape}, dtype={_PMX_TO_NP[self.dtype_code].__name__})"


class DeviceRecordSeq(DeviceValue):
    """[{l: a}] as structure of arrays: one DeviceSeq per field."""

    def __init__(self, fields: dict):
        self.fields = fields
        n = {len(v) for v in fields.values()}
        assert len(n) <= 1
        self.n = n.pop() if n else 0

    def __len__(self) -> int:
        return self.n

    def __getitem__(self, label: str) -> DeviceSeq:
        return self.fields[label]


@dataclass
class DeviceTensor(DeviceValue):
    """A tensor view rebased into a device root buffer (Alg. 2)."""
    root: Any          # _Root
    offset: int
    shape: tuple
    elem: str

    @property
    def dtype_code(self) -> int:
        return self.root.dtype_code

    @property
    def size(self) -> int:
        return math.prod(self.shape)

    def as_pmx_array(self, write: bool = True) -> _lib.Array:
        if len(self.shape) > _lib.MAX_RANK:
            raise runtime_error(f"tensor rank {len(self.shape)} exceeds the device bound {_lib.MAX_RANK}")
        a = _lib.Array()
        a.data = self.root.data.data_ptr()
        a.offset = self.offset
        for i, d in enumerate(self.shape):
            a.shape[i] = d
        a.rank = len(self.shape)
        a.dtype = self.root.dtype_code
        if write:                   # only a root some kernel stores into is copied back
            self.root.dirty = True
        return a


def _lib_elem(code: int) -> str:
    return "float" if code in (_lib.PMX_F32, _lib.PMX_F64) else ("bool" if code == _lib.PMX_BOOL else "int")


@dataclass
class _Root:
    data: Any                 # torch device tensor (1-D)
    host_buffer: int
    start: int
    end: int
    dtype_code: int
    dirty: bool = False


@dataclass
class DeviceArena:
    roots: list = field(default_factory=list)
    by_host: dict = field(default_factory=dict)
    h2d_bytes: int = 0
    d2h_bytes: int = 0

    def root_for(self, v: TensorView) -> _Root:
        for r in self.by_host[v.buffer]:
            if r.start <= v.offset and v.offset + max(v.size, 1) <= r.end:
                return r
        raise AssertionError("input tensor not covered by any root interval")


def _device():
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 backend has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(arr, arena: Optional[DeviceArena] = None):
    """H2D copy of a contiguous host array through pinned memory.

    A pinned torch CPU tensor is copied directly (async); numpy arrays are
    first staged into a pinned buffer (the caching host allocator keeps the
    staging buffer alive until the async copy has completed)."""
    if torch is not None and isinstance(arr, torch.Tensor):
        t = arr.reshape(-1)
        nbytes = t.numel() * t.element_size()
        if not t.is_pinned():
            t = t.pin_memory()
    else:
        arr = np.ascontiguousarray(arr)
        if arr.dtype == np.bool_:
            arr = arr.astype(np.uint8)
        nbytes = arr.nbytes
        t = torch.from_numpy(arr.reshape(-1))
        if t.numel():
            pinned = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            pinned.copy_(t)
            t = pinned
    dev = torch.empty(t.shape, dtype=t.dtype, device=_device())
    if t.numel():
        dev.copy_(t, non_blocking=True)
    if arena is not None:
        arena.h2d_bytes += nbytes
    return dev


def lengths_to_offsets(lens, arena: Optional[DeviceArena] = None):
    """Row offsets of an irregular sequence, built on the device: the row
    lengths are copied up and pmx_scan_lengths writes the n+1 offsets
    (flatten is then the values buffer itself, pmx/interp.py:161-166)."""
    d_lens = to_device(np.asarray(lens, np.int64), arena)
    offs = torch.empty(len(lens) + 1, dtype=torch.int64, device=_device())
    _lib.check(_lib.load().pmx_scan_lengths(d_lens.data_ptr(), offs.data_ptr(), len(lens),
                                            torch.cuda.current_stream().cuda_stream), "scan lengths")
    return offs


def _is_char_list(v) -> bool:
    return isinstance(v, list) and v and all(isinstance(c, str) and len(c) == 1 for c in v)


def seq_to_device(v, arena: Optional[DeviceArena] = None) -> DeviceValue:
    """Flatten a host sequence into SoA device buffers (see module docstring)."""
    if isinstance(v, np.ndarray):
        code = _NP_TO_PMX.get(v.dtype)
        if code is None:
            raise runtime_error(f"cannot marshal array of dtype {v.dtype}")
        return DeviceSeq(to_device(v, arena), v.shape, code)
    if torch is not None and isinstance(v, torch.Tensor):
        t = v.contiguous().reshape(-1) if v.is_cuda else to_device(v.contiguous(), arena)
        return DeviceSeq(t, tuple(v.shape), pmx_code_of_torch(v.dtype))
    assert isinstance(v, list)
    if not v:
        return DeviceSeq(to_device(np.zeros(0, np.float64), arena), (0,), _lib.PMX_F64)
    if _is_char_list(v):
        return DeviceSeq(to_device(np.array([ord(c) for c in v], np.int64), arena), (len(v),),
                         _lib.PMX_I64, elem_tag="char")
    x0 = v[0]
    if isinstance(x0, dict):
        labels = list(x0.keys())
        return DeviceRecordSeq({l: seq_to_device([r[l] for r in v], arena) for l in labels})
    if isinstance(x0, list):
        lens = [len(r) for r in v]
        if len(set(lens)) == 1 and (not x0 or not isinstance(x0[0], (list, dict))):
            arr = np.array(v)
            inner = seq_to_device(arr if arr.dtype != object else v, arena)
            return inner
        flat = [x for r in v for x in r]
        inner = seq_to_device(flat, arena) if flat else DeviceSeq(to_device(np.zeros(0, np.int64), arena), (0,), _lib.PMX_I64)
        return DeviceSeq(inner.data, (len(v),), inner.dtype_code, offsets=lengths_to_offsets(lens, arena),
                         elem_tag=inner.elem_tag)
    if isinstance(x0, bool):
        return DeviceSeq(to_device(np.array(v, np.uint8), arena), (len(v),), _lib.PMX_BOOL)
    if isinstance(x0, int):
        return DeviceSeq(to_device(np.array(v, np.int64), arena), (len(v),), _lib.PMX_I64)
    if isinstance(x0, float):
        return DeviceSeq(to_device(np.array(v, np.float64), arena), (len(v),), _lib.PMX_F64)
    raise runtime_error(f"cannot marshal a sequence of {type(x0).__name__}")


def marshal_in(args: list, heap: Heap, device_views: bool = True):
    """Copy arguments to the device, reconstructing tensor aliases (Alg. 2,
    pmx/runtime.py:227-259).  Returns (device args, arena)."""
    arena = DeviceArena()
    by_buffer: dict[int, list] = {}
    for t in collect_tensors(args):
        by_buffer.setdefault(t.buffer, []).append(t)
    for hb in sorted(by_buffer):
        for iv in merge_overlapping_intervals(by_buffer[hb]):
            host = heap.buffers[hb][iv.start:iv.end]
            code = _NP_TO_PMX[np.asarray(host).dtype]
            root = _Root(to_device(np.asarray(host), arena), hb, iv.start, iv.end, code)
            arena.roots.append(root)
            arena.by_host.setdefault(hb, []).append(root)

    def copy_in(v):
        if isinstance(v, TensorView):
            r = arena.root_for(v)
            return DeviceTensor(r, v.offset - r.start, v.shape, v.elem)
        if isinstance(v, (list, np.ndarray)) or (torch is not None and isinstance(v, torch.Tensor)):
            if isinstance(v, list) and any(isinstance(x, TensorView) for x in v):
                return [copy_in(x) for x in v]
            return seq_to_device(v, arena)
        if isinstance(v, dict):
            return {l: copy_in(x) for l, x in v.items()}
        if callable(v) and not isinstance(v, (int, float, bool, str)):
            raise AssertionError("cannot marshal a function value")
        return v

    return [copy_in(v) for v in args], arena


def seq_to_host(v: DeviceSeq, arena: Optional[DeviceArena] = None):
    """Device sequence -> numpy array (regular) or list of arrays (irregular)."""
    host = v.data.detach().to("cpu").numpy()
    if arena is not None:
        arena.d2h_bytes += host.nbytes
    if v.offsets is not None:
        offs = v.offsets.to("cpu").numpy()
        return [host[offs[i]:offs[i + 1]] for i in range(len(offs) - 1)]
    return host.reshape(v.shape)


def marshal_out(arena: DeviceArena, heap: Heap, result):
    """Copy every written root back once, convert the result to host values
    (pmx/runtime.py:262-282).  Device sequences come back as numpy arrays."""
    for r in arena.roots:
        if r.dirty:
            host = r.data.to("cpu").numpy()
            arena.d2h_bytes += host.nbytes
            heap.buffers[r.host_buffer][r.start:r.end] = host

    def copy_out(v):
        if isinstance(v, DeviceTensor):
            return TensorView(v.root.host_buffer, v.root.start + v.offset, v.shape, v.elem)
        if isinstance(v, DeviceSeq):
            return seq_to_host(v, arena)
        if isinstance(v, DeviceRecordSeq):
            cols = {l: seq_to_host(s, arena) for l, s in v.fields.items()}
            return [{l: cols[l][i].item() if hasattr(cols[l][i], "item") else cols[l][i] for l in cols}
                    for i in range(len(v))]
        if hasattr(v, "materialize"):
            return copy_out(v.materialize())
        if isinstance(v, DeviceScalar):
            return v.get(arena)
        if isinstance(v, list):
            return [copy_out(x) for x in v]
        if isinstance(v, tuple):
            return tuple(copy_out(x) for x in v)
        if isinstance(v, dict):
            return {l: copy_out(x) for l, x in v.items()}
        return v

    return copy_out(result)


class DeviceScalar(DeviceValue):
    """A scalar result left on the device (e.g. a reduction) until read."""

    def __init__(self, buf, is_float: bool, err=None, span: Span = NO_SPAN, what="element"):
        self.buf = buf          # torch 8-byte buffer (float64 or int64)
        self.is_float = is_float
        self.err = err
        self.span = span
        self.what = what

    def get(self, arena: Optional[DeviceArena] = None):
        from .skeletons import raise_if_error
        raise_if_error(self.err, self.span, self.what)
        v = self.buf.to("cpu")
        if arena is not None:
            arena.d2h_bytes += 8
        return float(v.item()) if self.is_float else int(v.item())

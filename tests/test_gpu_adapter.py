"""Replay, on the B200, every parallel construct of the reference's corpus as
translated by the whole-program adapter (tests/golden/make_golden.py records the
adapter's lambda IR for each construct together with its inputs and the
reference's own result; tests/test_adapter.py checks the translation itself on
CPU).  Results must match the reference: integers exactly, floats within the
corpus tolerance (tests/corpus.py)."""
import math

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2211_00621_b200 import _lib, ir_json
from paper_2211_00621_b200.runtime import DeviceSeq, DeviceTensor, _Root, seq_to_device, seq_to_host, to_device
from paper_2211_00621_b200.skeletons import (
    Ctx, _ctx_stack, _materialize, eval_loop, eval_map, eval_map2, eval_reduce, map_rows_fold,
)

pytestmark = pytest.mark.gpu

RECORDS = [(name, i, c, entry["float_rel"]) for name, entry in sorted(GOLDEN.get("adapter", {}).items())
           for i, c in enumerate(entry["constructs"])]


def _make_array(h: ir_json.HostArray):
    if h.is_tensor:
        is_f = h.elem == "float"
        data = to_device(np.array(h.data, dtype=np.float64 if is_f else np.int64))
        root = _Root(data, -1, 0, len(h.data), _lib.PMX_F64 if is_f else _lib.PMX_I64)
        return DeviceTensor(root, h.offset, tuple(h.shape), h.elem)
    return seq_to_device(list(h.data))


def _seq(xs, elem):
    s = seq_to_device(list(xs))
    if elem == "char":
        s.elem_tag = "char"
    return s


def _close(a, b, rel):
    if isinstance(b, float) or isinstance(a, float):
        return math.isclose(float(a), float(b), rel_tol=rel, abs_tol=rel)
    return int(a) == int(b)


@pytest.mark.parametrize("rec", RECORDS, ids=[f"{n}-{i}-{c['kind']}" for n, i, c, _ in RECORDS])
def test_adapter_construct_on_device(rec):
    name, _, c, rel = rec
    rel = rel or 1e-12
    lam, arrays = ir_json.load(c["lam"], _make_array) if "lam" in c else (None, [])
    ctx = Ctx()
    ctx.device = True
    _ctx_stack.append(ctx)
    try:
        kind = c["kind"]
        if kind == "map":
            out = seq_to_host(_materialize(eval_map(lam, _seq(c["xs"], c["x_elem"])))).tolist()
            assert len(out) == len(c["expected"])
            assert all(_close(a, b, rel) for a, b in zip(out, c["expected"])), (out, c["expected"])
        elif kind == "map2":
            out = seq_to_host(eval_map2(lam, _seq(c["xs"], c["x_elem"]), _seq(c["ys"], c["y_elem"]))).tolist()
            assert all(_close(a, b, rel) for a, b in zip(out, c["expected"])), (out, c["expected"])
        elif kind == "reduce":
            got = eval_reduce(lam, c["acc"], _seq(c["xs"], c["x_elem"])).get()
            assert _close(got, c["expected"], rel), (got, c["expected"])
        elif kind == "map_rows":          # row function over [[a]] (nested_map, foldl_in_accel)
            g = ir_json.load(c["g"], _make_array)[0] if c["g"] is not None else None
            op = ir_json.load(c["op"], _make_array)[0]
            out = seq_to_host(map_rows_fold(g, op, c["acc"], seq_to_device(c["rows"]))).tolist()
            assert all(_close(a, b, rel) for a, b in zip(out, c["expected"])), (out, c["expected"])
        elif kind == "loop":
            eval_loop(c["n"], lam)
            tensors = [a for a in arrays if isinstance(a, DeviceTensor)]
            for t, want in zip(tensors, c["tensors_after"]):
                got = t.root.data.to("cpu").numpy().tolist()
                assert all(_close(a, b, rel) for a, b in zip(got, want)), (got, want)
        ctx.check_errors()
    finally:
        _ctx_stack.pop()


def test_adapter_records_present():
    assert len(RECORDS) >= 35
    assert {c["kind"] for _, _, c, _ in RECORDS} >= {"map", "map2", "reduce", "loop", "map_rows"}

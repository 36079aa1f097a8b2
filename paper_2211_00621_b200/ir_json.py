"""JSON form of the lambda IR (plus the host data of captured sequences and
tensors), so a translated reference closure can be stored and replayed on
another machine — used by the golden fixtures of the pmx adapter
(tests/golden/make_golden.py -> tests/test_gpu_adapter.py)."""
from __future__ import annotations

from . import lambdas as L


class HostArray:
    """Captured host data: a sequence (rank 1) or a tensor view of a buffer."""

    def __init__(self, data: list, elem: str, shape=None, offset: int = 0):
        self.data = list(data)
        self.elem = elem                    # "int" | "float" | "bool" | "char"
        self.shape = tuple(shape) if shape is not None else (len(self.data),)
        self.offset = offset
        self.is_tensor = shape is not None


def dump(lam: L.Lam) -> dict:
    arrays: list = []
    ids: dict = {}

    def arr(a) -> int:
        if id(a) not in ids:
            ids[id(a)] = len(arrays)
            arrays.append({"data": a.data, "elem": a.elem, "shape": list(a.shape), "offset": a.offset,
                           "tensor": a.is_tensor})
        return ids[id(a)]

    def go(e):
        if isinstance(e, L.Var):
            return ["Var", e.name]
        if isinstance(e, L.Const):
            return ["Const", e.value, e.ty]
        if isinstance(e, L.Prim):
            return ["Prim", e.name, [go(a) for a in e.args]]
        if isinstance(e, L.If):
            return ["If", go(e.cond), go(e.then), go(e.els)]
        if isinstance(e, L.LetE):
            return ["Let", e.name, go(e.value), go(e.body)]
        if isinstance(e, L.Get):
            return ["Get", arr(e.arr), go(e.index)]
        if isinstance(e, L.Len):
            return ["Len", arr(e.arr)]
        if isinstance(e, L.TGet):
            return ["TGet", arr(e.tensor), [go(i) for i in e.index]]
        if isinstance(e, L.TSet):
            return ["TSet", arr(e.tensor), [go(i) for i in e.index], go(e.value)]
        if isinstance(e, L.Do):
            return ["Do", [go(x) for x in e.exprs]]
        if isinstance(e, L.Never):
            return ["Never"]
        if isinstance(e, L.Field):
            return ["Field", go(e.rec), e.label]
        if isinstance(e, L.Iterate):
            return ["Iterate", e.var, go(e.lo), go(e.hi), e.acc, go(e.init), go(e.body),
                    [[n, go(x)] for n, x in e.more]]
        raise TypeError(type(e).__name__)

    return {"params": lam.params, "body": go(lam.body), "arrays": arrays}


def load(d: dict, make_array) -> L.Lam:
    """`make_array(HostArray)` returns the object to store in Get/TGet/TSet
    nodes (a device array on the B200)."""
    arrays = [make_array(HostArray(a["data"], a["elem"], a["shape"] if a["tensor"] else None, a["offset"]))
              for a in d["arrays"]]

    def go(x):
        k = x[0]
        if k == "Var":
            return L.Var(x[1])
        if k == "Const":
            return L.Const(x[1], x[2])
        if k == "Prim":
            return L.Prim(x[1], [go(a) for a in x[2]])
        if k == "If":
            return L.If(go(x[1]), go(x[2]), go(x[3]))
        if k == "Let":
            return L.LetE(x[1], go(x[2]), go(x[3]))
        if k == "Get":
            return L.Get(arrays[x[1]], go(x[2]))
        if k == "Len":
            return L.Len(arrays[x[1]])
        if k == "TGet":
            return L.TGet(arrays[x[1]], [go(i) for i in x[2]])
        if k == "TSet":
            return L.TSet(arrays[x[1]], [go(i) for i in x[2]], go(x[3]))
        if k == "Do":
            return L.Do([go(a) for a in x[1]])
        if k == "Never":
            return L.Never()
        if k == "Field":
            return L.Field(go(x[1]), x[2])
        if k == "Iterate":
            more = tuple((n, go(v)) for n, v in x[7]) if len(x) > 7 else ()
            return L.Iterate(x[1], go(x[2]), go(x[3]), x[4], go(x[5]), go(x[6]), more)
        raise ValueError(k)

    return L.Lam(d["params"], go(d["body"])), arrays

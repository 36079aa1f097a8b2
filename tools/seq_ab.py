"""A/B the seqLoop entry points on the bench stencil (2^24 fp64 states, 20
steps): pmx_seq_loop on a copied state vs pmx_seq_loop_from reading the
caller's state in step 0.  Median ms of 20 calls each, interleaved."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_00621_b200 as P  # noqa: E402
from paper_2211_00621_b200 import _lib  # noqa: E402
from paper_2211_00621_b200.runtime import DeviceSeq  # noqa: E402
from paper_2211_00621_b200.skeletons import _compile, default_ctx  # noqa: E402

m, steps = 1 << 24, int(sys.argv[1]) if len(sys.argv) > 1 else 20
s = torch.arange(m, dtype=torch.float64, device="cuda") % 97
stencil = P.lam("x", "j", "t", P.mulf(0.5, P.addf("x", P.get(P.PREV, P.modi(P.addi("j", 1), m)))))
prog = _compile(stencil, ["float", "int", "int"], None, state_array=P.PREV)
ctx = default_ctx()
err = ctx.new_err(None)
lib = _lib.load()
a = torch.empty(m, dtype=torch.float64, device="cuda")
b = torch.empty(m + 8, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def old():
    a.copy_(s)
    _lib.check(lib.pmx_seq_loop(C.byref(prog.program), a.data_ptr(), b.data_ptr(), m, steps, err.data_ptr(), st), "sl")


def new():
    _lib.check(lib.pmx_seq_loop_from(C.byref(prog.program), s.data_ptr(), a.data_ptr(), b.data_ptr(), m, steps,
                                     err.data_ptr(), st), "slf")


def api():
    P.seq_loop(steps, stencil, DeviceSeq(s, (m,), _lib.PMX_F64))


res = {"old": [], "new": [], "api": []}
for _ in range(30):
    for k, fn in (("old", old), ("new", new), ("api", api)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        res[k].append(e0.elapsed_time(e1))
for k, v in res.items():
    v = sorted(v[5:])
    print(k, "steps", steps, "median ms", round(v[len(v) // 2], 4), "min", round(v[0], 4))

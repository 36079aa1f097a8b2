"""Throughput of the skeleton kernels on lambdas the library does not
recognise (interpreter / JIT path) at the microbench size, 2^28 fp32:

    map     y = x*x + 1         (8 B/elem)
    map2    z = x*y - x         (12 B/elem)
    reduce  sum (map (x*x) s)   (4 B/elem)
    loop    tensorSet y [i] (2 * tensorGet x [i] + 1)   (8 B/elem)

Prints one JSON line per case: ms, GB/s, fraction of the measured HBM peak.
"""
from __future__ import annotations

import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2211_00621_b200 as P  # noqa: E402
from paper_2211_00621_b200 import _lib, synth  # noqa: E402
from paper_2211_00621_b200.runtime import DeviceSeq, DeviceTensor, _Root  # noqa: E402
from paper_2211_00621_b200.skeletons import default_ctx  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
    P.load_library()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6544.0) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6544.0
    dev = torch.device("cuda", 0)
    x = synth.mapreduce_x_device(n, dev)
    yv = torch.roll(x, 1)
    xs = DeviceSeq(x, (n,), _lib.PMX_F32)
    ys = DeviceSeq(yv, (n,), _lib.PMX_F32)
    ctx = default_ctx()
    out = []

    def rep(name, ms, bytes_per_elem):
        gbs = bytes_per_elem * n / (ms * 1e-3) / 1e9
        out.append({"case": name, "ms": round(ms, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 3)})
        print(json.dumps(out[-1]), flush=True)

    f = P.lam("x", P.addf(P.mulf("x", "x"), 1.0))
    rep("map x*x+1", timeit(lambda: P.eval_map(f, xs).materialize()), 8)
    g = P.lam("a", "b", P.subf(P.mulf("a", "b"), "a"))
    rep("map2 a*b-a", timeit(lambda: P.eval_map2(g, xs, ys)), 12)
    sq = P.lam("x", P.mulf("x", "x"))
    rep("reduce addf (map x*x)", timeit(lambda: P.eval_reduce(P.addf, 0.0, P.eval_map(sq, xs))), 4)
    yt = torch.empty_like(x)
    rx = _Root(x, 0, 0, n, _lib.PMX_F32)
    ry = _Root(yt, 1, 0, n, _lib.PMX_F32)
    tx = DeviceTensor(rx, 0, (n,), "float")
    ty = DeviceTensor(ry, 0, (n,), "float")
    body = P.lam("i", P.tensor_set(ty, ["i"], P.addf(P.mulf(2.0, P.tensor_get(tx, ["i"])), 1.0)))
    rep("loop y[i] = 2x[i]+1", timeit(lambda: P.eval_loop(n, body)), 8)
    gop = P.lam("a", "b", P.addf("a", P.mulf("b", 1.0)))
    rep("reduce generic op (ordered tree)", timeit(lambda: P.eval_reduce(gop, 0.0, xs)), 4)
    ms_, st_ = 1 << 24, 20
    s_state = DeviceSeq(torch.arange(ms_, dtype=torch.float64, device=dev) % 97, (ms_,), _lib.PMX_F64)
    stencil = P.lam("x", "j", "t", P.mulf(0.5, P.addf("x", P.get(P.PREV, P.modi(P.addi("j", 1), ms_)))))
    t_ms = timeit(lambda: P.seq_loop(st_, stencil, s_state), reps=3, warm=1)
    gbs = 16.0 * ms_ * st_ / (t_ms * 1e-3) / 1e9
    print(json.dumps({"case": "seq_loop 20 steps m=2^24 f64", "ms": round(t_ms, 3), "GB/s": round(gbs, 1),
                      "frac": round(gbs / peak, 3)}), flush=True)
    ctx.check_errors()
    torch.cuda.synchronize()
    ref = x.double() * 2 + 1
    assert torch.equal(yt.double(), ref.float().double()), "loop result mismatch"


if __name__ == "__main__":
    main()

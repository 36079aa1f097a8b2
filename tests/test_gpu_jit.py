"""Run-time specialised skeleton kernels (csrc/jit.cu) at sizes above the
JIT threshold, through the C ABI: bit-exact against a numpy restatement of the
reference's fp64 / int64 semantics, on aligned and misaligned views, with the
reference's first-failing-element error reporting."""
import numpy as np
import pytest
import torch

import paper_2211_00621_b200 as P
from paper_2211_00621_b200 import _lib
from paper_2211_00621_b200.runtime import DeviceSeq, DeviceTensor, _Root
from paper_2211_00621_b200.skeletons import default_ctx

pytestmark = pytest.mark.gpu

N = (1 << 18) + 3          # above the auto threshold, ragged tail


@pytest.fixture(autouse=True)
def auto_mode():
    lib = _lib.load()
    prev = lib.pmx_jit_set_mode(2)
    yield
    lib.pmx_jit_set_mode(prev)


def _launched():
    return _lib.jit_stats()[1]


def _f32(n, seed=0):
    return np.random.default_rng(seed).standard_normal(n).astype(np.float32)


def test_map_f32_storage_is_fp64_then_rounded():
    x = _f32(N)
    f = P.lam("x", P.addf(P.mulf("x", "x"), P.mulf(0.1, "x")))
    before = _launched()
    got = P.accelerate(lambda s: P.eval_map(f, s), torch.from_numpy(x))
    assert _launched() > before
    xd = x.astype(np.float64)
    want = (xd * xd + 0.1 * xd).astype(np.float32)       # fp64 ops, one rounding to f32 storage
    assert np.array_equal(np.asarray(got, dtype=np.float32).view(np.uint32), want.view(np.uint32))


def test_map_misaligned_view_uses_scalar_kernel():
    x = torch.from_numpy(_f32(N + 1, 1)).cuda()
    xs = DeviceSeq(x[1:], (N,), _lib.PMX_F32)
    f = P.lam("x", P.subf(P.mulf(3.0, "x"), "x"))
    y = P.eval_map(f, xs).materialize().data.cpu().numpy()
    xd = x[1:].cpu().numpy().astype(np.float64)
    assert np.array_equal(y, (3.0 * xd - xd).astype(np.float32))


def test_map2_int_and_float():
    a = np.arange(N, dtype=np.int64) * 7919 - 12345
    b = (np.arange(N, dtype=np.int64) % 13) - 6
    g = P.lam("a", "b", P.addi(P.muli("a", "b"), P.modi("a", 5)))
    got = np.asarray(P.accelerate(lambda s, t: P.eval_map2(g, s, t), a, b))
    want = a * b + np.fmod(a, 5)                          # modi truncates toward zero
    assert np.array_equal(got, want)
    xf, yf = _f32(N, 2), _f32(N, 3)
    h = P.lam("a", "b", P.subf(P.mulf("a", "b"), "a"))
    got = P.accelerate(lambda s, t: P.eval_map2(h, s, t), torch.from_numpy(xf), torch.from_numpy(yf))
    xd, yd = xf.astype(np.float64), yf.astype(np.float64)
    assert np.array_equal(np.asarray(got, dtype=np.float32), (xd * yd - xd).astype(np.float32))


def test_map_reduce_generic_map_recognised_sum():
    x = _f32(N, 4)
    sq = P.lam("x", P.mulf("x", "x"))
    before = _launched()
    got = P.accelerate(lambda s: P.eval_reduce(P.addf, 0.0, P.eval_map(sq, s)), torch.from_numpy(x))
    assert _launched() > before
    xd = x.astype(np.float64)
    want = float(np.sum(xd * xd))
    assert abs(got - want) <= 1e-12 * abs(want)
    # int: wrap-around product is exact in any order
    xi = (np.arange(N, dtype=np.int64) % 7) + 1
    got = P.accelerate(lambda s: P.eval_reduce(P.muli, 1, P.eval_map(P.lam("x", P.addi("x", 0)), s)), xi)
    want = 1
    for v in xi.tolist():
        want = (want * v) & 0xFFFFFFFFFFFFFFFF
    assert got == (want - (1 << 64) if want >= 1 << 63 else want)


def test_loop_tensor_map_matches():
    n = N
    dev = torch.device("cuda", 0)
    x = torch.from_numpy(_f32(n, 5)).to(dev)
    y = torch.empty_like(x)
    tx = DeviceTensor(_Root(x, 0, 0, n, _lib.PMX_F32), 0, (n,), "float")
    ty = DeviceTensor(_Root(y, 1, 0, n, _lib.PMX_F32), 0, (n,), "float")
    body = P.lam("i", P.tensor_set(ty, ["i"], P.addf(P.mulf(2.0, P.tensor_get(tx, ["i"])), 1.0)))
    before = _launched()
    P.eval_loop(n, body)
    default_ctx().check_errors()
    assert _launched() > before
    xd = x.cpu().numpy().astype(np.float64)
    assert np.array_equal(y.cpu().numpy(), (2.0 * xd + 1.0).astype(np.float32))


def test_loop_rank2_and_out_of_bounds_first_index():
    n, m = 512, 600
    dev = torch.device("cuda", 0)
    y = torch.zeros(n * m, dtype=torch.int64, device=dev)
    ty = DeviceTensor(_Root(y, 0, 0, n * m, _lib.PMX_I64), 0, (n, m), "int")
    body = P.lam("i", P.tensor_set(ty, [P.divi("i", m), P.modi("i", m)], P.muli("i", 3)))
    P.eval_loop(n * m, body)
    default_ctx().check_errors()
    assert np.array_equal(y.cpu().numpy(), np.arange(n * m, dtype=np.int64) * 3)
    # iteration i writes row i // 500: rows >= 512 fail; the first failing iteration is 256000
    body = P.lam("i", P.tensor_set(ty, [P.divi("i", 500), P.modi("i", 500)], 1))
    with pytest.raises(P.Diagnostics, match="out of bounds") as ei:
        P.accelerate(lambda: P.eval_loop(n * m, body))
    assert "iteration 256000)" in str(ei.value)


def test_first_failing_element_reported():
    x = np.arange(N, dtype=np.int64) + 1
    x[200_001] = 0
    x[250_000] = 0
    f = P.lam("x", P.divi(10, "x"))
    with pytest.raises(P.Diagnostics, match="integer division by zero") as ei:
        P.accelerate(lambda s: P.eval_map(f, s), x)
    assert "element 200001)" in str(ei.value)


def test_f32_range_error():
    x = np.ones(N, np.float32)
    x[77_777] = 3.0e38
    f = P.lam("x", P.mulf("x", 10.0))
    with pytest.raises(P.Diagnostics, match="f32"):
        P.accelerate(lambda s: P.eval_map(f, s), torch.from_numpy(x))


def test_gather_from_captured_sequence():
    data = (np.arange(N, dtype=np.int64) * 31) % 1000
    idx = (np.arange(N, dtype=np.int64) * 7) % N
    got = P.accelerate(lambda d, s: P.eval_map(P.lam("i", P.addi(P.get(d, "i"), 1)), s), data, idx)
    assert np.array_equal(np.asarray(got), data[idx] + 1)
    bad = idx.copy()
    bad[123_456] = N
    with pytest.raises(P.Diagnostics, match="out of bounds") as ei:
        P.accelerate(lambda d, s: P.eval_map(P.lam("i", P.get(d, "i")), s), data, bad)
    assert "element 123456)" in str(ei.value)


def _tensor(t, bid):
    return DeviceTensor(_Root(t, bid, 0, t.numel(), {torch.float32: _lib.PMX_F32, torch.float64: _lib.PMX_F64,
                                                      torch.int64: _lib.PMX_I64}[t.dtype]), 0, (t.numel(),), "float")


def test_elementwise_loop_inplace_and_types():
    # vectorised elementwise loop: in-place update, f64 and i64 views, ragged n
    n = N
    dev = torch.device("cuda", 0)
    y = torch.arange(n, dtype=torch.float64, device=dev) * 0.5
    ty = _tensor(y, 0)
    before = _launched()
    P.eval_loop(n, P.lam("i", P.tensor_set(ty, ["i"], P.subf(P.mulf(P.tensor_get(ty, ["i"]), 3.0), 1.0))))
    default_ctx().check_errors()
    assert _launched() > before
    ref = np.arange(n, dtype=np.float64) * 0.5 * 3.0 - 1.0
    assert np.array_equal(y.cpu().numpy(), ref)
    z = torch.zeros(n, dtype=torch.int64, device=dev)
    tz = DeviceTensor(_Root(z, 1, 0, n, _lib.PMX_I64), 0, (n,), "int")
    P.eval_loop(n, P.lam("i", P.tensor_set(tz, ["i"], P.addi(P.muli("i", "i"), P.modi("i", 7)))))
    default_ctx().check_errors()
    i = np.arange(n, dtype=np.int64)
    assert np.array_equal(z.cpu().numpy(), i * i + i % 7)


def test_elementwise_loop_misaligned_view_and_short_tensor():
    n = 100_001
    dev = torch.device("cuda", 0)
    base = torch.arange(n + 3, dtype=torch.float32, device=dev)
    out = torch.zeros(n + 3, dtype=torch.float32, device=dev)
    # views starting at element 1 (not on a 16-byte boundary): lane path
    tx = DeviceTensor(_Root(base, 0, 0, n + 3, _lib.PMX_F32), 1, (n,), "float")
    ty = DeviceTensor(_Root(out, 1, 0, n + 3, _lib.PMX_F32), 1, (n,), "float")
    P.eval_loop(n, P.lam("i", P.tensor_set(ty, ["i"], P.addf(P.tensor_get(tx, ["i"]), 0.5))))
    default_ctx().check_errors()
    o = out.cpu().numpy()
    assert o[0] == 0 and np.array_equal(o[1:n + 1], np.arange(1, n + 1, dtype=np.float32) + 0.5)
    # loop longer than the tensor: the first out-of-bounds iteration is reported
    short = _tensor(torch.zeros(n - 10, dtype=torch.float32, device=dev), 2)
    with pytest.raises(P.Diagnostics, match="out of bounds") as ei:
        P.accelerate(lambda: P.eval_loop(n, P.lam("i", P.tensor_set(short, ["i"], 1.0))))
    assert f"iteration {n - 10})" in str(ei.value)


def test_elementwise_loop_error_index():
    n = N
    dev = torch.device("cuda", 0)
    x = torch.ones(n, dtype=torch.int64, device=dev)
    x[123_457] = 0
    y = torch.zeros(n, dtype=torch.int64, device=dev)
    tx = DeviceTensor(_Root(x, 0, 0, n, _lib.PMX_I64), 0, (n,), "int")
    ty = DeviceTensor(_Root(y, 1, 0, n, _lib.PMX_I64), 0, (n,), "int")
    with pytest.raises(P.Diagnostics, match="integer division by zero") as ei:
        P.accelerate(lambda: P.eval_loop(n, P.lam("i", P.tensor_set(ty, ["i"], P.divi(5, P.tensor_get(tx, ["i"]))))))
    assert "iteration 123457)" in str(ei.value)


def test_seq_loop_specialised_persistent_kernel():
    # seqLoop above the threshold: run-time specialised persistent kernel with
    # a software grid barrier per step; odd step count (result in scratch,
    # copied back), neighbour reads through the previous state
    m, steps = (1 << 16) + 5, 7
    s0 = np.arange(m, dtype=np.float64) % 97
    step = P.lam("x", "j", "t", P.mulf(0.5, P.addf("x", P.get(P.PREV, P.modi(P.addi("j", 1), m)))))
    before = _launched()
    got = np.asarray(P.accelerate(lambda s: P.seq_loop(steps, step, s), s0))
    assert _launched() > before
    want = s0.copy()
    for _ in range(steps):
        want = 0.5 * (want + np.roll(want, -1))
    assert np.array_equal(got, want)
    # an error in step 3 at element 4242 (division by zero) is reported
    bad = P.lam("x", "j", "t", P.match(P.eqi("t", 3), True,
                                       P.divf("x", P.int2float(P.subi("j", 4242))), "x"))
    with pytest.raises(P.Diagnostics, match="float division by zero") as ei:
        P.accelerate(lambda s: P.seq_loop(steps, bad, s), s0)
    assert "element 4242)" in str(ei.value)


def test_seq_loop_multi_lane_passes_and_tail():
    # m large enough that the specialised kernel runs its 8-elements-per-thread
    # passes (grid-strided) and then a ragged scalar tail; an error raised in two
    # elements of the multi-lane region reports the smaller one
    m, steps = (1 << 22) + 3, 3
    s0 = np.arange(m, dtype=np.float64) % 89
    step = P.lam("x", "j", "t", P.addf(P.mulf(0.5, P.addf("x", P.get(P.PREV, P.modi(P.addi("j", 7), m)))),
                                       P.mulf(0.25, P.int2float(P.modi("j", 5)))))
    got = np.asarray(P.accelerate(lambda s: P.seq_loop(steps, step, s), s0))
    want = s0.copy()
    jm = (np.arange(m) % 5).astype(np.float64)
    for _ in range(steps):
        want = 0.5 * (want + np.roll(want, -7)) + 0.25 * jm
    assert np.array_equal(got, want)
    # straight-line (so the multi-lane path runs it): zero divisor at two elements
    bad = P.lam("x", "j", "t", P.divf("x", P.int2float(P.muli(P.subi("j", 1_000_003), P.subi("j", 3_000_017)))))
    with pytest.raises(P.Diagnostics, match="float division by zero") as ei:
        P.accelerate(lambda s: P.seq_loop(steps, bad, s), s0)
    assert "element 1000003)" in str(ei.value)


def test_reduce_unrecognised_operator_is_an_ordered_fold():
    # leftmost non-zero: associative, not commutative -> only an order-keeping
    # tree gives the sequential answer
    n = (1 << 20) + 13
    x = np.zeros(n, dtype=np.int64)
    x[777_777] = 5
    x[900_001] = 9
    x[3] = 0
    first_nz = P.lam("a", "b", P.if_(P.eqi("a", 0), "b", "a"))
    before = _launched()
    got = P.accelerate(lambda s: P.eval_reduce(first_nz, 0, s), x)
    assert _launched() > before
    assert got == 5
    x[123] = -4
    assert P.accelerate(lambda s: P.eval_reduce(first_nz, 0, s), x) == -4
    # generic map feeding a generic (sum written as two instructions) operator
    xi = (np.arange(n, dtype=np.int64) % 1000) - 500
    add2 = P.lam("a", "b", P.addi("a", P.muli("b", 1)))
    sq = P.lam("v", P.muli("v", "v"))
    got = P.accelerate(lambda s: P.eval_reduce(add2, 7, P.eval_map(sq, s)), xi)
    assert got == 7 + int(np.sum(xi * xi))
    # mirrored float max (not the recognised form): exact fold semantics
    xf = np.random.default_rng(1).standard_normal(n)
    mx = P.lam("a", "b", P.if_(P.gtf("b", "a"), "b", "a"))
    assert P.accelerate(lambda s: P.eval_reduce(mx, -1e300, s), xf) == float(np.max(xf))

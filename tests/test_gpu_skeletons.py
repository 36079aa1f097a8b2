"""Parity of the sm_100a skeleton kernels with the reference (golden fixtures
produced by the reference interpreter) and with the CPU oracle.  Every call
goes through the C ABI (libpmxb200.so)."""
import math

import numpy as np
import torch
import pytest

import oracle as O
from cases import FOLD_CASES, MAP2_CASES, MAP_CASES, REDUCE_CASES
from conftest import parse_tokens
from paper_2211_00621_b200 import (
    Ctx, Diagnostics, Heap, TensorView, accelerate, addf, addi, char, eval_loop, eval_map, eval_map2,
    eval_reduce, flatten, fold, lam, match, modi, mulf, muli, seq_loop, synth, tensor_get, tensor_set,
    get, gti, lti, if_, field_, divf, int2float, PREV, subi, divi,
)

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[0, 1], ids=["vm", "jit"], autouse=True)
def jit_mode(request):
    """Every case runs twice: bytecode interpreter only, and always through
    the run-time specialised kernels (csrc/jit.cu)."""
    from paper_2211_00621_b200 import _lib
    lib = _lib.load()
    prev = lib.pmx_jit_set_mode(request.param)
    yield request.param
    lib.pmx_jit_set_mode(prev)

TRANSCENDENTAL = {"exp", "log", "sin_cos", "float_math"}


def _host(v):
    if isinstance(v, np.ndarray):
        return v.tolist()
    return v


def _check_values(got, want, name):
    assert len(got) == len(want), (got, want)
    for g, w in zip(got, want):
        if isinstance(w, float):
            if name in TRANSCENDENTAL:   # CUDA libm vs glibc: <= 1-2 ulp
                assert math.isclose(g, w, rel_tol=1e-15, abs_tol=1e-300), (name, g, w)
            else:
                assert g == w and math.copysign(1, g) == math.copysign(1, w), (name, g, w)
        else:
            assert int(g) == w, (name, g, w)


@pytest.mark.parametrize("case", MAP_CASES, ids=[c[0] for c in MAP_CASES])
def test_map_matches_reference(case, golden):
    name, _, build, ty, xs = case
    entry = golden["map"][name]
    body = lambda s: eval_map(build(), s)
    if "error" in entry:
        with pytest.raises(Diagnostics) as ei:
            accelerate(body, list(xs))
        assert entry["error"] in str(ei.value)
        return
    got = _host(accelerate(body, list(xs)))
    _check_values(got, parse_tokens(entry["stdout"]), name)


@pytest.mark.parametrize("case", REDUCE_CASES, ids=[c[0] for c in REDUCE_CASES])
def test_reduce_matches_reference(case, golden):
    name, _, build, _, acc, ty, xs = case
    want = parse_tokens(golden["reduce"][name]["stdout"])[0]
    seq = np.array(xs, dtype=np.float64 if ty == "float" else np.int64)
    got = accelerate(lambda s: eval_reduce(build(), acc, s), seq)
    assert got == want


@pytest.mark.parametrize("case", FOLD_CASES, ids=[c[0] for c in FOLD_CASES])
def test_foldl_matches_reference(case, golden):
    name, _, build, _, acc, ty, xs = case
    want = parse_tokens(golden["foldl"][name]["stdout"])[0]
    assert accelerate(lambda s: fold(build(), acc, s), list(xs)) == want


@pytest.mark.parametrize("case", MAP2_CASES, ids=[c[0] for c in MAP2_CASES])
def test_map2_matches_reference(case, golden):
    name, _, build, ty, xs, ys = case
    entry = golden["map2"][name]
    if "error" in entry:
        with pytest.raises(Diagnostics, match="different lengths"):
            accelerate(lambda a, b: eval_map2(build(), a, b), list(xs), list(ys))
        return
    got = _host(accelerate(lambda a, b: eval_map2(build(), a, b), list(xs), list(ys)))
    _check_values(got, parse_tokens(entry["stdout"]), name)


# ------------------------------------------------------------ known answers

def test_accel_sum_schedule_independent(golden):
    # tests/test_interp.py:99-114 : reduce addi 0 (map (lam x. muli x x) [1..10]) = 385
    f = lambda s: eval_reduce(addi, 0, eval_map(lam("x", muli("x", "x")), s))
    want = {int(v["stdout"]) for v in golden["accel_sum"].values() if isinstance(v, dict)}
    assert want == {385}
    for _ in range(20):
        assert accelerate(f, list(range(1, 11))) == 385


def test_alias_end_to_end(golden):
    # tests/test_acceptance.py:219-241: views (0,4) and (1,5) of one buffer share
    # one device root; loop writes 7 through b1, host sees t[1] == 7.
    for _ in range(10):
        heap = Heap()
        buf = heap.alloc(np.zeros(8, np.int64))
        v1 = TensorView(buf, 0, (4,), "int")
        v2 = TensorView(buf, 1, (5,), "int")

        def kernel(b1, b2):
            eval_loop(4, lam("i", tensor_set(b1, ["i"], 7)))
            return eval_map(lam("x", tensor_get(b2, [3])), [0])  # read after the loop

        ctx = Ctx(heap=heap)
        accelerate(kernel, v1, v2, ctx=ctx)
        assert heap.buffers[buf][1] == 7 == int(golden["alias"]["2"]["stdout"])
        assert len(ctx.last_arena.roots) == 1


def test_loop_squares_and_arith(golden):
    # corpus loop_squares / loop_arith (tests/corpus.py:42-52, 184-196)
    heap = Heap()
    b = heap.alloc(np.zeros(8, np.int64))
    t = TensorView(b, 0, (8,), "int")
    accelerate(lambda tt: eval_loop(8, lam("i", tensor_set(tt, ["i"], muli("i", "i")))), t, ctx=Ctx(heap=heap))
    out = golden["corpus"]["loop_squares"]["stdout"].split()
    assert int(heap.buffers[b][7]) == int(out[0]) and int(heap.buffers[b][3]) == int(out[1])
    heap = Heap()
    b = heap.alloc(np.zeros(10, np.int64))
    t = TensorView(b, 0, (10,), "int")
    accelerate(lambda tt: eval_loop(10, lam("i", tensor_set(tt, ["i"], addi(divi(muli("i", "i"), 2), modi("i", 3))))),
               t, ctx=Ctx(heap=heap))
    out = golden["corpus"]["loop_arith"]["stdout"].split()
    assert int(heap.buffers[b][9]) == int(out[0]) and int(heap.buffers[b][4]) == int(out[1])


def test_tensor_sub_alias(golden):
    # corpus tensor_sub_alias: left = t[0:4], right = t[2:6]; loop sets right[i] = i+1
    heap = Heap()
    b = heap.alloc(np.full(6, 10, np.int64))
    left, right = TensorView(b, 0, (4,), "int"), TensorView(b, 2, (4,), "int")
    r = accelerate(lambda v1, v2: (eval_loop(4, lam("i", tensor_set(v2, ["i"], addi("i", 1)))),
                                   eval_map(lam("z", tensor_get(v1, [2])), [0]))[1], left, right,
                   ctx=Ctx(heap=heap))
    out = golden["corpus"]["tensor_sub_alias"]["stdout"].split()
    assert int(r[0]) == int(out[0]) and int(heap.buffers[b][5]) == int(out[1])


def test_read_only_view_not_copied_back():
    # a root that no kernel stores into (only tensor_get) is not copied back
    # by marshal_out; a written one is (pmx/runtime.py:262-282)
    heap = Heap()
    b = heap.alloc(np.arange(16, dtype=np.int64))
    t = TensorView(b, 0, (16,), "int")
    ctx = Ctx(heap=heap)
    r = accelerate(lambda tt: eval_reduce(addi, 0, eval_map(lam("i", tensor_get(tt, ["i"])), list(range(16)))),
                   t, ctx=ctx)
    assert r == sum(range(16))
    assert not any(root.dirty for root in ctx.last_arena.roots)
    assert ctx.last_arena.d2h_bytes <= 8                  # the scalar result only
    ctx = Ctx(heap=heap)
    accelerate(lambda tt: eval_loop(16, lam("i", tensor_set(tt, ["i"], muli("i", 2)))), t, ctx=ctx)
    assert all(root.dirty for root in ctx.last_arena.roots)
    assert int(heap.buffers[b][15]) == 30


def test_tensor_oob_is_an_error():
    heap = Heap()
    b = heap.alloc(np.zeros(2, np.int64))
    t = TensorView(b, 0, (2,), "int")
    with pytest.raises(Diagnostics, match="out of bounds"):
        accelerate(lambda tt: eval_loop(3, lam("i", tensor_set(tt, ["i"], 1))), t, ctx=Ctx(heap=heap))


def test_corpus_programs(golden):
    c = golden["corpus"]
    assert accelerate(lambda s: eval_reduce(addi, 0, eval_map(lam("x", addi("x", 1)), s)), [1, 2, 3, 4, 5]) \
        == int(c["map_increment"]["stdout"])
    u = [float(i + 1) for i in range(9)]
    v = [float(10 - i) for i in range(9)]
    d = accelerate(lambda a, b: eval_reduce(addf, 0.0, eval_map2(mulf, a, b)), u, v)
    assert math.isclose(d, float(c["dot_product"]["stdout"]), rel_tol=1e-6)
    assert accelerate(lambda s: eval_reduce(muli, 1, s), list(range(1, 11))) == int(c["reduce_product"]["stdout"])
    r = accelerate(lambda s: {"len": len(flatten(s)), "total": eval_reduce(addi, 0, flatten(s))},
                   [[1, 2], [3, 4], [5, 6]])
    assert f"{r['len']} {r['total']}" == c["flatten_sum"]["stdout"]
    r = accelerate(lambda s: {"lo": eval_reduce(lam("x", "y", if_(lti("x", "y"), "x", "y")), 99, s),
                              "hi": eval_reduce(lam("x", "y", if_(gti("x", "y"), "x", "y")), 0, s)},
                   [17, 4, 42, 8, 23])
    assert f"{r['lo']} {r['hi']}" == c["record_result"]["stdout"]
    assert accelerate(lambda s: eval_reduce(addi, 0, eval_map(lam("x", match(modi("x", 2), 0, 1, 0)), s)),
                      [i * 3 for i in range(20)]) == int(c["count_evens"]["stdout"])
    assert accelerate(lambda s: eval_reduce(addi, 0, eval_map(lam("c", match("c", char("a"), 1, 0)), s)),
                      list("abracadabra")) == int(c["char_count"]["stdout"])
    r = accelerate(lambda s: eval_map(lam("x", "x"), s), [1, 2, 3])   # identity map
    assert list(r) == [1, 2, 3]
    assert accelerate(lambda s: eval_reduce(addi, 0, eval_map(lam("p", field_("p", "age")), s)),
                      [{"age": 31, "id": 1}, {"age": 27, "id": 2}, {"age": 45, "id": 3}]) \
        == int(c["map_records"]["stdout"])
    s = [(i * 17) % 31 for i in range(30)]
    assert accelerate(lambda s: eval_reduce(lam("x", "y", if_(gti("x", "y"), "x", "y")), 0, s), s) \
        == int(c["reduce_max"]["stdout"])
    # captured host data: offset = [100,200,300] captured, scale = 3
    assert accelerate(lambda s, off: eval_reduce(addi, 0, eval_map2(lam("x", "o", addi(muli(3, "x"), "o")), s, off)),
                      [1, 2, 3], [100, 200, 300]) == int(c["captured_host_data"]["stdout"])
    assert accelerate(lambda s: eval_reduce(addi, 0, eval_map(lam("x", modi(muli("x", 7), 13)), s)),
                      list(range(1000))) == int(c["large_map_sum"]["stdout"])
    r = accelerate(lambda s: eval_map(lam("x", addi(divi("x", 3), modi("x", 3))), s), [-7, -4, -1, 1, 4, 7])
    assert " ".join(str(int(v)) for v in r) == c["negative_arith"]["stdout"].strip()
    r = accelerate(lambda s: eval_reduce(addf, 0.0, eval_map(lam("x", divf(1.0, int2float("x"))), s)),
                   list(range(1, 201)))
    assert math.isclose(r, float(c["float_reduce_large"]["stdout"]), rel_tol=1e-6)
    # sequential accelerates: double then total
    s2 = accelerate(lambda s: eval_map(lam("x", muli(2, "x")), s), [1, 2, 3])
    assert accelerate(lambda s: eval_reduce(addi, 0, s), s2) == int(c["sequential_accelerates"]["stdout"])


def test_get_on_captured_sequence():
    # map (lam i. get data i) over indices; out-of-bounds get is an error
    data = np.array([5, 6, 7], np.int64)
    r = accelerate(lambda d, idx: eval_map(lam("i", get(d, "i")), idx), data, [2, 0, 1])
    assert list(r) == [7, 5, 6]
    with pytest.raises(Diagnostics, match="out of bounds"):
        accelerate(lambda d, idx: eval_map(lam("i", get(d, "i")), idx), data, [0, 3])


# --------------------------------------------------------- microbench config

def test_mapreduce_parity_with_golden(golden):
    for e in golden["mapreduce"]:
        x = synth.mapreduce_x(e["N"])
        r = accelerate(lambda s: eval_reduce(addf, 0.0, eval_map(lam("x", addf(mulf(2.0, "x"), 1.0)), s)), x)
        assert r == float(e["stdout"])            # exact: fp64 accumulation of exact data


@pytest.mark.parametrize("n", [1, 3, 4, 5, 1023, 4097, (1 << 20) + 3])
def test_mapreduce_sizes_and_tails(n):
    x = synth.mapreduce_x(n)
    f = lam("x", addf(mulf(2.0, "x"), 1.0))
    r = accelerate(lambda s: eval_reduce(addf, 0.0, eval_map(f, s)), x)
    assert r == synth.mapreduce_exact_sum(n) == O.map_affine_reduce_add(x, workers=4)
    y = accelerate(lambda s: eval_map(f, s), x)
    assert np.array_equal(y, (2.0 * x.astype(np.float64) + 1.0).astype(np.float32))


def test_mapreduce_misaligned_view():
    import torch
    x = torch.from_numpy(synth.mapreduce_x(10001)).cuda()
    xs = x[1:]                                  # 4-byte aligned only -> scalar path
    f = lam("x", addf(mulf(2.0, "x"), 1.0))
    r = accelerate(lambda s: eval_reduce(addf, 0.0, eval_map(f, s)), xs)
    want = O.map_affine_reduce_add(synth.mapreduce_x(10001)[1:])
    assert r == want


def test_mapreduce_full_config_exact():
    """2^28 fp32 elements, device-resident: the fused map->reduce must equal the
    exact rational sum (fp64 accumulation), and the materialised map must be
    bit-exact against 2x+1."""
    import torch
    from paper_2211_00621_b200.skeletons import LazyMap, default_ctx
    n = 1 << 28
    x = synth.mapreduce_x_device(n, torch.device("cuda"))
    f = lam("x", addf(mulf(2.0, "x"), 1.0))
    from paper_2211_00621_b200.runtime import DeviceSeq
    from paper_2211_00621_b200 import _lib
    s = DeviceSeq(x, (n,), _lib.PMX_F32)
    lm = eval_map(f, s)
    tot = eval_reduce(addf, 0.0, lm, keep_map=True).get()
    assert tot == synth.mapreduce_exact_sum(n)
    y = lm.materialize().data
    ref = torch.addcmul(torch.ones_like(x), x, torch.full_like(x, 2.0))
    assert torch.equal(y, ref)
    default_ctx().check_errors()


def test_empty_sequences():
    assert accelerate(lambda s: eval_reduce(addi, 7, s), np.zeros(0, np.int64)) == 7
    r = accelerate(lambda s: eval_map(lam("x", addi("x", 1)), s), np.zeros(0, np.int64))
    assert len(r) == 0
    assert accelerate(lambda: eval_loop(0, lam("i", "i"))) == {}


def test_seq_loop_persistent_iteration():
    # state'[j] = 0.5 * (prev[j] + prev[(j+1) mod m]) iterated 50 times
    m = 1000
    s0 = np.arange(m, dtype=np.float64)
    step = lam("x", "j", "t", mulf(0.5, addf("x", get(PREV, modi(addi("j", 1), m)))))
    got = accelerate(lambda s: seq_loop(50, step, s), s0)
    ref = s0.copy()
    for _ in range(50):
        ref = 0.5 * (ref + np.roll(ref, -1))
    assert np.allclose(got, ref, rtol=1e-14)


@pytest.mark.parametrize("steps", [0, 1, 2, 7])
@pytest.mark.parametrize("m", [1000, 1 << 16])
def test_seq_loop_leaves_input_and_counts_steps(steps, m):
    # the initial state is an immutable value: step 0 reads it (pmx_seq_loop_from)
    # and the caller's device sequence is unchanged afterwards; odd step counts
    # land in the right buffer; both the interpreter (small m) and the
    # specialised kernel (large m) paths
    from paper_2211_00621_b200.runtime import seq_to_device
    s0 = np.arange(m, dtype=np.float64) % 97
    step = lam("x", "j", "t", addf(mulf(0.5, addf("x", get(PREV, modi(addi("j", 1), m)))), 1.0))

    def body(s):
        dev = seq_to_device(s) if not hasattr(s, "data") else s
        before = dev.data.clone()
        out = seq_loop(steps, step, dev)
        assert torch.equal(dev.data, before)
        return out
    got = accelerate(body, s0)
    ref = s0.copy()
    for _ in range(steps):
        ref = 0.5 * (ref + np.roll(ref, -1)) + 1.0
    assert np.allclose(got, ref, rtol=1e-13)


def test_map_rows_fold_irregular_and_regular(jit_mode):
    # map (lam row. reduce addi 0 (map (lam x. muli x x) row)) over irregular rows,
    # foldl with a non-commutative operator (left fold order), float rows
    from paper_2211_00621_b200 import map_rows_fold, subf
    rows = [[1, 2, 3], [], [4], [5, 6, 7, 8]]
    got = accelerate(lambda s: map_rows_fold(lam("x", muli("x", "x")), addi, 0, s), rows)
    assert [int(v) for v in got] == [14, 0, 16, 174]
    got = accelerate(lambda s: map_rows_fold(None, subi, 100, s), rows)
    assert [int(v) for v in got] == [94, 100, 96, 74]
    frows = [[0.5, 0.25, 0.125], [1.5, -2.0, 3.25]]
    got = accelerate(lambda s: map_rows_fold(None, subf, 1.0, s), frows)
    assert list(got) == [((1.0 - 0.5) - 0.25) - 0.125, ((1.0 - 1.5) + 2.0) - 3.25]


def test_map_rows_fold_error_reports_row(jit_mode):
    from paper_2211_00621_b200 import map_rows_fold
    rows = [[1, 2], [3, 0], [0]]
    with pytest.raises(Diagnostics, match="integer division by zero") as ei:
        accelerate(lambda s: map_rows_fold(lam("x", divi(12, "x")), addi, 0, s), rows)
    assert "element 1)" in str(ei.value)


def test_linear_recursion_loop(jit_mode):
    """Iterate (a linear recursion run base case upward, lambdas.py) on the
    device vs the oracle's evaluator: Int and Float accumulators, and the
    recursion-depth error for an argument below the base case."""
    from paper_2211_00621_b200 import lambdas as L
    fact = L.Lam(["n"], L.Iterate("m", L.Const(1, "int"), L.Var("n"), "a", L.Const(1, "int"),
                                  L.Prim("muli", [L.Var("m"), L.Var("a")])))
    harm = L.Lam(["n"], L.Iterate("m", L.Const(1, "int"), L.Var("n"), "a", L.Const(0.0, "float"),
                                  L.Prim("addf", [L.Var("a"), L.Prim("divf", [L.Const(1.0, "float"),
                                                                            L.Prim("int2float", [L.Var("m")])])])))
    xs = list(range(0, 300, 7)) + [1000, 4096]
    for f in (fact, harm):
        got = accelerate(lambda s: eval_map(f, s), xs)
        _check_values(_host(got), [O.ir_apply(f, x) for x in xs], "recursion")
    with pytest.raises(Diagnostics, match="maximum recursion depth exceeded") as ei:
        accelerate(lambda s: eval_map(fact, s), [3, 4, -1, 5, -7])
    assert "element 2)" in str(ei.value)
    with pytest.raises(Diagnostics, match="maximum recursion depth exceeded"):
        accelerate(lambda s: eval_map(fact, s), [1 << 40])

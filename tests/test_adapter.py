"""The whole-program adapter's translation of reference closures, checked on CPU
against the reference itself: every parallel construct of the reference's
24-program corpus (tests/corpus.py) is translated from the reference's
Closure/BuiltinPartial to this repo's lambda IR and evaluated with the oracle's
IR evaluator; the program's output must equal the reference's own.  Needs the
reference (present in the build container only; skipped elsewhere).  The GPU
replay of the same translated constructs is tests/test_gpu_adapter.py."""
import pathlib
import sys

import pytest

REF = pathlib.Path("/root/reference/pkg")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference interpreter not available")

# constructs the device cannot run: nested sequences as elements, recursion
UNSUPPORTED: set = set()   # recursion_pow runs as a device loop (linear recursion)


def _pmx():
    sys.path.insert(0, str(REF / "src"))
    sys.path.insert(0, str(REF / "tests"))
    import pmx
    import pmx.interp as interp
    return pmx, interp


def install_checker(interp):
    """Replace the reference skeletons with: translate f (adapter) -> evaluate
    the IR with the oracle.  Mirrors pmx_adapter.install but on the CPU
    checker instead of the device (test infrastructure only)."""
    import oracle as O
    from paper_2211_00621_b200 import pmx_adapter
    from paper_2211_00621_b200.ir_json import HostArray
    import pmx.runtime as rt
    import pmx.syntax as syn

    orig = {n: getattr(interp, n) for n in ("eval_map", "eval_map2", "eval_reduce", "eval_loop")}

    def tr(f, n, ctx, span):
        def host_array(v):
            if isinstance(v, rt.TensorView):
                h = HostArray([], v.elem, v.shape, v.offset)
                h.data = ctx.heap.buffers[v.buffer]          # live buffer: effects land in the heap
                return h
            return HostArray([ord(x) if isinstance(x, str) else x for x in v], "int")
        try:
            return pmx_adapter.to_lam(f, n, syn, rt, host_array)
        except pmx_adapter.Unsupported as exc:
            raise rt.runtime_error(f"not supported on the B200 device: {exc}", span) from None

    def conv(s):
        return [ord(x) if isinstance(x, str) else x for x in s]

    def wrap(fn):
        def g(*a):
            try:
                return fn(*a)
            except O.OracleError as exc:
                raise rt.runtime_error(str(exc)) from None
        return g

    @wrap
    def eval_map(f, s, ctx, span):
        if not ctx.run_parallel or not s:
            return orig["eval_map"](f, s, ctx, span)
        if isinstance(s[0], list):                   # row function: left fold per row
            try:
                g, op, acc = pmx_adapter.to_row_fold(f, syn, rt, lambda v: HostArray(conv(v), "int"))
            except pmx_adapter.Unsupported as exc:
                raise rt.runtime_error(f"not supported on the B200 device: {exc}", span) from None
            out = []
            for row in s:
                a = acc
                for x in conv(row):
                    a = O.ir_apply(op, a, O.ir_apply(g, x) if g is not None else x)
                out.append(a)
            return out
        return O.ir_map(tr(f, 1, ctx, span), conv(s))

    @wrap
    def eval_map2(f, s1, s2, ctx, span):
        if not ctx.run_parallel or not s1:
            return orig["eval_map2"](f, s1, s2, ctx, span)
        return O.ir_map2(tr(f, 2, ctx, span), conv(s1), conv(s2))

    @wrap
    def eval_reduce(f, acc, s, ctx, span):
        if not ctx.run_parallel or not s:
            return orig["eval_reduce"](f, acc, s, ctx, span)
        return O.ir_fold(tr(f, 2, ctx, span), acc, conv(s))

    @wrap
    def eval_loop(n, f, ctx, span):
        if not ctx.run_parallel or n <= 0:
            return orig["eval_loop"](n, f, ctx, span)
        lam = tr(f, 1, ctx, span)
        for i in range(n):
            O.ir_apply(lam, i)

    interp.eval_map, interp.eval_map2, interp.eval_reduce, interp.eval_loop = eval_map, eval_map2, eval_reduce, eval_loop

    def uninstall():
        for k, v in orig.items():
            setattr(interp, k, v)
    return uninstall


def _corpus():
    sys.path.insert(0, str(REF / "tests"))
    from corpus import CORPUS
    return CORPUS


@pytest.mark.parametrize("case", _corpus() if REF.exists() else [], ids=lambda c: c[0])
def test_corpus_program_through_adapter(case, golden):
    pmx, interp = _pmx()
    from conftest import tokens_match
    name, src, rel = case
    un = install_checker(interp)
    try:
        if name in UNSUPPORTED:
            with pytest.raises(pmx.Diagnostics, match="not supported on the B200 device"):
                pmx.run_source(src, mode="accel", workers=4, capture_output=True)
            return
        out = pmx.run_source(src, mode="accel", workers=4, capture_output=True).stdout
    finally:
        un()
    assert tokens_match(out, golden["corpus"][name]["stdout"], float_rel=rel or 1e-12), (out,)


def test_interp_known_answers_through_adapter(golden):
    pmx, interp = _pmx()
    ACCEL_SUM = golden["accel_sum"]["program"]          # tests/test_interp.py:99-104
    ALIAS_PROGRAM = golden["alias"]["program"]          # tests/test_acceptance.py:219-229
    un = install_checker(interp)
    try:
        for w in (1, 2, 3, 8, 16):
            assert pmx.run_source(ACCEL_SUM, mode="accel", workers=w, capture_output=True).stdout == "385"
        for w in (1, 2, 8):
            assert pmx.run_source(ALIAS_PROGRAM, mode="accel", workers=w, capture_output=True).stdout == "7"
    finally:
        un()


def test_runtime_errors_keep_reference_messages():
    pmx, interp = _pmx()
    un = install_checker(interp)
    try:
        src = "let f = lam s. map (lam x. divi 10 x) s in let r = accelerate (f [1, 0]) in print (int2string (reduce addi 0 r))"
        with pytest.raises(pmx.Diagnostics, match="integer division by zero"):
            pmx.run_source(src, mode="accel", workers=2, capture_output=True)
    finally:
        un()


RECURSIVE = [
    # linear recursion -> device loop (pmx_adapter._Translator.linear_recursion)
    ("fact", "recursive let fact = lam n. match n with 0 then 1 else muli n (fact (subi n 1)) in "
             "let r = accelerate (map fact [0, 1, 5, 12, 20]) in print (int2string (reduce addi 0 r))", True),
    ("harmonic", "recursive let h = lam n. match n with 0 then 0.0 else addf (h (subi n 1)) "
                 "(divf 1.0 (int2float n)) in "
                 "let r = accelerate (map h [1, 2, 10, 100]) in print (float2string (reduce addf 0.0 r))", True),
    ("base_second", "recursive let p = lam n. lam k. match n with 1 then k else addi (muli k 3) (p (subi n 1) k) in "
                    "let r = accelerate (map (lam x. p x 7) [1, 2, 6]) in print (int2string (reduce addi 0 r))", True),
    ("let_in_step", "recursive let g = lam n. match n with 0 then 2 else let t = g (subi n 1) in "
                    "modi (addi (muli t t) n) 1000003 in "
                    "let r = accelerate (map g [0, 4, 50]) in print (int2string (reduce addi 0 r))", True),
    # k-term recurrences -> device loop with k accumulators (kterm_recursion)
    ("fib", "recursive let fib = lam n. match n with 0 then 0 else match n with 1 then 1 else "
            "addi (fib (subi n 1)) (fib (subi n 2)) in "
            "let r = accelerate (map fib [3, 7]) in print (int2string (reduce addi 0 r))", True),
    ("fib_bases_only", "recursive let fib = lam n. match n with 0 then 0 else match n with 1 then 1 else "
                       "addi (fib (subi n 1)) (fib (subi n 2)) in "
                       "let r = accelerate (map fib [0, 1, 2, 15]) in print (int2string (reduce addi 0 r))", True),
    ("trib_bases_reordered", "recursive let t = lam n. match n with 3 then 1 else match n with 1 then 0 else "
                             "match n with 2 then 0 else addi (t (subi n 3)) (addi (t (subi n 1)) (t (subi n 2))) in "
                             "let r = accelerate (map t [1, 2, 3, 4, 10, 13]) in "
                             "print (int2string (reduce addi 0 r))", True),
    ("kterm_float_let", "recursive let g = lam x. lam n. match n with 0 then x else match n with 1 then 1.0 else "
                        "let a = g x (subi n 1) in let b = g x (subi n 2) in addf (mulf 0.5 a) (mulf x b) in "
                        "let r = accelerate (map (lam n. g 0.25 n) [0, 1, 2, 9, 14]) in "
                        "print (float2string (reduce addf 0.0 r))", True),
    # recursive calls under a match of the step: the reference may skip levels, not lowered
    ("kterm_lazy_call", "recursive let f = lam n. match n with 0 then 1 else match n with 1 then 2 else "
                        "match modi n 2 with 0 then f (subi n 1) else addi (f (subi n 1)) (f (subi n 2)) in "
                        "let r = accelerate (map f [5]) in print (int2string (reduce addi 0 r))", False),
    # no f (n-1) call: the reference visits every other level only, not lowered
    ("kterm_stride_two", "recursive let f = lam n. match n with 0 then 1 else match n with 1 then 1 else "
                         "muli 3 (f (subi n 2)) in "
                         "let r = accelerate (map f [6, 7]) in print (int2string (reduce addi 0 r))", False),
]


@pytest.mark.parametrize("name,src,supported", RECURSIVE, ids=[r[0] for r in RECURSIVE])
def test_linear_recursion_matches_reference(name, src, supported):
    pmx, interp = _pmx()
    want = pmx.run_source(src, mode="debug", capture_output=True).stdout
    un = install_checker(interp)
    try:
        if not supported:
            with pytest.raises(pmx.Diagnostics, match="not supported on the B200 device"):
                pmx.run_source(src, mode="accel", workers=2, capture_output=True)
            return
        got = pmx.run_source(src, mode="accel", workers=2, capture_output=True).stdout
    finally:
        un()
    assert got == want


def test_kterm_recursion_below_the_base_cases_is_an_error():
    """fib n for n < 0 recurses forever in the reference; the device loop
    reports the recursion error instead of returning a base case."""
    pmx, interp = _pmx()
    src = ("recursive let fib = lam n. match n with 0 then 0 else match n with 1 then 1 else "
           "addi (fib (subi n 1)) (fib (subi n 2)) in "
           "let r = accelerate (map fib [3, -1]) in print (int2string (reduce addi 0 r))")
    un = install_checker(interp)
    try:
        with pytest.raises(pmx.Diagnostics, match="maximum recursion depth exceeded"):
            pmx.run_source(src, mode="accel", workers=2, capture_output=True)
    finally:
        un()


def test_recursion_that_never_reaches_the_base_case_is_an_error():
    """pow b n for n < 0 recurses forever in the reference (stack overflow);
    the device loop reports it instead of returning the base case."""
    pmx, interp = _pmx()
    src = ("recursive let pow = lam b. lam n. match n with 0 then 1 else muli b (pow b (subi n 1)) in "
           "let r = accelerate (map (pow 2) [3, -1]) in print (int2string (reduce addi 0 r))")
    un = install_checker(interp)
    try:
        with pytest.raises(pmx.Diagnostics, match="maximum recursion depth exceeded"):
            pmx.run_source(src, mode="accel", workers=2, capture_output=True)
    finally:
        un()

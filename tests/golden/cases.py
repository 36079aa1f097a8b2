"""Skeleton / scalar-semantics cases shared by the golden generator and the tests.

Each case pairs the PMExpr text of a function argument (run by the reference
interpreter in tests/golden/make_golden.py to produce the expected output)
with the same function built in this repo's lambda IR (run on the B200 by
tests/test_gpu_skeletons.py and by the CPU IR evaluator in oracle/ir_eval.py).
"""
from paper_2211_00621_b200.lambdas import (
    addf, addi, cos, divf, divi, exp, floor, gti, if_, int2float, lam, log, lti, match, modi, mulf,
    muli, negf, negi, sin, sqrtf, subf, subi, gtf, ltf,
)

I64_MAX = 9223372036854775807

# (name, pmexpr lambda, IR builder, element type, inputs)
MAP_CASES = [
    ("addi_wrap", "lam x. addi x 9223372036854775807", lambda: lam("x", addi("x", I64_MAX)), "int", [0, 1, -5]),
    ("muli_wrap", "lam x. muli x 4611686018427387904", lambda: lam("x", muli("x", 4611686018427387904)), "int", [1, 2, 3]),
    ("subi_neg", "lam x. subi 3 x", lambda: lam("x", subi(3, "x")), "int", [5, -9]),
    ("negi", "lam x. negi x", lambda: lam("x", negi("x")), "int", [4, -9223372036854775807]),
    ("divi_trunc", "lam x. divi x 3", lambda: lam("x", divi("x", 3)), "int", [-7, -4, -1, 0, 1, 4, 7]),
    ("modi_trunc", "lam x. modi x 3", lambda: lam("x", modi("x", 3)), "int", [-7, -4, -1, 0, 1, 4, 7]),
    ("divi_neg_div", "lam x. divi x (negi 2)", lambda: lam("x", divi("x", negi(2))), "int", [7, -7]),
    ("divi_zero", "lam x. divi 10 x", lambda: lam("x", divi(10, "x")), "int", [1, 0]),
    ("modi_zero", "lam x. modi 10 x", lambda: lam("x", modi(10, "x")), "int", [3, 0]),
    ("affine_i", "lam x. addi (muli 3 x) 7", lambda: lam("x", addi(muli(3, "x"), 7)), "int", [0, 5, -2]),
    ("count_even", "lam x. match modi x 2 with 0 then 1 else 0",
     lambda: lam("x", match(modi("x", 2), 0, 1, 0)), "int", [0, 3, 6, 9]),
    ("lazy_branch", "lam x. match lti x 5 with true then muli x 2 else divi x 0",
     lambda: lam("x", if_(lti("x", 5), muli("x", 2), divi("x", 0))), "int", [1, 2, 7]),
    ("lazy_branch_ok", "lam x. match lti x 5 with true then muli x 2 else divi x 1",
     lambda: lam("x", if_(lti("x", 5), muli("x", 2), divi("x", 1))), "int", [1, 2, 7]),
    ("int2float", "lam x. int2float x", lambda: lam("x", int2float("x")), "int", [3, -7, 9007199254740993]),
    ("affine_f", "lam x. addf (mulf 2.0 x) 1.0", lambda: lam("x", addf(mulf(2.0, "x"), 1.0)), "float", [0.0, 0.25, -3.5]),
    ("mul_f", "lam x. mulf x 0.1", lambda: lam("x", mulf("x", 0.1)), "float", [3.0, 7.0]),
    ("sub_f", "lam x. subf x 0.3", lambda: lam("x", subf("x", 0.3)), "float", [0.1, 1.0]),
    ("divf", "lam x. divf 1.0 x", lambda: lam("x", divf(1.0, "x")), "float", [2.0, 3.0, -4.0]),
    ("divf_zero", "lam x. divf 1.0 x", lambda: lam("x", divf(1.0, "x")), "float", [1.0, 0.0]),
    ("negf", "lam x. negf x", lambda: lam("x", negf("x")), "float", [0.0, 1.5]),
    ("log", "lam x. log x", lambda: lam("x", log("x")), "float", [1.0, 2.5, 10.0]),
    ("log_zero", "lam x. log x", lambda: lam("x", log("x")), "float", [1.0, 0.0]),
    ("log_neg", "lam x. log x", lambda: lam("x", log("x")), "float", [-1.0]),
    ("exp", "lam x. exp x", lambda: lam("x", exp("x")), "float", [0.0, 1.5, -1000.0]),
    ("exp_range", "lam x. exp x", lambda: lam("x", exp("x")), "float", [1.0, 1000.0]),
    ("sqrt", "lam x. sqrtf x", lambda: lam("x", sqrtf("x")), "float", [4.0, 2.0, 0.0]),
    ("sqrt_neg", "lam x. sqrtf x", lambda: lam("x", sqrtf("x")), "float", [-1.0]),
    ("floor", "lam x. floor x", lambda: lam("x", floor("x")), "float", [2.9, -2.5, 1.0e20, -1.0e19]),
    ("sin_cos", "lam x. addf (sin x) (cos x)", lambda: lam("x", addf(sin("x"), cos("x"))), "float", [0.5, -2.0, 10.0]),
    ("float_math", "lam x. addf (sin x) (addf (cos x) (sqrtf (addf 1.0 (exp x))))",
     lambda: lam("x", addf(sin("x"), addf(cos("x"), sqrtf(addf(1.0, exp("x")))))), "float", [0.0, 0.5, 1.0, 1.5]),
    ("gtf_select", "lam x. match gtf x 0.5 with true then x else 0.0",
     lambda: lam("x", if_(gtf("x", 0.5), "x", 0.0)), "float", [0.25, 0.75]),
]

# (name, pmexpr operator, IR builder, acc literal (pmexpr), acc value, type, inputs)
REDUCE_CASES = [
    ("sum_i", "addi", lambda: addi, "0", 0, "int", list(range(1, 11))),
    ("prod_i", "muli", lambda: muli, "1", 1, "int", list(range(1, 11))),
    ("prod_wrap", "muli", lambda: muli, "1", 1, "int", [3037000500, 3037000500, 7]),
    ("min_i", "lam x. lam y. match lti x y with true then x else y",
     lambda: lam("x", "y", if_(lti("x", "y"), "x", "y")), "99", 99, "int", [17, 4, 42, 8, 23]),
    ("max_i", "lam x. lam y. match gti x y with true then x else y",
     lambda: lam("x", "y", if_(gti("x", "y"), "x", "y")), "0", 0, "int", [17, 4, 42, 8, 23]),
    ("sum_f", "addf", lambda: addf, "0.0", 0.0, "float", [0.5, 0.25, 0.125, 4.0]),
    ("max_f", "lam x. lam y. match gtf x y with true then x else y",
     lambda: lam("x", "y", if_(gtf("x", "y"), "x", "y")), "0.0", 0.0, "float", [1.5, -3.0, 2.25]),
    ("generic_i", "lam x. lam y. addi (addi x y) 0",
     lambda: lam("x", "y", addi(addi("x", "y"), 0)), "0", 0, "int", list(range(100))),
    ("empty_sum", "addi", lambda: addi, "7", 7, "int", []),
]

# foldl: sequential left fold, non-associative operators exercise the order
FOLD_CASES = [
    ("foldl_subi", "subi", lambda: subi, "100", 100, "int", [1, 2, 3, 4]),
    ("foldl_divf", "divf", lambda: divf, "1000.0", 1000.0, "float", [2.0, 5.0, 0.5]),
    ("foldl_poly", "lam a. lam x. addi (muli a 10) x", lambda: lam("a", "x", addi(muli("a", 10), "x")),
     "0", 0, "int", [1, 2, 3, 4, 5]),
    ("foldl_max_f", "lam a. lam x. match gtf x a with true then x else a",
     lambda: lam("a", "x", if_(gtf("x", "a"), "x", "a")), "0.0", 0.0, "float", [0.5, 2.5, 1.0]),
]

MAP2_CASES = [
    ("map2_mulf", "mulf", lambda: mulf, "float", [1.0, 2.0, 3.0], [4.0, 5.0, 6.0]),
    ("map2_affine", "lam x. lam o. addi (muli 3 x) o", lambda: lam("x", "o", addi(muli(3, "x"), "o")),
     "int", [1, 2, 3], [100, 200, 300]),
    ("map2_mismatch", "addi", lambda: addi, "int", [1, 2], [1]),
]

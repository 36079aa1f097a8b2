"""Recognition of the case-study accelerated bindings by the drop-in
(paper_2211_00621_b200/dropin_programs.py), on CPU: the reference compiles and
runs each golden program with a hook on pmx.interp.device_call that records
what the B200 drop-in would dispatch (nothing runs on a device here).  Needs
the reference (baseline/_ref or /root/reference)."""
import pathlib
import sys

import pytest

from conftest import GOLDEN

ROOT = pathlib.Path(__file__).resolve().parent.parent
REFS = [ROOT / "baseline" / "_ref", pathlib.Path("/root/reference/pkg/src")]
REF = next((p for p in REFS if (p / "pmx").exists()), None)
pytestmark = pytest.mark.skipif(REF is None, reason="reference package not available")


def _recognised(src: str):
    sys.path.insert(0, str(REF))
    import pmx
    import pmx.interp as interp
    import pmx.runtime as rt
    import pmx.syntax as syn
    from paper_2211_00621_b200 import dropin_programs as D
    seen = []
    orig = interp.device_call

    def hook(fn, args, ctx, span):
        h = D.recognise(fn, args, syn, rt)
        seen.append(h[0] if h else None)
        return orig(fn, args, ctx, span)
    interp.device_call = hook
    try:
        pmx.run_source(src, mode="accel", workers=2, capture_output=True)
    finally:
        interp.device_call = orig
    return seen


CASES = [("program_rk4", None, "rk4"), ("program_viterbi", None, "viterbi"), ("program_nn", None, "nn"),
         ("rk4_param", 0, "rk4"), ("rk4_param", 1, "rk4"), ("hmm_forward", 0, "hmm_forward"),
         ("hmm_forward", 2, "hmm_forward"), ("knn", 0, "knn"), ("knn", 2, "knn"), ("kmer", 0, "hmm_kmer"),
         ("kmer", 1, "hmm_kmer")]


@pytest.mark.parametrize("sec,i,family", CASES, ids=[f"{c[0]}{'' if c[1] is None else c[1]}" for c in CASES])
def test_case_study_bindings_are_recognised(sec, i, family):
    e = GOLDEN[sec] if i is None else GOLDEN[sec][i]
    assert _recognised(e["program"]) == [family]


def test_changed_model_constant_is_not_recognised():
    # the kernel hard-codes the pendulum's coefficients: a different model must
    # not be dispatched to it (it then takes the generic path)
    src = GOLDEN["program_rk4"]["program"].replace("9.81", "9.80")
    assert _recognised(src) == [None]


def test_other_programs_are_not_recognised():
    for name in ("dot_product", "nested_map", "loop_squares"):
        seen = _recognised(GOLDEN["corpus"][name]["program"])
        assert all(s is None for s in seen), (name, seen)


def test_knn_with_non_integer_coordinates_is_not_recognised():
    # fp32 distance ranking equals the reference's fp64 one only when every
    # distance is exact: fractional coordinates keep the generic path
    src = GOLDEN["knn"][0]["program"].replace("int2float (subi (modi (h (addi (muli p dim) i) 2654435761) 17) 8)",
                                              "divf (int2float (subi (modi (h (addi (muli p dim) i) 2654435761) 17) 8)) 3.0")
    assert src != GOLDEN["knn"][0]["program"]
    assert _recognised(src) == [None]

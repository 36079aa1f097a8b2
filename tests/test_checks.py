"""Assumption checks (paper §5.1): mirrors the reference's
tests/test_runtime.py:51-62 (check_regular / check_rank) and
tests/test_acceptance.py:288-301 (checks off by default, on demand, verdict
selection, configurable rank bound), against paper_2211_00621_b200.checks and
the accelerate entry point.  The raising cases fail before marshalling, so they
run without a GPU."""
import numpy as np
import pytest

from paper_2211_00621_b200 import Diagnostics
from paper_2211_00621_b200.checks import check_arg, check_rank, check_regular
from paper_2211_00621_b200.runtime import TensorView
from paper_2211_00621_b200 import skeletons as K


def test_check_regular():
    check_regular([[1, 2], [3, 4]])
    check_regular({"a": [[1], [2]], "b": 3})
    check_regular(np.zeros((3, 4)))
    with pytest.raises(Diagnostics, match="irregular"):
        check_regular([[1], [2, 3]])
    with pytest.raises(Diagnostics, match="irregular"):
        check_regular({"rows": [[[1, 2]], [[1], [2]]]})


def test_check_regular_path_in_message():
    with pytest.raises(Diagnostics, match=r"irregular sequence at argument\.rows: inner lengths \[1, 2\]"):
        check_regular({"rows": [[[1, 2]], [[1], [2, 3]]]})
    with pytest.raises(Diagnostics, match=r"irregular sequence at argument\.rows\[0\]: inner lengths \[1, 2\]"):
        check_regular({"rows": [[[1, 2], [3]], [[4], [5, 6]]]})


def test_check_rank():
    check_rank(TensorView(0, 0, (1, 2, 3), "int"), 3)
    with pytest.raises(Diagnostics, match="rank 4 exceeds bound 3"):
        check_rank(TensorView(0, 0, (1, 1, 1, 1), "int"), 3)


@pytest.mark.parametrize("verdict,irregular_raises,rank_raises", [
    (None, True, True),          # unknown backend: both checks
    ("futhark", True, False),    # Classification.FUTHARK -> check_regular
    ("cuda", False, True),       # Classification.CUDA -> check_ranks
    ("any", False, False),       # Classification.ANY -> no check (interp.py:223-227)
])
def test_check_arg_verdict_selection(verdict, irregular_raises, rank_raises):
    irregular = [[1], [2, 3]]
    rank4 = TensorView(0, 0, (1, 1, 1, 1), "int")
    if irregular_raises:
        with pytest.raises(Diagnostics, match="irregular sequence"):
            check_arg(irregular, 3, verdict)
    else:
        check_arg(irregular, 3, verdict)
    if rank_raises:
        with pytest.raises(Diagnostics, match="rank 4 exceeds bound 3"):
            check_arg([rank4], 3, verdict)
    else:
        check_arg([rank4], 3, verdict)
    check_arg([rank4], 4, verdict)   # the bound is configurable


def test_check_arg_accepts_reference_enum():
    import enum

    class Classification(enum.Enum):     # same member names as pmx/classify.py:22-26
        ANY = "Any"
        FUTHARK = "Futhark"
        CUDA = "CUDA"

    with pytest.raises(Diagnostics, match="irregular"):
        check_arg([[1], [2, 3]], 3, Classification.FUTHARK)
    check_arg([[1], [2, 3]], 3, Classification.CUDA)


def test_accelerate_runs_checks_on_demand():
    def body(s):
        return s
    with pytest.raises(Diagnostics, match="irregular sequence"):
        K.accelerate(body, [[1], [2, 3]], ctx=K.Ctx(checks=True))
    with pytest.raises(Diagnostics, match="irregular sequence"):
        K.accelerate(body, [[1], [2, 3]], ctx=K.Ctx(checks=True), verdict="futhark")


@pytest.mark.gpu
def test_accelerate_checks_off_by_default_gpu():
    # accel mode skips the checks by default: an irregular argument is
    # marshalled (offsets layout) and the body runs
    out = K.accelerate(lambda s: K.length(s), [[1], [2, 3], [4]])
    assert out == 3
    # a CUDA verdict does not look at regularity
    out = K.accelerate(lambda s: K.length(s), [[1], [2, 3], [4]], ctx=K.Ctx(checks=True), verdict="cuda")
    assert out == 3

import json
import math
import pathlib
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
sys.path.insert(0, str(ROOT / "oracle"))
sys.setrecursionlimit(100_000)

GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


def _cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return GOLDEN


def tokens(s: str) -> list:
    return s.split()


def parse_tokens(s: str) -> list:
    out = []
    for t in s.split():
        try:
            out.append(int(t))
        except ValueError:
            out.append(float(t))
    return out


def tokens_match(a: str, b: str, *, float_rel: float) -> bool:
    """tests/conftest.py:21-38 of the reference: token-wise, floats by rel tol."""
    ta, tb = a.split(), b.split()
    if len(ta) != len(tb):
        return False
    for x, y in zip(ta, tb):
        try:
            fx, fy = float(x), float(y)
        except ValueError:
            if x != y:
                return False
            continue
        if "." in x or "e" in x or "." in y or "e" in y:
            if not math.isclose(fx, fy, rel_tol=float_rel, abs_tol=float_rel):
                return False
        elif x != y:
            return False
    return True

"""Runtime assumption checks (§5.1 of the paper), run on the host before
marshalling when `Ctx(checks=True)` — mirrors pmx/runtime.py:115-138 and
pmx/interp.py:223-227 (`_check_arg`).  The reference picks the check by the
binding's backend verdict (Classification.FUTHARK -> regular sequences,
Classification.CUDA -> tensor rank <= max_rank); `check_arg` does the same when
given a verdict ("futhark" / "cuda", or the reference's enum member) and
applies both when the verdict is unknown (None)."""
from __future__ import annotations

import numpy as np

from .diagnostics import runtime_error
from .runtime import TensorView, collect_tensors


def check_regular(value, path: str = "argument") -> None:
    """Nested sequences must have uniform inner lengths (runtime.py:115-127)."""
    if isinstance(value, np.ndarray):
        return                          # numpy arrays are regular by construction
    if isinstance(value, list):
        lengths = {len(v) for v in value if isinstance(v, (list, np.ndarray))}
        if len(lengths) > 1:
            raise runtime_error(f"irregular sequence at {path}: inner lengths {sorted(lengths)}")
        for i, v in enumerate(value):
            check_regular(v, f"{path}[{i}]")
    elif isinstance(value, dict):
        for label, v in value.items():
            check_regular(v, f"{path}.{label}")


def check_rank(t: TensorView, max_rank: int) -> None:
    if len(t.shape) > max_rank:
        raise runtime_error(f"tensor rank {len(t.shape)} exceeds bound {max_rank}")


def check_ranks(value, max_rank: int) -> None:
    for t in collect_tensors(value):
        check_rank(t, max_rank)


def _verdict_name(verdict) -> str | None:
    if verdict is None:
        return None
    name = getattr(verdict, "name", verdict)      # pmx.classify.Classification member or a string
    return str(name).lower()


def check_arg(value, max_rank: int, verdict=None) -> None:
    """`_check_arg(verdict, value, ctx)` (pmx/interp.py:223-227)."""
    v = _verdict_name(verdict)
    if v in (None, "futhark"):
        check_regular(value)
    if v in (None, "cuda"):
        check_ranks(value, max_rank)

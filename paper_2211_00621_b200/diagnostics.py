"""Error convention of the reference (pmx/syntax.py:382-405, pmx/runtime.py:20-21).

Runtime errors abort with `Diagnostics([Diagnostic("RuntimeError", msg, span)])`
and render as `<file>:<line>:<col>: RuntimeError: msg`.  Device kernels report
errors through a 64-bit error word; `raise_device_error` converts it into the
same exception, naming the first failing element.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional


@dataclass(frozen=True)
class Span:
    line: int = 0
    col: int = 0

    def __str__(self) -> str:
        return f"{self.line}:{self.col}"


NO_SPAN = Span()


@dataclass
class Diagnostic(Exception):
    kind: str
    message: str
    span: Span = NO_SPAN
    rule: Optional[str] = None

    def render(self, filename: str = "<input>") -> str:
        tag = f" [{self.rule}]" if self.rule else ""
        return f"{filename}:{self.span.line}:{self.span.col}:{tag} {self.kind}: {self.message}"

    def __str__(self) -> str:
        return self.render()


class Diagnostics(Exception):
    def __init__(self, items: list[Diagnostic]):
        super().__init__(f"{len(items)} diagnostic(s)")
        self.items = items

    def __str__(self) -> str:
        return "\n".join(str(d) for d in self.items)


def runtime_error(message: str, span: Span = NO_SPAN) -> Diagnostics:
    return Diagnostics([Diagnostic("RuntimeError", message, span)])


def device_error(word: int, span: Span = NO_SPAN, what: str = "element") -> Diagnostics:
    from ._lib import ERROR_MESSAGES
    code = word & 0xFF
    index = word >> 8
    msg = ERROR_MESSAGES.get(code, f"device error {code}")
    return runtime_error(f"{msg} (at {what} {index})", span)

"""CPU oracle executor — restates the reference harness call shape.

Every function cites the reference line it follows.  Test infrastructure
only (see oracle/__init__.py).
"""

from __future__ import annotations

import contextlib
import io
import itertools
import linecache
import logging
import sys
import types

import torch

FLOAT_RTOL = 1e-6   # runner.py:30
FLOAT_ATOL = 1e-7   # runner.py:31

_ids = itertools.count()


# runner.py:114-125 `_make_args` (manual_seed, then per arg a value tensor,
# uniform `rand*(hi-lo)+lo` or `randn`; BASELINE reshaping and dtype casts of
# the fp32 draws): ONE copy, the harness's — the draws are the harness call
# contract, not the computation under test, and tests/test_oracle.py pins them
# bit-exactly against the reference harness's own outputs
from paper_2509_16248_b200.harness import make_args  # noqa: E402,F401


def load_program(text: str, tag: str = "prog") -> types.ModuleType:
    """runner.py:105-111 `_load_module`, from source text instead of a path."""
    name = f"_gm_oracle_{tag}_{next(_ids)}"
    filename = f"<oracle:{name}>"
    linecache.cache[filename] = (len(text), None, text.splitlines(True), filename)
    module = types.ModuleType(name)
    module.__file__ = filename
    sys.modules[name] = module
    exec(compile(text, filename, "exec"), module.__dict__)
    return module


class _LogCapture(logging.Handler):
    """runner.py:128-135."""

    def __init__(self):
        super().__init__(level=logging.DEBUG)
        self.lines: list[str] = []

    def emit(self, record: logging.LogRecord) -> None:
        self.lines.append(record.getMessage())


@contextlib.contextmanager
def capture_side_effects():
    """runner.py:138-151: stdout text and root-logger lines around a call."""
    handler = _LogCapture()
    root = logging.getLogger()
    old_level = root.level
    root.addHandler(handler)
    root.setLevel(logging.DEBUG)
    buf = io.StringIO()
    try:
        with contextlib.redirect_stdout(buf):
            yield buf, handler
    finally:
        root.removeHandler(handler)
        root.setLevel(old_level)


def call_captured(fn, args):
    """runner.py:154-157: fn(*clones) with side effects captured; returns
    (result, stdout lines + log lines)."""
    with capture_side_effects() as (buf, handler):
        result = fn(*[a.clone() if isinstance(a, torch.Tensor) else a for a in args])
    return result, buf.getvalue().splitlines() + handler.lines


def diffs(a: torch.Tensor, b: torch.Tensor) -> tuple[float, float]:
    """runner.py:160-168: max abs / max rel difference in fp64."""
    if a.shape != b.shape:
        return float("inf"), float("inf")
    fa, fb = a.double(), b.double()
    abs_diff = (fa - fb).abs()
    denom = fa.abs().clamp_min(1e-12)
    return (float(abs_diff.max()) if abs_diff.numel() else 0.0,
            float((abs_diff / denom).max()) if abs_diff.numel() else 0.0)


def count_breaks(fn, args) -> int:
    """runner.py:171-177: graph splits reported by torch._dynamo.explain."""
    torch._dynamo.reset()
    explanation = torch._dynamo.explain(fn)(*[a.clone() if isinstance(a, torch.Tensor) else a for a in args])
    return explanation.graph_break_count


def reference_callable(text: str, callable_name: str, dtype: torch.dtype | None = None):
    """Load a transformed program and return its entry callable on CPU in
    `dtype` (modules are cast; functions take the cast inputs)."""
    mod = load_program(text, callable_name)
    fn = getattr(mod, callable_name)
    # a `@torch.compile`-decorated entry runs eagerly here, as the reference's
    # own equivalence tests do when Inductor is unavailable (TORCHDYNAMO_DISABLE)
    fn = getattr(fn, "_torchdynamo_orig_callable", fn)
    if dtype is not None and isinstance(fn, torch.nn.Module):
        fn.to(dtype)
    return fn


def run_reference(text: str, callable_name: str, args: list, dtype: torch.dtype | None = None):
    """The reference's hot path on CPU: (output, side-effect lines)."""
    fn = reference_callable(text, callable_name, dtype)
    return call_captured(fn, args)

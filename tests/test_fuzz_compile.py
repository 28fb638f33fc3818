"""The randomised programs of tests/test_gpu_fuzz.py on the CPU: every region
of every program is specialised for its recorded arguments (split into side
and main kernels where it mixes iteration spaces, split.py), generated and
compiled for sm_100a with NVRTC — the code-generation half of the fuzzer,
without a GPU."""

import pytest
import torch

from paper_2509_16248_b200 import _native as nat
from paper_2509_16248_b200 import codegen, lowering
from paper_2509_16248_b200.ir import Unsupported, fold_host_predicates
from paper_2509_16248_b200.rowgen import RowPlan, has_row_ops
from paper_2509_16248_b200.split import is_mixed, split
from test_gpu_fuzz import CASES, _program


def _plans(graph, outs, args, depth=0):
    """The kernels a region specialises into for `args` (mirrors
    region._SplitSpec / _Spec, CPU tensors allowed)."""
    if not is_mixed(graph, outs, args):
        cls = RowPlan if has_row_ops(outs) else codegen.Plan
        return [cls(graph, outs, args, "fuzz", allow_cpu=True)]
    steps, (mg, mouts) = split(graph, outs, args)
    ext, res = list(args), []
    for sg, souts, _idx in steps:
        res += _plans(sg, souts, ext, depth + 1)
        ext.append(torch.empty(tuple(souts[0].shape), dtype=souts[0].dtype))
    return res + _plans(mg, mouts, ext, depth + 1)


def _sample():
    """A dozen programs (NVRTC takes seconds per program): those holding the
    row-statistics forms (layer_norm / var / std / softmax) first, both
    dtypes."""
    keys = ("layer_norm(", ".std(", ".var(", "softmax(")
    rows = [c for c in CASES if any(k in _program(c[0], True) for k in keys)]
    rest = [c for c in CASES if c not in rows]
    return rows[::3][:9] + rest[::17][:3]


SAMPLE = _sample()


@pytest.mark.parametrize("seed,dtype,shape", SAMPLE, ids=[f"s{c[0]}-{str(c[1])[6:]}" for c in SAMPLE])
def test_random_program_compiles(seed, dtype, shape):
    text = _program(seed, rows=True)
    torch.manual_seed(seed)
    x = torch.randn(shape).to(dtype)
    y = torch.randn(shape[-1]).to(dtype) if seed % 2 else torch.randn(shape).to(dtype)
    b = torch.randn(shape[-1]).to(dtype)
    mod, low = lowering.load(text, allow_eager=True)
    for r in low.regions:
        r.trace = []
    mod.f(x, y, b)
    n = 0
    for r in low.regions:
        assert r.trace, (r.name, text)
        args = list(r.trace[0])
        try:
            graph, outs = fold_host_predicates(r.graph, r.out_nodes, args)
        except Unsupported as exc:
            pytest.fail(f"{r.name}: {exc}\n{text}")
        for p in _plans(graph, outs, args):
            assert len(nat.compile_cubin(p.source, (10, 0))) > 0
            n += 1
    assert n >= len(low.regions)

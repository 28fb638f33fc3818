"""torch.compile front door: `torch.compile(model, backend="gm_b200")` on a
GraphMend-transformed program lowers Dynamo's FX graphs into fused regions
(paper_2509_16248_b200/dynamo.py)."""

import functools

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import dynamo  # noqa: F401  (registers the backend)
from paper_2509_16248_b200.harness import make_args
from parity import assert_parity


def _callable(prog):
    ns = {}
    exec(compile(prog["transformed"], prog["callable"], "exec"), ns)
    return ns[prog["callable"]]


@pytest.mark.parametrize("name", ["phi4_like", "qwen_audio_like", "blenderbot_like", "bigbird_like"])
def test_backend_on_cpu_equals_eager(programs, name):
    """On CPU tensors the lowered FX graph runs its statements eagerly:
    bit-identical to the uncompiled transformed program (bigbird_like: a
    module whose Linear parameters Dynamo lifts into graph inputs)."""
    torch._dynamo.reset()
    prog = programs[name]
    fn = _callable(prog)
    shapes = [[1, 64, 768]] if name == "bigbird_like" else None
    for spec in prog["inputs"]:
        args = make_args(spec["args"], spec["seed"], shapes=shapes)
        ref = fn(*[a.clone() for a in args])
        out = torch.compile(fn, backend=functools.partial(dynamo.gm_b200_backend, allow_eager=True))(
            *[a.clone() for a in args])
        assert torch.equal(out, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name,dtype", [("bigbird_like", torch.bfloat16), ("phi4_like", torch.float32),
                                        ("qwen_audio_like", torch.bfloat16)])
def test_backend_on_b200(programs, name, dtype):
    """On the B200 the FX graph runs as fused regions inside a CUDA graph and
    matches the reference's CPU eager execution of the same program."""
    torch._dynamo.reset()
    prog = programs[name]
    shapes = None if name == "bigbird_like" else [[8, 1024, 768]]
    fn = _callable(prog)
    if isinstance(fn, torch.nn.Module):
        fn.to("cuda", dtype)
    compiled = torch.compile(fn, backend="gm_b200")
    from paper_2509_16248_b200 import _native as nat

    for spec in prog["inputs"]:
        args = make_args(spec["args"], spec["seed"], dtype, shapes)
        ref, _ = orc.run_reference(prog["transformed"], prog["callable"], args, dtype)
        c0 = nat.launch_count
        out = compiled(*[a.cuda() for a in args])
        assert_parity(out, ref, dtype, what=name)
        assert nat.launch_count > c0 or spec is not prog["inputs"][0], "no fused region launched"


@pytest.mark.gpu
def test_branch_select_custom_op():
    """torch.ops.gm.branch_select (the precompiled phi4 block) in eager and
    under torch.compile (fake implementation for tracing)."""
    torch.manual_seed(0)
    x = torch.randn(8, 1024, 768, device="cuda") + 0.01
    ref = torch.where(x.sum() > 0, x * 1.0 + 1.0, x * 1.0 - 1.0)
    out = torch.ops.gm.branch_select(x, 0, 0, 0.0, 1.0, 1.0, 1.0, -1.0)
    assert torch.equal(out, ref)
    f = torch.compile(lambda t: torch.ops.gm.branch_select(t, 0, 0, 0.0, 1.0, 1.0, 1.0, -1.0) * 2, backend="gm_b200",
                      fullgraph=True)
    assert torch.equal(f(x), ref * 2)

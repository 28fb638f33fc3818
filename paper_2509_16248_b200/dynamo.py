"""torch.compile front door.

`gm_b200_backend` is a Dynamo backend: `torch.compile(model,
backend="gm_b200")` on a GraphMend-transformed module hands each captured FX
graph here.  After the reference's rewrite those graphs contain exactly the
vocabulary the fused regions implement — predicate reductions, arm
arithmetic, `torch.where` selects — plus library calls (Linear / matmul)
that stay on cuBLAS.  The graph's own Python source (`GraphModule.code`) is
lowered by the same path as a transformed program (lowering.load): maximal
runs of fusable statements become sm_100a region kernels, the rest stays
PyTorch, and the forward is wrapped in a B200Executor (one CUDA graph per
input signature, no host sync inside).  Parameters lifted into graph inputs
are read in place, not copied per call.

`torch.ops.gm.branch_select` is the precompiled canonical predicated block
(gm_branch_select_f32: `red(x) cmp thr ? a1*x + b1 : a2*x + b2`) as a
torch.library custom op with a fake implementation, so it traces.
"""

from __future__ import annotations

import ctypes
import functools
import textwrap

import torch

from . import _native as nat
from .executor import B200Executor
from .lowering import load
from .region import RegionUnsupported

_PRELUDE = "import math\nimport operator\nimport torch\n\n"


def gm_b200_backend(gm: torch.fx.GraphModule, example_inputs, allow_eager: bool = False,
                    static_outputs: bool = False):
    """Dynamo backend: lower the FX graph's source into fused regions and run
    it as one CUDA graph per input signature.

    torch.compile semantics are kept: every call returns fresh tensors (the
    graph's static outputs are cloned unless `static_outputs=True`, the
    make_graphed_callables contract), and a call that needs autograd (grad
    mode on and an input requiring grad) runs the FX graph itself, so
    gradients flow — the fused kernels are inference-only.  CPU inputs raise
    unless `allow_eager` (then the lowered statements run eagerly with
    PyTorch, bit-identical to the graph): there is no silent CPU path.
    `functools.partial(gm_b200_backend, allow_eager=True)` opts in."""
    module, lowered = load(_PRELUDE + textwrap.dedent(gm.code), allow_eager=allow_eager)
    forward = functools.partial(module.forward, gm)
    on_cuda = any(torch.is_tensor(a) and a.is_cuda for a in example_inputs)
    if not on_cuda:
        if not allow_eager:
            raise RegionUnsupported("gm_b200 backend: no CUDA input (the B200 path has no CPU fallback; "
                                    "use functools.partial(gm_b200_backend, allow_eager=True) to run the lowered "
                                    "statements eagerly)")
        return forward
    dev = next(a.device for a in example_inputs if torch.is_tensor(a) and a.is_cuda)
    executor = B200Executor(forward, dev)
    stats = {"graph_calls": 0, "autograd_calls": 0}

    def run(*args):
        if torch.is_grad_enabled() and any(torch.is_tensor(a) and a.requires_grad for a in args):
            stats["autograd_calls"] += 1
            return gm(*args)
        stats["graph_calls"] += 1
        with torch.no_grad():
            out = executor(*args)
        if not static_outputs:
            out = torch.utils._pytree.tree_map(lambda t: t.clone() if torch.is_tensor(t) else t, out)
        executor.flush()
        return out

    run.executor = executor
    run.lowered = lowered
    run.stats = stats
    return run


try:  # `torch.compile(model, backend="gm_b200")`
    from torch._dynamo import register_backend

    register_backend(name="gm_b200")(gm_b200_backend)
except Exception:  # pragma: no cover - an older / newer Dynamo without the registry
    pass


@torch.library.custom_op("gm::branch_select", mutates_args=())
def branch_select(x: torch.Tensor, red: int, cmp: int, thr: float, a1: float, b1: float, a2: float,
                  b2: float) -> torch.Tensor:
    """`torch.where(x.<red>() <cmp> thr, a1*x + b1, a2*x + b2)` for an fp32
    CUDA tensor in one launch (red: 0 sum, 1 mean, 2 max, 3 min, 4 norm;
    cmp: 0 >, 1 >=, 2 <, 3 <=) — transform.py:359-376 on the phi4 block shape.
    Raises NativeError without the library; there is no fallback."""
    if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()):
        raise ValueError("gm::branch_select takes a contiguous fp32 CUDA tensor")
    lib = nat.lib()
    nat.init(x.device.index if x.device.index is not None else torch.cuda.current_device())
    out = torch.empty_like(x)
    scratch = torch.zeros(lib.gm_branch_select_scratch_bytes(), dtype=torch.uint8, device=x.device)
    nat.count_launches()
    nat.check(lib.gm_branch_select_f32(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), x.numel(),
                                       red, cmp, thr, a1, b1, a2, b2, ctypes.c_void_p(scratch.data_ptr()), None,
                                       ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)),
              "gm_branch_select_f32")
    return out


@branch_select.register_fake
def _(x, red, cmp, thr, a1, b1, a2, b2):
    return torch.empty_like(x)

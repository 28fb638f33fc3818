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

_PRELUDE = "import math\nimport operator\nimport torch\n\n"


def gm_b200_backend(gm: torch.fx.GraphModule, example_inputs):
    """Dynamo backend: lower the FX graph's source into fused regions and run
    it as one CUDA graph per input signature (CPU inputs run the lowered
    statements eagerly, bit-identical to the graph)."""
    module, lowered = load(_PRELUDE + textwrap.dedent(gm.code))
    forward = functools.partial(module.forward, gm)
    on_cuda = any(torch.is_tensor(a) and a.is_cuda for a in example_inputs)
    if not on_cuda:
        return forward
    dev = next(a.device for a in example_inputs if torch.is_tensor(a) and a.is_cuda)
    executor = B200Executor(forward, dev)

    def run(*args):
        with torch.no_grad():
            out = executor(*args)
        executor.flush()
        return out

    run.executor = executor
    run.lowered = lowered
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

"""B200-native execution path for GraphMend-transformed PyTorch programs.

GraphMend (arXiv 2509.16248) rewrites graph breaks at the source level: a
tensor-dependent `if` becomes `torch.where` over both arms and `print` /
`logger.*` calls are deferred to the epilogue (reference:
pkg/src/graphmend/transform.py).  Its transform API — source in, rewritten
source and graph-break counts out — is used unchanged.  This package is what
runs the rewritten program on a B200:

    lowered module  = lowering.load(transformed_text)      # regions + replay sites
    forward         = getattr(lowered_module, "model")     # as in the manifest
    executor        = B200Executor(forward)                # one CUDA graph per shape
    out             = executor(x)                          # no host sync inside
    executor.flush()                                       # deferred prints / logs

See DESIGN.md for the kernels and INTEGRATION.md for the C ABI binding.
"""

from __future__ import annotations

from .executor import B200Executor, count_syncs
from .lowering import Lowered, load, lower

__all__ = ["B200Executor", "Lowered", "count_syncs", "load", "lower", "compile_program"]


def compile_program(text: str, callable_name: str, device=None, dtype=None, use_graphs: bool = True,
                    allow_eager: bool = False):
    """Lower `text` (a GraphMend-transformed program), move its callable to
    the GPU and wrap it in a B200Executor.  Returns (executor, module, lowered).
    A region the fused kernels cannot run raises region.RegionUnsupported
    unless `allow_eager` (then it runs its statements with PyTorch)."""
    import torch

    module, lowered = load(text, allow_eager=allow_eager)
    fn = getattr(module, callable_name)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if isinstance(fn, torch.nn.Module):
        fn.to(dev)
        if dtype is not None:
            fn.to(dtype)
    return B200Executor(fn, dev, use_graphs=use_graphs), module, lowered

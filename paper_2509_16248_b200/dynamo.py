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

import ast
import functools
import gc
import os
import textwrap

import torch

from .executor import B200Executor
from .lowering import load
from .region import RegionUnsupported, check_status

_PRELUDE = "import math\nimport operator\nimport torch\n\n"
OUTPUT_SLOTS = 2   # captured copies whose outputs are handed out without a copy (GM_OUTPUT_SLOTS)


def gm_b200_backend(gm: torch.fx.GraphModule, example_inputs, allow_eager: bool = False,
                    static_outputs: bool = False):
    """Dynamo backend: lower the FX graph's source into fused regions and run
    it as one CUDA graph per input signature.

    torch.compile semantics are kept.  Every call returns tensors no later
    call overwrites: the outputs of one of OUTPUT_SLOTS captured copies that
    nothing the caller holds still references (checked before the replay,
    by storage use count), else copies (`static_outputs=True` returns the
    graph's static outputs, the make_graphed_callables contract).  A call
    that needs autograd (grad mode on and an input requiring grad) runs the
    FX graph itself, so
    gradients flow — the fused kernels are inference-only.  CPU inputs raise
    unless `allow_eager` (then the lowered statements run eagerly with
    PyTorch, bit-identical to the graph): there is no silent CPU path.
    `functools.partial(gm_b200_backend, allow_eager=True)` opts in."""
    module, lowered = load(_PRELUDE + _fx_source(gm), allow_eager=allow_eager)
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

    tree_flatten = torch.utils._pytree.tree_flatten
    use_count = torch._C._storage_Use_Count
    n_slots = int(os.environ.get("GM_OUTPUT_SLOTS", OUTPUT_SLOTS))
    held: dict[int, list] = {}   # id(slot entry) -> [(static output, storage use count with no alias out)]
    stats["aliased"] = stats["cloned"] = 0

    def slot_entry(args):
        """The first output slot (a captured copy of this signature's entry)
        none of whose outputs, nor views of them, the caller still holds —
        storage use counts back at the entry's own, checked BEFORE the replay
        that would overwrite them (the test cudagraph trees use) — or None
        when every slot is held."""
        for s in range(1, n_slots + 1):
            e = executor.prepare(*args, slot=s)
            h = held.get(id(e))
            if h is None:
                gc.collect()   # the capture's reference cycles: steady baseline counts
                leaves = tree_flatten(e.outputs)[0] if e.graph is not None else []
                h = held[id(e)] = [(t, use_count(t.untyped_storage()._cdata)) for t in leaves if torch.is_tensor(t)]
            if all(use_count(t.untyped_storage()._cdata) == n for t, n in h):
                return e
        return None

    def run(*args):
        if torch.is_grad_enabled():
            if any(torch.is_tensor(a) and a.requires_grad for a in args):
                stats["autograd_calls"] += 1
                return gm(*args)
            with torch.no_grad():
                return run(*args)
        stats["graph_calls"] += 1
        if static_outputs:
            out = executor(*args)
        else:
            check_status()
            e = slot_entry(args)
            if e is not None:
                e.load(args)
                stats["aliased"] += 1
                # aliases (new tensor objects on the static storage): while
                # the caller keeps one, or a view of one, the slot is held
                out = _map_tensors(torch.Tensor.detach, e.run())
            else:
                # every slot's outputs are still held: replay the scratch
                # entry (slot 0) and hand out copies
                stats["cloned"] += 1
                out = _map_tensors(torch.Tensor.clone, executor(*args))
        executor.flush()
        return out

    run.executor = executor
    run.lowered = lowered
    run.stats = stats
    return run


def _map_tensors(fn, out):
    """fn over the tensors of an output structure (Dynamo graphs return a
    tuple of tensors: mapped without pytree)."""
    if type(out) is tuple:
        return tuple(fn(t) if isinstance(t, torch.Tensor) else t for t in out)
    if isinstance(out, torch.Tensor):
        return fn(out)
    return torch.utils._pytree.tree_map(lambda t: fn(t) if isinstance(t, torch.Tensor) else t, out)


def _fx_source(gm: torch.fx.GraphModule) -> str:
    """The graph's Python source as the lowering wants it.  Traced with
    `capture_scalar_outputs` / `capture_dynamic_output_shape_ops` (gm_compile)
    the graph keeps `.item()` and nonzero / unique / masked_select inside, with
    runtime asserts on the unbacked sizes (`_assert_scalar(sym_size(v) >= 0)`):
    those are dropped (the lowering gives every such value a fixed shape, so
    no size is ever unbacked), dead size computations are eliminated, and the
    `v = None` frees FX emits are removed — they would read as rebindings."""
    g = gm.graph
    changed = False
    for node in list(g.nodes):
        if node.op == "call_function" and node.target in (torch.ops.aten._assert_scalar.default,
                                                          getattr(torch.ops.aten, "_assert_async", None)):
            g.erase_node(node)
            changed = True
    if changed:
        g.eliminate_dead_code()
        gm.recompile()
    tree = ast.parse(textwrap.dedent(gm.code))

    class _Frees(ast.NodeTransformer):
        def visit_Assign(self, node):
            if isinstance(node.value, ast.Constant) and node.value.value is None \
                    and all(isinstance(t, ast.Name) for t in node.targets):
                return None
            return node

    tree = ast.fix_missing_locations(_Frees().visit(tree))
    return ast.unparse(tree) + "\n"


def gm_compile(model, **kwargs):
    """`torch.compile(model, backend="gm_b200")` traced so that GraphMend's
    residual breaks do not split the graph: `.item()` reads and dynamic-shape
    ops (the reference reports them unfixable, analysis.py:597-605,
    data/dynamic_shape_ops.cfg) are captured into the FX graph, where the
    lowering turns them into device scalars and fixed-shape reductions
    (SURVEY §8f ranks 1-2).  The whole forward is then one FX graph, one
    CUDA graph, no host sync — as on the direct path (compile_program)."""
    # Dynamo reads these when it traces (first call, recompiles); set once,
    # process-wide, rather than entering a config patch on every call (a
    # per-call patch costs more than the whole forward of small programs)
    torch._dynamo.config.capture_scalar_outputs = True
    torch._dynamo.config.capture_dynamic_output_shape_ops = True
    return torch.compile(model, backend="gm_b200", **kwargs)


try:  # `torch.compile(model, backend="gm_b200")`
    from torch._dynamo import register_backend

    register_backend(name="gm_b200")(gm_b200_backend)
except Exception:  # pragma: no cover - an older / newer Dynamo without the registry
    pass


_RED = ("sum", "mean", "max", "min", "norm")
_CMP = (">", ">=", "<", "<=")
_bs_programs: dict = {}


def _branch_select_program(red: int, cmp: int):
    """The canonical predicated block as a transformed program (the shape
    transform.py:359-376 emits), lowered once per (red, cmp) into one fused
    region: the same codegen and kernels as every other region, any fusable
    dtype, and barrier scratch per (stream, graph) — nothing allocated or
    zeroed per call."""
    key = (red, cmp)
    if key not in _bs_programs:
        text = ("import torch\n\ndef branch_select(x, thr, a1, b1, a2, b2):\n"
                f"    __gm_pred_0 = x.{_RED[red]}() {_CMP[cmp]} thr\n"
                "    __gm_then_y_0 = x * a1 + b1\n    __gm_else_y_0 = x * a2 + b2\n"
                "    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)\n    return y\n")
        mod, low = load(text)
        _bs_programs[key] = (mod.branch_select, low)
    return _bs_programs[key]


@torch.library.custom_op("gm::branch_select", mutates_args=())
def branch_select(x: torch.Tensor, red: int, cmp: int, thr: float, a1: float, b1: float, a2: float,
                  b2: float) -> torch.Tensor:
    """`torch.where(x.<red>() <cmp> thr, a1*x + b1, a2*x + b2)` for a CUDA
    tensor of any fusable dtype (fp32 / bf16 / fp16) in ONE fused region
    launch (red: 0 sum, 1 mean, 2 max, 3 min, 4 norm; cmp: 0 >, 1 >=, 2 <,
    3 <=) — transform.py:359-376 on the phi4 block shape.  Raises for CPU
    tensors (no fallback) and NativeError without the library."""
    if not x.is_cuda:
        raise ValueError("gm::branch_select takes a CUDA tensor (the B200 path has no CPU fallback)")
    if not (0 <= red < len(_RED) and 0 <= cmp < len(_CMP)):
        raise ValueError("gm::branch_select: red in 0..4, cmp in 0..3")
    fn, _ = _branch_select_program(red, cmp)
    return fn(x, float(thr), float(a1), float(b1), float(a2), float(b2))


@branch_select.register_fake
def _(x, red, cmp, thr, a1, b1, a2, b2):
    return torch.empty_like(x)


@torch.library.custom_op("gm::log_capture", mutates_args=())
def log_capture(t: torch.Tensor, record_id: int) -> None:
    """Capture the elements of `t` its repr would print into the device log
    ring as record `record_id` (gm_logring_capture): one gather kernel, no
    device-to-host read inside the forward; the drain delivers the record to
    the handler registered with logring.on_record(record_id, fn).  Inside a
    B200Executor forward the record joins that forward's step (and its CUDA
    graph); a bare call opens and commits a one-record step.  Registered as
    an ORDERED effectful op, so a Dynamo-traced graph keeps it in place
    (replaces the replay of a deferred print, transform.py:707-708)."""
    if not t.is_cuda:
        raise ValueError("gm::log_capture takes a CUDA tensor")
    from . import logring

    ring = logring.active_ring()
    if ring is not None and ring.active:
        ring.capture(t, record_id)
        return
    ring = logring.ring_for(t.device)
    ring.begin()
    ring.capture(t, record_id)
    ring.enqueue(ring.end())


@log_capture.register_fake
def _(t, record_id):
    return None


try:
    from torch._higher_order_ops.effects import _EffectType, _register_effectful_op

    _register_effectful_op(torch.ops.gm.log_capture.default, _EffectType.ORDERED)
except Exception:  # pragma: no cover - API moved
    pass

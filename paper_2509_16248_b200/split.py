"""Regions whose statements run over more than one iteration space.

A run of fusable statements may mix shapes: a predicate over a `[C]` bias
(`p = b.sum() > 0`) guarding full `[B, L, C]` arms, a `[C]`-shaped value
returned beside the activations, a softmax over one tensor and a reduction
over another.  One grid-stride or row kernel covers one iteration space, so
such a region is specialised as a short sequence of kernels:

  * the main space M is the largest (by element count) among the non-alias
    elementwise outputs and the row operands (with scalar outputs only, the
    largest reduction operand);
  * every reduction, row operator or output over another shape is a *side*
    computation: its cone (everything it reads, back to the region's free
    values) becomes its own region graph — split again recursively if it
    mixes shapes itself — and runs first;
  * the main graph reads each side result as one more free value (a 0-d
    tensor for a reduction, a tensor of its shape otherwise).

A side cone reads only the region's free values, never the main kernel's
results, so the sides can always run first; nodes a side shares with the
main cone are recomputed (they are pure).  Every kernel is an ordinary
specialised region (codegen.Plan / rowgen.RowPlan); the sequence is stream-
ordered and graph-capturable like a single launch.  Found by the randomised
differential test (tests/test_gpu_fuzz.py): a quarter of its random
programs mixed a `[C]` input into full-shape regions.
"""

from __future__ import annotations

import math

import torch

from .ir import REDUCE, ROW_OPS, ROW_RED, FreeVar, Graph, Node, Unsupported, infer, topo


def _numel(shape) -> int:
    return math.prod(shape) if shape else 1


def sinks(outputs: list[Node]) -> list[tuple[Node, tuple]]:
    """(node, iteration shape) for every node that defines an iteration
    space: reductions and row operators (their operand's shape) and the
    non-alias elementwise outputs (their own shape)."""
    res = []
    for n in topo(outputs):
        if n.op in REDUCE or n.op in ROW_OPS:
            res.append((n, tuple(n.args[0].shape)))
    for o in outputs:
        if o.kind == "elem" and o.op != "free" and o.op not in ROW_RED:
            res.append((o, tuple(o.shape)))
    return res


def main_shape(outputs: list[Node]) -> tuple | None:
    """Where the main kernel writes: the largest elementwise output or row
    operand; with scalar outputs only, the largest reduction operand.  (A
    reduction over a larger space than the outputs becomes a side, so a side
    graph never re-elects the shape its own output was split off from.)"""
    written = [s for n, s in sinks(outputs) if n.op not in REDUCE]
    if written:
        return max(written, key=_numel)
    # scalar outputs only: the reductions that produce them directly (through
    # scalar arithmetic, not through another reduction's operand) — so a side
    # split off for its own reduction is the main kernel of its graph
    direct, seen, stack = [], set(), list(outputs)
    while stack:
        n = stack.pop()
        if n.uid in seen:
            continue
        seen.add(n.uid)
        if n.op in REDUCE:
            direct.append(tuple(n.args[0].shape))
            continue
        if n.kind != "elem":
            stack.extend(n.args)
    shapes = direct or [s for _, s in sinks(outputs)]
    if not shapes:
        return None
    return max(shapes, key=_numel)


def is_mixed(graph: Graph, outputs: list[Node], args: list) -> bool:
    infer(graph, args, outputs)
    shapes = {s for _, s in sinks(outputs)}
    return len(shapes) > 1


def _copy(graph: Graph, roots: list[Node], replace: dict[int, Node], nfree: int) -> tuple[Graph, list[Node]]:
    """A new graph holding the cones of `roots`; nodes in `replace` (by
    uid) become the given new free nodes.  The original frees keep their
    indices 0..nfree-1."""
    g = Graph()
    memo: dict[int, Node] = {}
    for fv in graph.frees:
        nn = g.add(Node("free", value=fv.node.value))
        g.frees.append(FreeVar(fv.text, nn))
        memo[fv.node.uid] = nn
    extra = {}
    for uid, (idx, text) in replace.items():
        nn = g.add(Node("free", value=idx))
        g.frees.append(FreeVar(text, nn))
        extra[uid] = nn

    def cp(n: Node) -> Node:
        if n.uid in extra:
            return extra[n.uid]
        if n.uid in memo:
            return memo[n.uid]
        r = g.add(Node(n.op, tuple(cp(a) for a in n.args), value=n.value))
        memo[n.uid] = r
        return r

    outs = [cp(r) for r in roots]
    return g, outs


def split(graph: Graph, outputs: list[Node], args: list, depth: int = 0):
    """[(side graph, side outputs, index its result takes in the extended
    argument list)] + (main graph, main outputs): the sides to run first, in
    order, and the main graph over the extended arguments."""
    if depth > 8:
        raise Unsupported("shape split too deep")
    infer(graph, args, outputs)
    M = main_shape(outputs)
    nfree = len(args)
    sides = []
    replace: dict[int, tuple] = {}
    for node, shape in sinks(outputs):
        if shape == M or node.uid in replace:
            continue
        if node.op in ROW_OPS and node.op not in ROW_RED and node.kind == "elem" and tuple(node.shape) == M:
            continue
        idx = nfree + len(sides)
        replace[node.uid] = (idx, f"__gm_side_{idx}")
        sides.append(node)
    if not sides:
        return [], (graph, outputs)
    steps = []
    for i, node in enumerate(sides):
        sg, souts = _copy(graph, [node], {}, nfree)
        steps.append((sg, souts, nfree + i))
    mg, mouts = _copy(graph, outputs, replace, nfree)
    return steps, (mg, mouts)

"""Region specialisation and CUDA code generation (sm_100a, via NVRTC).

Given a region DAG (ir.py) and the runtime arguments, `Plan` decides

  * the iteration space S (the common shape of the elementwise outputs and
    of every reduction operand) and how each input is read (full, periodic,
    strided broadcast, or scalar);
  * the passes: a reduction whose operand needs only scalars known before
    pass p runs in pass p; an elementwise output is stored in the first pass
    where all its scalars are known.  A predicated block is one reduction
    pass plus one select pass (transform.py:386-388 then :374-376);
  * speculation (`spec`): when every reduction-derived scalar the later
    passes read is a boolean branch decision, the kernel runs one pass under
    the previous launch's decisions, verifies them after one grid reduce and
    falls back to the exact passes in the same launch;
  * monotone hoisting (`_hoist`): a max/min of `Y * s`, `Y + s`, `Y - s` is
    taken from max/min(Y) at an earlier grid reduce, guarded on the device;
  * guards: an elementwise node that feeds only one side of a `where` with a
    uniform (scalar) predicate is evaluated under that predicate, so the
    untaken arm costs nothing — the reference evaluates both arms eagerly
    (transform.py:404-412), which is equivalent because arms are pure;
  * the launch layout (`_plan_layout`): 2 CTAs x 512 threads per SM over a
    grid-stride vector map, every load of a register block issued first, and
    register or thread-private shared-memory staging of inputs that exact
    later passes re-read;

and `_emit()` writes the kernel on top of csrc/gm_region.cuh.

Numerics follow torch's CPU eager kernels (the reference executes the
transformed program eagerly on CPU, runner.py:154-157), measured in this
repo's tests: one rounding per operator to the result dtype; Python scalars
are rounded to the tensor dtype for add/sub/compare/clamp but kept in fp32
for mul/div; `s / x` is `s * reciprocal(x)`; mean = (float)sum / N rounded
once; reductions accumulate in fp32 per thread and fp64 across threads.
"""

from __future__ import annotations

import hashlib
import math
import os
import re
from dataclasses import dataclass, field

import torch

from . import _native as nat
from .ir import (BOOL_AND, BOOL_NOT, BOOL_OR, COMPARE, INT_REDUCE, ITEM, NZSUM, REDUCE, Graph, Node, Unsupported,
                 infer, is_fusable_dtype, topo)

DT_CODE = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2, torch.bool: 4}
DT_SIZE = {torch.float32: 4, torch.bfloat16: 2, torch.float16: 2, torch.bool: 1}
RED_OP = {"sum": 0, "mean": 0, "norm": 0, "count_nonzero": 0, "nzsum": 0, "amax": 1, "amin": 2, "prod": 3,
          "argmax": 6, "argmin": 6,
          "any": 4, "all": 5}

MODE_FULL, MODE_PERIODIC, MODE_STRIDED, MODE_SCALAR = "full", "periodic", "strided", "scalar"

STATIC_SMEM_RESERVE = 8 * 1024
SMEM_PER_SM = 233472    # B200: 228 KB of shared memory per SM (shared by its resident CTAs)
B200_DEVICE = (148, 232448)  # SMs, opt-in dynamic shared memory per block
DATA_REGS = 40  # raw-vector registers per thread: register stage + one block's loads (GM_DATA_REGS)


def _data_regs() -> int:
    return int(os.environ.get("GM_DATA_REGS", DATA_REGS))
VEC_REGS = {torch.float32: 8, torch.bfloat16: 4, torch.float16: 4, torch.bool: 2}
MAX_DECISIONS = 24      # predicted decisions per speculative region (scratch ints at barrier + 288)
# adaptive speculation: speculate once the confidence counter reaches
# SPEC_CONFIDENT (two launches in a row that repeated their decisions)
SPEC_CONFIDENT = int(os.environ.get("GM_SPEC_CONFIDENT", "2"))
SPEC_CONF_MAX = 3


def _round_f(dtype) -> str:
    """Float-code rounding wrapper for a result dtype."""
    if dtype == torch.bfloat16:
        return "gm::rbf"
    if dtype == torch.float16:
        return "gm::rh"
    return ""


def _round_d(dtype) -> str:
    """Double-code rounding to a scalar dtype."""
    if dtype == torch.float32:
        return "(double)(float)"
    if dtype == torch.bfloat16:
        return "gm::rbf_d"
    if dtype == torch.float16:
        return "gm::rh_d"
    if dtype == torch.bool:
        return "gm_bool"
    if dtype in (torch.int64, torch.int32, torch.int16, torch.int8, torch.uint8):
        return "gm_trunc"
    return ""  # Python float/int/bool host values: double


def _fl(v: float) -> str:
    """Exact float literal."""
    f = float(v)
    if math.isnan(f):
        return "__int_as_float(0x7fc00000)"
    if math.isinf(f):
        return "__int_as_float(0x7f800000)" if f > 0 else "__int_as_float(0xff800000)"
    return f"{f!r}"


@dataclass
class InputPlan:
    free_index: int
    node: Node
    mode: str
    dtype: torch.dtype
    slot: int              # index into P.in
    passes: set = field(default_factory=set)


class Plan:
    """One specialisation of a region for concrete argument types/shapes."""

    def __init__(self, graph: Graph, outputs: list[Node], args: list, name: str = "region",
                 device_info: tuple[int, int] = B200_DEVICE, allow_cpu: bool = False):
        self.device_info = device_info
        self.allow_cpu = allow_cpu
        self.graph = graph
        self.outputs = outputs
        self.name = name
        infer(graph, args, outputs)
        self.order = topo(outputs)
        # host scalars exactly representable in bf16 (part of the region key)
        self.host_exact = {n.uid: self._bf16_exact(args[n.value]) for n in self.order
                           if n.op == "free" and n.kind == "host"}
        self._classify(args)
        self._passes()
        self._inputs(args)
        self._hoist()
        self.source = self._emit()
        digest = hashlib.sha1(self.source.encode()).hexdigest()[:16]
        self.kernel = f"gm_region_{digest}"
        self.source = self.source.replace("GM_KERNEL_NAME", self.kernel)

    # -- classification -----------------------------------------------------
    def _classify(self, args) -> None:
        elem_roots = [o for o in self.outputs if o.kind == "elem" and o.op != "free"]  # (free: an alias)
        red_nodes = [n for n in self.order if n.op in REDUCE]
        for n in red_nodes:
            if n.args[0].kind != "elem":
                raise Unsupported("reduction of a scalar")
        shapes = {o.shape for o in elem_roots} | {n.args[0].shape for n in red_nodes}
        if len(shapes) > 1:
            raise Unsupported(f"outputs/reductions disagree on shape: {shapes}")
        self.shape = next(iter(shapes)) if shapes else ()
        self.n = math.prod(self.shape) if shapes else 0
        if self.n >= 2 ** 32 and any(n.op in ("argmax", "argmin") for n in red_nodes):
            raise Unsupported("argmax/argmin keys carry a 32-bit index")
        read = {a.uid for n in self.order for a in n.args}
        for node in self.order:
            if node.op == "free" and node.uid not in read:
                continue  # only passed through as an output alias
            if node.kind == "elem":
                if not is_fusable_dtype(node.dtype):
                    raise Unsupported(f"elementwise dtype {node.dtype}")
                try:
                    ok = tuple(torch.broadcast_shapes(node.shape, self.shape)) == tuple(self.shape)
                except RuntimeError:
                    ok = False
                if not ok:
                    raise Unsupported("node does not broadcast to the iteration space")
            elif node.kind == "dscalar":
                if node.dtype not in (torch.float32, torch.bfloat16, torch.float16, torch.bool, torch.int64,
                                      torch.int32):
                    raise Unsupported(f"scalar dtype {node.dtype}")
        for o in self.outputs:
            if o.kind == "host":
                raise Unsupported("host-only output")
            if o.kind == "elem" and o.op != "free" and tuple(o.shape) != tuple(self.shape):
                raise Unsupported("output shape differs from the iteration space")
        for node in self.order:
            if node.op == "free" and node.kind == "elem":
                t = args[node.value]
                if t.device.type != "cuda" and not self.allow_cpu:
                    raise Unsupported("tensor not on a CUDA device")

    # -- passes ---------------------------------------------------------------
    def _passes(self) -> None:
        avail: dict[int, int] = {}   # scalar node -> level it becomes known
        need: dict[int, int] = {}    # elem node -> pass it can run in
        for node in self.order:
            if node.kind == "elem":
                need[node.uid] = max(
                    [need[a.uid] if a.kind == "elem" else avail[a.uid] for a in node.args] or [0]
                )
            elif node.op in REDUCE:
                avail[node.uid] = need[node.args[0].uid] + 1
            else:  # host / dscalar
                avail[node.uid] = max([avail[a.uid] if a.kind != "elem" else 0 for a in node.args] or [0])
                if any(a.kind == "elem" for a in node.args):
                    raise Unsupported("scalar computed from an elementwise value without reduction")
        self.avail, self.need = avail, need
        self.reductions = [n for n in self.order if n.op in REDUCE]
        npass = 0
        for o in self.outputs:
            if o.kind == "elem" and o.op != "free":
                npass = max(npass, need[o.uid] + 1)
        for r in self.reductions:
            npass = max(npass, avail[r.uid])
        self.npass = npass
        self.pass_outputs = {p: [] for p in range(npass)}
        for j, o in enumerate(self.outputs):
            if o.kind == "elem" and o.op != "free":
                self.pass_outputs[need[o.uid]].append((j, o))
        self.pass_reds = {p: [r for r in self.reductions if need[r.args[0].uid] == p] for p in range(npass)}
        if len(self.reductions) > nat.MAX_RED:
            raise Unsupported("too many reductions in one region")
        # scalar slots
        self.scalars = [n for n in self.order if n.kind in ("host", "dscalar") and n.op != "const"]
        self.slot = {n.uid: i for i, n in enumerate(self.scalars)}

    # -- monotone reduction hoisting -----------------------------------------------
    def _hoist(self) -> None:
        """A max/min in pass p >= 1 of `E = Y ⋈ s` (⋈ in *, +, -; Y an
        elementwise value of an earlier pass q; s a scalar first known at
        level p) equals E's own elementwise code applied to max(Y) or min(Y):
        each such E is monotone in Y (direction from the sign of s for *),
        and rounding to the storage type is monotone too.  So pass q also
        reduces max(Y) and min(Y), and at level p — when s is known — the
        statistic is computed from them.  The exact sweep of pass p runs only
        when the guard fails: s, max(Y) or min(Y) not finite (NaN or inf
        would break the identity), checked on the device, uniform across
        CTAs.  Applied to a pass only when every reduction in it qualifies
        and it stores no output (longformer_like: 3 sweeps -> 2)."""
        self.hoisted: dict[int, list] = {}
        if os.environ.get("GM_HOIST", "1") == "0" or self.npass < 2:
            return
        aux = self.graph.__dict__.setdefault("_gm_aux", {})
        plans = {}
        for p in range(1, self.npass):
            reds = self.pass_reds[p]
            if not reds or self.pass_outputs[p]:
                continue
            items = []
            for r in reds:
                e = r.args[0]
                if r.op not in ("amax", "amin") or e.op not in ("mul", "add", "sub") or not e.dtype.is_floating_point:
                    break
                elem = [a for a in e.args if a.kind == "elem"]
                scal = [a for a in e.args if a.kind != "elem"]
                if len(elem) != 1 or len(scal) != 1 or elem[0].dtype != e.dtype:
                    break
                y, s = elem[0], scal[0]
                if self.need[y.uid] >= p or s.op == "const":
                    break
                if self._guard_expr(self._guards(p).get(e.uid, frozenset({frozenset()}))):
                    break
                # monotone direction: +1 increasing in Y, -1 decreasing, 0 = sign of s
                if e.op == "mul":
                    direction = 0
                elif e.op == "add":
                    direction = 1
                else:
                    direction = 1 if e.args[0] is y else -1
                items.append((r, e, y, s, direction))
            else:
                plans[p] = items
        if not plans:
            return
        for p, items in plans.items():
            for r, e, y, s, direction in items:
                ext = []
                for op in ("amax", "amin"):
                    key = (y.uid, op)
                    n = aux.get(key)
                    if n is None:
                        n = self.graph.add(Node(op, (y,)))
                        aux[key] = n
                    if n not in self.reductions:
                        v = y.meta.max() if op == "amax" else y.meta.min()
                        n.meta, n.kind, n.dtype, n.shape = v, "dscalar", v.dtype, ()
                        self.reductions.append(n)
                        q = self.need[y.uid]
                        self.pass_reds[q].append(n)
                        self.avail[n.uid] = q + 1
                        self.slot[n.uid] = len(self.scalars)
                        self.scalars.append(n)
                    ext.append(n)
                self.hoisted.setdefault(p, []).append((r, e, y, s, direction, ext[0], ext[1]))
        if len(self.reductions) > nat.MAX_RED:
            raise Unsupported("too many reductions in one region")

    def _emit_hoist_guard(self, w, p: int) -> None:
        """Thread 0, at scalar level p: decide whether pass p can be skipped
        and, if so, fill its statistics from the hoisted max/min."""
        items = self.hoisted[p]
        w(f"  __shared__ int s_hoist{p};")
        w("  if (threadIdx.x == 0) {")
        conds = []
        for r, e, y, s, d, hmax, hmin in items:
            for n in (s, hmax, hmin):
                v = self._sv(n)
                conds.append(f"(({v}) - ({v}) == 0.0)")  # finite
        w(f"    const int ok_ = ({' && '.join(conds)}) ? 1 : 0;")
        w(f"    s_hoist{p} = ok_;")
        w("    if (ok_) {")
        for r, e, y, s, d, hmax, hmin in items:
            want_max = r.op == "amax"
            if d == 0:
                inc = f"({self._sv(s)} >= 0.0)"
            else:
                inc = "true" if d > 0 else "false"
            pick_max = f"({inc} ? {'1' if want_max else '0'} : {'0' if want_max else '1'})"
            w("      {")
            w(f"        const double yx_ = {pick_max} ? {self._sv(hmax)} : {self._sv(hmin)};")
            w(f"        float n{y.uid}_h[GM_VEC];")
            w(f"        for (int l = 0; l < GM_VEC; ++l) n{y.uid}_h[l] = (float)yx_;")
            w(f"        const float sf{s.uid} = (float){self._sv(s)}; (void)sf{s.uid};")
            w(f"        float n{e.uid}_h[GM_VEC];")
            for line in self._elem_code(e, "h"):
                w("        " + line.replace("\n", "\n        "))
            w(f"        s_scal[{self.slot[r.uid]}] = (double)n{e.uid}_h[0];")
            w("      }")
        w("    }")
        w("  }")
        w("  __syncthreads();")

    # -- inputs ---------------------------------------------------------------
    def _inputs(self, args) -> None:
        self.inputs: list[InputPlan] = []
        self.host_frees: list[Node] = []
        used_passes: dict[int, set] = {}
        for p in range(self.npass):
            for node in self._pass_nodes(p):
                if node.op == "free" and node.kind == "elem":
                    used_passes.setdefault(node.uid, set()).add(p)
        for node in self.order:
            if node.op != "free":
                continue
            if node.kind == "host":
                self.host_frees.append(node)
        if len(self.host_frees) > nat.MAX_HS:
            raise Unsupported("too many host scalars")
        read = {a.uid for n in self.order for a in n.args}
        for node in self.order:
            if node.op == "free" and node.kind in ("elem", "dscalar") and node.uid in read:
                t = args[node.value]
                if node.kind == "dscalar":
                    mode = MODE_SCALAR
                else:
                    mode = self._mode(t)
                self.inputs.append(InputPlan(node.value, node, mode, t.dtype, len(self.inputs),
                                             passes=used_passes.get(node.uid, set())))
        # periods of the periodic inputs, fixed per specialisation (the
        # kernel divides by a constant)
        self._periods = {ip.slot: args[ip.free_index].numel() for ip in self.inputs if ip.mode == MODE_PERIODIC}
        if len(self.inputs) > nat.MAX_IN:
            raise Unsupported("too many tensor inputs")
        elem_out = [o for o in self.outputs if o.kind == "elem" and o.op != "free"]
        scal_out = [o for o in self.outputs if o.kind == "dscalar"]
        if len(elem_out) + len(scal_out) > nat.MAX_OUT:
            raise Unsupported("too many outputs")
        self.in_by_uid = {ip.node.uid: ip for ip in self.inputs}

    def _mode(self, t: torch.Tensor) -> str:
        S = tuple(self.shape)
        if t.numel() == 1:
            return MODE_SCALAR
        if tuple(t.shape) == S and t.is_contiguous() and t.data_ptr() % 16 == 0:
            return MODE_FULL
        # periodic: contiguous tensor equal to S's trailing dims (leading 1s)
        shp = list(t.shape)
        while shp and shp[0] == 1:
            shp.pop(0)
        if t.is_contiguous() and shp and tuple(shp) == S[len(S) - len(shp):] and t.data_ptr() % 16 == 0:
            return MODE_PERIODIC
        return MODE_STRIDED

    # -- guards -----------------------------------------------------------------
    def _pass_roots(self, p: int) -> list[Node]:
        return [o for _, o in self.pass_outputs[p]] + [r.args[0] for r in self.pass_reds[p]]

    def _pass_nodes(self, p: int) -> list[Node]:
        return self._nodes(self._pass_roots(p))

    def _guards(self, p: int) -> dict[int, frozenset]:
        return self._guards_roots(self._pass_roots(p))

    def _nodes(self, roots: list[Node]) -> list[Node]:
        """Elementwise nodes a sweep over `roots` evaluates (scalars come
        from s_scal, so the traversal stops at them)."""
        seen: set[int] = set()
        order: list[Node] = []

        def visit(n: Node) -> None:
            if n.uid in seen or n.kind != "elem":
                return
            seen.add(n.uid)
            for a in n.args:
                visit(a)
            order.append(n)

        for r in roots:
            visit(r)
        return order

    def _guards_roots(self, roots: list[Node]) -> dict[int, frozenset]:
        """DNF guard per elementwise node of a sweep over `roots`: a set of
        conjunctions of (scalar-node uid, polarity) literals."""
        TRUE = frozenset()
        dnf: dict[int, set] = {}

        def add(node: Node, conj: frozenset) -> bool:
            cur = dnf.setdefault(node.uid, set())
            if any(d <= conj for d in cur):
                return False
            for d in [d for d in cur if conj < d]:
                cur.discard(d)
            cur.add(conj)
            # resolution: X+{c} and X+{!c} -> X
            changed = True
            while changed:
                changed = False
                for a in list(cur):
                    for lit in a:
                        b = (a - {lit}) | {(lit[0], not lit[1])}
                        if b in cur:
                            cur.discard(a)
                            cur.discard(b)
                            merged = a - {lit}
                            if not any(d <= merged for d in cur):
                                cur.add(merged)
                            changed = True
                            break
                    if changed:
                        break
            return True

        work = [(r, TRUE) for r in roots]
        while work:
            node, conj = work.pop()
            if node.kind != "elem":
                continue
            if not add(node, conj):
                continue
            if node.op == "where" and node.args[0].kind != "elem":
                c = node.args[0]
                work.append((node.args[1], conj | {(c.uid, True)}))
                work.append((node.args[2], conj | {(c.uid, False)}))
            else:
                for a in node.args:
                    work.append((a, conj))
        return {uid: frozenset(v) for uid, v in dnf.items()}

    # -- emission ---------------------------------------------------------------
    def _sv(self, node: Node) -> str:
        """Scalar value (double expression) of a host/dscalar/const node."""
        if node.op == "const":
            v = node.value
            return "1.0" if v is True else ("0.0" if v is False else _fl(v))
        return f"s_scal[{self.slot[node.uid]}]"

    def _sf(self, node: Node) -> str:
        """Scalar value as a float local inside a pass."""
        if node.op == "const":
            v = node.value
            return "1.f" if v is True else ("0.f" if v is False else f"((float){_fl(v)})")
        return f"sf{node.uid}"

    def _ev(self, node: Node, lane: str, u: int) -> str:
        if node.kind == "elem":
            return f"n{node.uid}_{u}[{lane}]"
        return self._sf(node)

    def _scalar_operand(self, s: Node, op: str, res_dtype, operand_index: int) -> str:
        """torch CPU treatment of a scalar operand of an elementwise op."""
        v = self._sf(s)
        r = _round_f(res_dtype)
        if op in ("mul",):
            return v
        if op == "div":
            return v  # divisor stays fp32 (x / s == x / float(s)); dividend case handled by caller
        return f"{r}({v})" if r else v

    def _elem_code(self, node: Node, u: int) -> list[str]:
        L = "l"
        dst = f"n{node.uid}_{u}[{L}]"
        R = _round_f(node.dtype) if node.dtype != torch.bool else ""
        if getattr(self, "_no_round", False):
            R = ""
        a = node.args
        op = node.op

        def ev(x: Node, i: int = 0) -> str:
            if x.kind == "elem":
                return self._ev(x, L, u)
            return self._scalar_operand(x, op, node.dtype, i)

        def wrap(expr: str) -> str:
            return f"{R}({expr})" if R else expr

        if op == "free":
            ip = self.in_by_uid[node.uid]
            dt = DT_CODE[ip.dtype]
            k = ip.slot
            if ip.mode == MODE_FULL:
                if self._tail:
                    return [f"gm::load8_gmem<{dt}>(P.in[{k}], e{u}, nv{u}, n{node.uid}_{u});"]
                pre, raw = self._raw_for(ip, u)
                return pre + [f"gm::rcvt<{dt}>({raw}, n{node.uid}_{u});"]
            if ip.mode == MODE_PERIODIC:
                per = getattr(self, "_periods", {}).get(k)
                if per and not os.environ.get("GM_PERIODIC_RUNTIME"):
                    return [f"gm::load8_periodic_c<{dt}, {per}ll>(P.in[{k}], e{u}, nv{u}, n{node.uid}_{u});"]
                return [f"gm::load8_periodic<{dt}>(P.in[{k}], e{u}, nv{u}, n{node.uid}_{u});"]
            if ip.mode == MODE_STRIDED:
                return [f"gm::load8_strided<{dt}>(P.in[{k}], e{u}, nv{u}, n{node.uid}_{u});"]
            return [f"#pragma unroll\nfor (int l = 0; l < GM_VEC; ++l) n{node.uid}_{u}[l] = sin{k};"]
        body: str
        if op in ("add", "sub", "mul"):
            fn = {"add": "gm::add", "sub": "gm::sub", "mul": "gm::mul"}[op]
            body = wrap(f"{fn}({ev(a[0], 0)}, {ev(a[1], 1)})")
        elif op == "div":
            if a[0].kind != "elem" and a[1].kind == "elem":
                # s / x == s * reciprocal(x), reciprocal rounded to the dtype
                rr = _round_f(a[1].dtype if a[1].dtype != torch.bool else node.dtype)
                rec = f"gm::recip({self._ev(a[1], L, u)})"
                rec = f"{rr}({rec})" if rr else rec
                body = wrap(f"gm::mul({rec}, {self._sf(a[0])})")
            elif a[1].op == "const" and self._pow2_recip(a[1].value) is not None:
                # x / 2^k == x * 2^-k exactly (both are the correctly rounded x*2^-k)
                body = wrap(f"gm::mul({ev(a[0], 0)}, {_fl(self._pow2_recip(a[1].value))}f)")
            else:
                body = wrap(f"gm::div({ev(a[0], 0)}, {ev(a[1], 1)})")
        elif op == "pow":
            base = ev(a[0], 0)
            if a[1].op == "const" and a[0].kind == "elem":
                ex = float(a[1].value)
                special = {
                    2.0: f"gm::mul({base}, {base})",
                    3.0: f"gm::mul(gm::mul({base}, {base}), {base})",
                    0.5: f"gm::fsqrt({base})",
                    -0.5: f"gm::recip(gm::fsqrt({base}))",
                    1.0: f"{base}",
                    -1.0: f"gm::recip({base})",
                    -2.0: f"gm::recip(gm::mul({base}, {base}))",
                    0.0: "1.f",
                }
                body = wrap(special.get(ex, f"powf({base}, {_fl(ex)}f)"))
            else:
                body = wrap(f"powf({ev(a[0], 0)}, {ev(a[1], 1)})")
        elif op in COMPARE:
            cmpd = torch.result_type(a[0].meta, a[1].meta)
            rc = _round_f(cmpd)

            def cv(x: Node) -> str:
                s = self._ev(x, L, u) if x.kind == "elem" else self._sf(x)
                return f"{rc}({s})" if (rc and x.kind != "elem") else s

            sym = {"gt": ">", "ge": ">=", "lt": "<", "le": "<=", "eq": "==", "ne": "!="}[op]
            body = f"(({cv(a[0])} {sym} {cv(a[1])}) ? 1.f : 0.f)"
        elif op in ("maximum", "minimum"):
            fn = "gm::nmax" if op == "maximum" else "gm::nmin"
            body = wrap(f"{fn}({ev(a[0], 0)}, {ev(a[1], 1)})")
        elif op in ("floordiv", "mod", "fmod"):
            if not node.dtype.is_floating_point:
                raise Unsupported(f"{op} on {node.dtype}")
            fn = {"floordiv": "gm::floordiv", "mod": "gm::pymod", "fmod": "fmodf"}[op]
            body = wrap(f"{fn}({ev(a[0], 0)}, {ev(a[1], 1)})")
        elif op == "logical_and":
            body = f"((({ev(a[0])}) != 0.f && ({ev(a[1])}) != 0.f) ? 1.f : 0.f)"
        elif op == "logical_or":
            body = f"((({ev(a[0])}) != 0.f || ({ev(a[1])}) != 0.f) ? 1.f : 0.f)"
        elif op == "logical_not":
            body = f"((({ev(a[0])}) == 0.f) ? 1.f : 0.f)"
        elif op == "where":
            if a[0].kind != "elem":
                return self._uniform_select(node, u)
            body = wrap(f"(({self._ev(a[0], L, u)}) != 0.f ? {ev(a[1], 1)} : {ev(a[2], 2)})")
        elif op == "clamp":
            has_lo, has_hi = node.value
            x = ev(a[0])
            i = 1
            if has_lo:
                x = f"gm::nmax({x}, {ev(a[i], i)})"
                i += 1
            if has_hi:
                x = f"gm::nmin({x}, {ev(a[i], i)})"
            body = wrap(x)
        else:
            x = ev(a[0])
            un = {
                "neg": f"(-{x})", "pos": f"({x})", "abs": f"fabsf({x})", "relu": f"gm::relu({x})",
                "sigmoid": f"gm::sigmoid({x})", "tanh": f"tanhf({x})", "exp": f"expf({x})",
                "log": f"logf({x})", "sqrt": f"gm::fsqrt({x})", "rsqrt": f"gm::recip(gm::fsqrt({x}))",
                "sin": f"sinf({x})", "cos": f"cosf({x})", "silu": f"gm::silu({x})",
                "gelu": f"gm::gelu({x})", "gelu_tanh": f"gm::gelu_tanh({x})", "erf": f"erff({x})",
                "square": f"gm::mul({x}, {x})", "reciprocal": f"gm::recip({x})",
            }
            if op == "gelu" and node.dtype in (torch.bfloat16, torch.float16) and not os.environ.get("GM_ACCURATE_GELU16"):
                # 16-bit outputs: erf from an erfc fit with relative error
                # < 1.2e-7 on the SFU (gm::gelu16); the accurate erff made
                # the bf16 GELU region ALU-bound
                un["gelu"] = f"gm::gelu16({x})"
            if op not in un:
                raise Unsupported(f"codegen for {op}")
            body = wrap(un[op])
        return [f"#pragma unroll\nfor (int l = 0; l < GM_VEC; ++l) {dst.replace('[l]', '[l]')} = {body};"]

    def _uniform_select(self, node: Node, u: int) -> list[str]:
        c, ta, ea = node.args
        R = _round_f(node.dtype) if node.dtype != torch.bool else ""

        def val(x: Node) -> str:
            if x.kind == "elem":
                s = f"n{x.uid}_{u}[l]"
                # promote/round into the result dtype (exact when widening)
                return f"{R}({s})" if (R and x.dtype != node.dtype) else s
            s = self._sf(x)
            return f"{R}({s})" if R else s

        cond = f"sb{c.uid}"
        return [
            f"if ({cond}) {{\n#pragma unroll\nfor (int l = 0; l < GM_VEC; ++l) n{node.uid}_{u}[l] = {val(ta)};\n}} "
            f"else {{\n#pragma unroll\nfor (int l = 0; l < GM_VEC; ++l) n{node.uid}_{u}[l] = {val(ea)};\n}}"
        ]

    def _guard_expr(self, dnf: frozenset) -> str:
        if any(len(c) == 0 for c in dnf):
            return ""
        terms = []
        for conj in sorted(dnf, key=lambda c: sorted(c)):
            lits = [f"sb{uid}" if pol else f"!sb{uid}" for uid, pol in sorted(conj)]
            terms.append("(" + " && ".join(lits) + ")")
        return " || ".join(terms)

    def _scalar_code(self, node: Node) -> str:
        """Double-precision statement computing scalar slot of `node`."""
        slot = self.slot[node.uid]
        dst = f"s_scal[{slot}]"
        if node.op == "free":
            if node.kind == "host":
                j = self.host_frees.index(node)
                return f"{dst} = P.hs[{j}];"
            ip = self.in_by_uid[node.uid]
            if ip.dtype == torch.int64:
                return f"{dst} = (double)(*(const long long*)P.in[{ip.slot}].ptr);"
            if ip.dtype == torch.int32:
                return f"{dst} = (double)(*(const int*)P.in[{ip.slot}].ptr);"
            return f"{dst} = (double)gm::load_scalar<{DT_CODE[ip.dtype]}>(P.in[{ip.slot}]);"
        if node.op in REDUCE:
            raise AssertionError("reductions are finished by _finish_reduction")
        if node.op == ITEM:
            # the 0-d tensor's value as a Python number (exact in double)
            return f"{dst} = {self._sv(node.args[0])};"
        R = _round_d(node.dtype) if node.kind == "dscalar" else ""
        a = node.args
        op = node.op

        def sv(x: Node) -> str:
            return self._sv(x)

        if op in COMPARE:
            cmpd = torch.result_type(a[0].meta, a[1].meta) if any(torch.is_tensor(x.meta) for x in a) else None
            rc = _round_d(cmpd) if cmpd is not None else ""
            sym = {"gt": ">", "ge": ">=", "lt": "<", "le": "<=", "eq": "==", "ne": "!="}[op]
            l0 = f"{rc}({sv(a[0])})" if rc else sv(a[0])
            l1 = f"{rc}({sv(a[1])})" if rc else sv(a[1])
            return f"{dst} = (({l0}) {sym} ({l1})) ? 1.0 : 0.0;"
        if op in ("add", "sub", "mul", "div"):
            sym = {"add": "+", "sub": "-", "mul": "*", "div": "/"}[op]
            # operands are first converted to the common dtype
            if node.kind == "dscalar" and node.dtype in (torch.float32, torch.bfloat16, torch.float16):
                rcast = _round_d(node.dtype)
                e = f"({rcast}({sv(a[0])}) {sym} {rcast}({sv(a[1])}))"
            else:
                e = f"({sv(a[0])} {sym} {sv(a[1])})"
            return f"{dst} = {R}({e});" if R else f"{dst} = {e};"
        if op in ("floordiv", "mod", "fmod"):
            fn = {"floordiv": "gm::floordiv_t", "mod": "gm::pymod_t", "fmod": "fmod"}[op]
            if node.kind == "dscalar" and node.dtype == torch.float32:
                e = f"(double){fn.replace('_t', '')}((float){sv(a[0])}, (float){sv(a[1])})" if op != "fmod" \
                    else f"(double)fmodf((float){sv(a[0])}, (float){sv(a[1])})"
            else:
                e = f"{fn}({sv(a[0])}, {sv(a[1])})" if op == "fmod" else f"{fn}<double>({sv(a[0])}, {sv(a[1])})"
            return f"{dst} = {R}({e});" if R else f"{dst} = {e};"
        if op == "pow":
            e = f"pow({sv(a[0])}, {sv(a[1])})"
            return f"{dst} = {R}({e});" if R else f"{dst} = {e};"
        if op == "where":
            return f"{dst} = ({sv(a[0])} != 0.0) ? {R}({sv(a[1])}) : {R}({sv(a[2])});" if R else \
                f"{dst} = ({sv(a[0])} != 0.0) ? {sv(a[1])} : {sv(a[2])};"
        if op in ("maximum", "minimum"):
            fn = "gm::dmax" if op == "maximum" else "gm::dmin"
            return f"{dst} = {R}({fn}({sv(a[0])}, {sv(a[1])}));"
        if op in ("logical_and", BOOL_AND):
            return f"{dst} = ({sv(a[0])} != 0.0 && {sv(a[1])} != 0.0) ? 1.0 : 0.0;"
        if op in ("logical_or", BOOL_OR):
            return f"{dst} = ({sv(a[0])} != 0.0 || {sv(a[1])} != 0.0) ? 1.0 : 0.0;"
        if op in ("logical_not", BOOL_NOT):
            return f"{dst} = ({sv(a[0])} == 0.0) ? 1.0 : 0.0;"
        if op == "clamp":
            has_lo, has_hi = node.value
            x = sv(a[0])
            i = 1
            if has_lo:
                x = f"gm::dmax({x}, {sv(a[i])})"
                i += 1
            if has_hi:
                x = f"gm::dmin({x}, {sv(a[i])})"
            return f"{dst} = {R}({x});" if R else f"{dst} = {x};"
        x = sv(a[0])
        un = {
            "neg": f"(-{x})", "pos": f"({x})", "abs": f"fabs({x})", "relu": f"({x} > 0.0 ? {x} : 0.0)",
            "sigmoid": f"(double)gm::sigmoid((float){x})", "tanh": f"(double)tanhf((float){x})",
            "exp": f"(double)expf((float){x})", "log": f"(double)logf((float){x})",
            "sqrt": f"(double)gm::fsqrt((float){x})", "rsqrt": f"(double)gm::recip(gm::fsqrt((float){x}))",
            "sin": f"(double)sinf((float){x})", "cos": f"(double)cosf((float){x})",
            "silu": f"(double)gm::silu((float){x})", "square": f"({x} * {x})",
            "gelu": f"(double)gm::gelu((float){x})", "gelu_tanh": f"(double)gm::gelu_tanh((float){x})",
            "erf": f"(double)erff((float){x})",
            "reciprocal": f"(1.0 / {x})",
        }
        if op not in un:
            raise Unsupported(f"scalar codegen for {op}")
        return f"{dst} = {R}({un[op]});" if R else f"{dst} = {un[op]};"

    def _finish_reduction(self, r: Node, k: int) -> str:
        """Scalar slot of reduction `r` from the grid-reduced double s_red[k]."""
        dst = f"s_scal[{self.slot[r.uid]}]"
        R = _round_d(r.dtype)
        x = f"s_red[{k}]"
        if r.op == "mean":
            e = f"(double)__fdiv_rn((float){x}, (float){self.n}.0)"
            return f"{dst} = {R}({e});"
        if r.op == "norm":
            return f"{dst} = {R}((double)gm::fsqrt((float){x}));"
        if r.op in ("any", "all"):
            return f"{dst} = ({x} != 0.0) ? 1.0 : 0.0;"
        if r.op == "count_nonzero":
            return f"{dst} = {x};"
        if r.op in ("argmax", "argmin"):
            # index = ~(low word of the winning key)
            return (f"{dst} = (double)(0xffffffffu - (u32)((u64)__double_as_longlong({x}) & 0xffffffffull));")
        return f"{dst} = {R}({x});" if R else f"{dst} = {x};"

    # -- contexts ----------------------------------------------------------------
    # A context is one sweep over the iteration space: exact pass p (an int),
    # or "spec" — the speculative single pass that evaluates every pass's
    # roots under predicted decisions.
    def _ctx_roots(self, ctx) -> list[Node]:
        if ctx == "spec":
            roots: list[Node] = []
            for p in range(self.npass):
                roots += self._pass_roots(p)
            return roots
        return self._pass_roots(ctx)

    def _used_scalars(self, elem_nodes: list[Node], guards: dict) -> list[Node]:
        used: list[Node] = []
        for n in elem_nodes:
            for a in n.args:
                if a.kind != "elem" and a.op != "const" and a not in used:
                    used.append(a)
        for conj_set in guards.values():
            for conj in conj_set:
                for uid, _ in conj:
                    node = self.graph.nodes[uid]
                    if node not in used:
                        used.append(node)
        return used

    def _decisions(self) -> list[Node]:
        """Scalars computed from reductions (level >= 1) that elementwise code
        reads: the branch decisions a speculative pass predicts."""
        out: list[Node] = []
        for p in range(self.npass):
            roots = self._pass_roots(p)
            for s in self._used_scalars(self._nodes(roots), self._guards_roots(roots)):
                if self.avail.get(s.uid, 0) >= 1 and s not in out:
                    out.append(s)
        return out

    def _spec_ok(self) -> bool:
        if os.environ.get("GM_SPEC", "1") == "0":
            return False
        if not self.reductions or self.npass < 2 or not self.decisions or len(self.decisions) > MAX_DECISIONS:
            return False
        return all(d.dtype == torch.bool for d in self.decisions)

    # -- sampled branch prediction -------------------------------------------------------
    SAMPLE_SCALED = ("sum", "mean", "norm", "count_nonzero")
    SAMPLE_PLAIN = ("amax", "amin", "any", "all")

    def _cta_ok(self) -> bool:
        """Per-CTA prediction (GM_SAMPLE=cta; not the default): every CTA
        predicts the decisions from the first vector of each of its threads —
        data the speculative sweep has just loaded — so the prediction costs a
        CTA-wide combine, not a pass of its own.  CTAs may disagree; the grid
        reduce carries every decision's min and max over CTAs (and whether
        all certified), so all CTAs reach the same verdict."""
        # Measured slower than the sampled pass on every workload (the
        # CTA-wide combine inside the sweep waits for vector 0 of every warp
        # and adds registers; phi4's randn draw then mispredicts instead of
        # taking the exact entry): bigbird fp32 16.2 / 18.2 us per kernel vs
        # 15.1 / 16.0, qwen 19.7 vs 16.9 (profiles/r02_ab_prediction.jsonl).
        # Kept behind GM_SAMPLE=cta.
        if os.environ.get("GM_SAMPLE") != "cta" or self.vfull < 1:
            return False
        if not all(r.op in self.SAMPLE_SCALED + self.SAMPLE_PLAIN for r in self.reductions):
            return False
        return len(self.reductions) + 2 * len(self.decisions) + 1 <= nat.MAX_RED

    def extra_slots(self) -> int:
        """Grid-reduce slots beyond the reductions (per-CTA prediction)."""
        return 2 * len(self.decisions) + 1 if getattr(self, "cta_pred", False) else 0

    def _cta_predict_lines(self) -> list[str]:
        """Inside the speculative sweep's first register block, after its
        loads are issued: the region's decision chain evaluated on each
        thread's first vector (the loaded raw registers), combined CTA-wide,
        scaled to the whole space, certified (4 standard errors), and the
        decisions handed to the sweep through sb/sf."""
        L: list[str] = []
        w = L.append
        scale_base = float(self.n)
        w("{ // ---- per-CTA prediction from this CTA's first vectors")
        w("  const bool sok_ = ok0;")
        w("  const double cnt_ = 8.0 * (double)max(0ll, min((i64)GM_THREADS, VF_ - (i64)blockIdx.x * GM_THREADS));")
        w("  int cert_ = 1;")
        levels = []
        for p in range(self.npass):
            reds = list(self.pass_reds[p])
            feeds = [d for d in self.decisions if self.avail[d.uid] > p]
            if reds and feeds:
                levels.append((p, reds))
        done_free: set[int] = set()
        for p, reds in levels:
            roots = [r.args[0] for r in reds]
            nodes = self._nodes(roots)
            guards = self._guards_roots(roots)
            w(f"  {{ // level {p}")
            for n in nodes:
                if n.op == "free" and n.uid in done_free:
                    continue
                w(f"  float n{n.uid}_q[GM_VEC];")
            cur = None
            for n in nodes:
                g = self._guard_expr(guards.get(n.uid, frozenset({frozenset()})))
                if g != cur:
                    if cur:
                        w("  }")
                    if g:
                        w(f"  if ({g}) {{")
                    cur = g
                if n.op == "free":
                    ip = self.in_by_uid[n.uid]
                    dt = DT_CODE[ip.dtype]
                    if ip.mode == MODE_SCALAR:
                        w(f"  for (int l = 0; l < GM_VEC; ++l) n{n.uid}_q[l] = sin{ip.slot};")
                    elif ip.mode == MODE_FULL and ip.slot in self._preloaded:
                        w(f"  gm::rcvt<{dt}>({self._preloaded[ip.slot].format(u=0)}, n{n.uid}_q);")
                    else:
                        fn = {MODE_FULL: "load8_gmem", MODE_PERIODIC: "load8_periodic"}.get(ip.mode, "load8_strided")
                        w(f"  gm::{fn}<{dt}>(P.in[{ip.slot}], e0, sok_ ? GM_VEC : 0, n{n.uid}_q);")
                    continue
                for line in self._elem_code(n, "q"):
                    w("  " + line.replace("\n", "\n  "))
            if cur:
                w("  }")
            for r in reds:
                k = self.red_index[r.uid]
                x = f"n{r.args[0].uid}_q"
                op = RED_OP[r.op]
                if r.op in self.SAMPLE_SCALED:
                    term = {"count_nonzero": f"(({x}[l] != 0.f) ? 1.0 : 0.0)",
                            "norm": f"((double){x}[l] * (double){x}[l])"}.get(r.op, f"(double){x}[l]")
                    w(f"  double t{k}_ = 0.0, q{k}_ = 0.0;")
                    w(f"  if (sok_) for (int l = 0; l < GM_VEC; ++l) {{ const double z_ = {term}; t{k}_ += z_; q{k}_ += z_ * z_; }}")
                    w(f"  gm::cta_sum2(t{k}_, q{k}_, s_w_);")
                    w(f"  if (threadIdx.x == 0) {{ s_red[{k}] = t{k}_ * ({scale_base!r} / fmax(cnt_, 1.0)); "
                      f"s_m1_[{k}] = t{k}_; s_m2_[{k}] = q{k}_; }}")
                else:
                    w(f"  const float a{k}_ = gm::acc8({op}, gm::acc_identity({op}), {x}, sok_ ? GM_VEC : 0);")
                    w(f"  const double v{k}_ = gm::cta_combine({op}, (double)a{k}_, s_w_);")
                    w(f"  if (threadIdx.x == 0) s_red[{k}] = v{k}_;")
            w("  if (threadIdx.x == 0) {")
            for r in reds:
                w("    " + self._finish_reduction(r, self.red_index[r.uid]))
            for n in self.scalars:
                if self.avail[n.uid] == p + 1 and n.op not in REDUCE:
                    w("    " + self._scalar_code(n))
            for j, d in enumerate(self.decisions):
                if self.avail[d.uid] != p + 1:
                    continue
                w(f"    s_pred[{j}] = (s_scal[{self.slot[d.uid]}] != 0.0) ^ ((s_force_ >> {j}) & 1);")
                form = self._simple_decision(d)
                if form is not None and form[0].op in self.SAMPLE_SCALED:
                    r, cmp, c, _left = form
                    k = self.red_index[r.uid]
                    est = f"s_scal[{self.slot[r.uid]}]"
                    w("    {")
                    w(f"      const double n_ = fmax(cnt_, 1.0), mu_ = s_m1_[{k}] / n_, "
                      f"var_ = fmax(s_m2_[{k}] / n_ - mu_ * mu_, 0.0);")
                    w("      double se_ = sqrt(var_ / n_);")
                    if r.op in ("sum", "count_nonzero"):
                        w(f"      se_ *= {float(self.n)!r};")
                    elif r.op == "norm":
                        w(f"      se_ = se_ * {float(self.n)!r} / (2.0 * fmax({est}, 1e-30));")
                    w(f"      if (!(fabs({est} - ({self._sv(c)})) > 4.0 * se_)) cert_ = 0;")
                    w("    }")
            w("    s_cert_ = cert_;")
            w("  }")
            w("  __syncthreads();")
            for j, d in enumerate(self.decisions):
                if self.avail[d.uid] == p + 1:
                    w(f"  sb{d.uid} = s_pred[{j}] != 0; sf{d.uid} = sb{d.uid} ? 1.f : 0.f;")
            w("  }")
        w("}")
        return L

    def _sample_ok(self) -> bool:
        """Can every predicted decision be estimated from a sample?  Sums,
        means, norms and counts scale with the sampled fraction; max / min /
        any / all are taken over the sample as they are.  prod, argmax /
        argmin and coordinate sums have no useful sample estimate: such
        regions keep the last launch's decisions as their prediction."""
        if os.environ.get("GM_SAMPLE", "1") == "0" or self.vfull < 1:
            return False
        if not all(r.op in self.SAMPLE_SCALED + self.SAMPLE_PLAIN for r in self.reductions):
            return False
        # The sample pass costs ~2 us at the kernel front.  It pays where the
        # exact entry is expensive: chains of decisions (>= 3 passes: qwen
        # 36 -> 25 us, phi4 53 -> 40 us per forward under rotating inputs)
        # and fp32 predicated blocks (bigbird 224 -> 219 us); a 2-pass 16-bit
        # block's exact entry is within ~1.5 us of its speculative hit, so it
        # keeps the history predictor (profiles/r02_ab_sampling*.jsonl)
        if os.environ.get("GM_SAMPLE") == "always":
            return True
        return self.npass >= 3 or any(DT_SIZE.get(ip.dtype, 2) >= 4 for ip in self.inputs if ip.mode == MODE_FULL)

    def _simple_decision(self, d: Node):
        """(reduction, comparison, other operand, reduction on the left) when
        decision `d` is a reduction compared with a host / constant scalar
        (the transform's `__gm_pred_k = P.red() ⋈ c`), else None."""
        if d.op not in ("gt", "ge", "lt", "le") or len(d.args) != 2:
            return None
        a, b = d.args
        if a.op in REDUCE and b.kind == "host":
            return a, d.op, b, True
        if b.op in REDUCE and a.kind == "host":
            return b, d.op, a, False
        return None

    def _emit_sample(self, w) -> None:
        """Predict the decisions from a sample, inside every CTA, before
        anything else (no grid barrier): the CTA evaluates the exact passes'
        reductions over the same GM_THREADS vectors of the iteration space —
        vector (t * 2654435761) mod VF_ for thread t, a golden-ratio scramble
        that spreads the sample over rows and columns — combines them
        CTA-wide, scales sums / counts by n / n_sampled, and runs the scalar
        levels on the estimates.  Every CTA computes the same sample, so all
        agree on the prediction.  The speculative sweep then verifies the
        prediction exactly; a wrong one costs the restart, never a wrong
        result.  Inputs whose decisions change from launch to launch (the
        bench rotates three draws whose decisions differ) are predicted from
        their own data instead of from the previous launch."""
        nsamp = min(self.vfull, self.threads)
        scale = float(self.n) / float(nsamp * nat.VEC)
        w("  { // ---- sampled prediction of the branch decisions")
        w("    __shared__ double s_w_[2 * GM_WARPS + 2];")
        w("    __shared__ double s_m1_[GM_MAX_RED], s_m2_[GM_MAX_RED];  // sample moments (unscaled)")
        if self.vfull <= self.threads:
            w("    const i64 vs_ = threadIdx.x;")
        else:
            w("    const i64 vs_ = (i64)(((u64)threadIdx.x * 2654435761ull) % (u64)VF_);")
        w("    const bool sok_ = vs_ < VF_;")
        w("    const i64 es = vs_ * GM_VEC;")
        w("    const int nvs = sok_ ? GM_VEC : 0; (void)nvs;")
        w("    const i64 les = 0; (void)les;")
        self._tail = True   # free inputs read with per-call gmem loads (e/nv)
        try:
            levels = []
            for p in range(self.npass):
                reds = [r for r in self.pass_reds[p]]
                feeds = [d for d in self.decisions if self.avail[d.uid] > p]
                if reds and feeds:
                    levels.append((p, reds))
            # every sampled input vector is loaded once, up front (one
            # round trip for the whole chain, not one per level)
            frees = []
            for p, reds in levels:
                for n in self._nodes([r.args[0] for r in reds]):
                    if n.op == "free" and n not in frees and self.in_by_uid[n.uid].mode != MODE_SCALAR:
                        frees.append(n)
            for n in frees:
                w(f"    float n{n.uid}_s[GM_VEC];")
            for n in frees:
                for line in self._elem_code(n, "s"):
                    w("    " + line.replace("\n", "\n    "))
            for p, reds in levels:
                roots = [r.args[0] for r in reds]
                nodes = [n for n in self._nodes(roots) if n not in frees]
                guards = self._guards_roots(roots)
                w(f"    {{ // sample of pass {p}")
                for sc in self._used_scalars(nodes, guards):
                    w(f"      const float sf{sc.uid} = (float)s_scal[{self.slot[sc.uid]}]; (void)sf{sc.uid};")
                    w(f"      const bool sb{sc.uid} = s_scal[{self.slot[sc.uid]}] != 0.0; (void)sb{sc.uid};")
                for ip in self.inputs:
                    if ip.mode == MODE_SCALAR and ip.node.kind == "elem" and ip.node in nodes:
                        w(f"      const float sin{ip.slot} = gm::load_scalar<{DT_CODE[ip.dtype]}>(P.in[{ip.slot}]);")
                for n in nodes:
                    w(f"      float n{n.uid}_s[GM_VEC] = {{}};")
                cur = None
                for n in nodes:
                    g = self._guard_expr(guards.get(n.uid, frozenset({frozenset()})))
                    if g != cur:
                        if cur:
                            w("      }")
                        if g:
                            w(f"      if ({g}) {{")
                        cur = g
                    for line in self._elem_code(n, "s"):
                        w("      " + line.replace("\n", "\n      "))
                if cur:
                    w("      }")
                for r in reds:
                    k = self.red_index[r.uid]
                    x = f"n{r.args[0].uid}_s"
                    op = RED_OP[r.op]
                    if r.op in self.SAMPLE_SCALED:
                        # first and second moments of the summed term (x, x != 0, or x^2 for norm)
                        term = {"count_nonzero": f"(({x}[l] != 0.f) ? 1.0 : 0.0)",
                                "norm": f"((double){x}[l] * (double){x}[l])"}.get(r.op, f"(double){x}[l]")
                        w(f"      double t{k}_ = 0.0, q{k}_ = 0.0;")
                        w(f"      for (int l = 0; l < nvs; ++l) {{ const double z_ = {term}; t{k}_ += z_; q{k}_ += z_ * z_; }}")
                        w(f"      double v{k}_ = t{k}_, m{k}_ = q{k}_;")
                        w(f"      gm::cta_sum2(v{k}_, m{k}_, s_w_);")
                        w(f"      v{k}_ *= {scale!r};")
                        w(f"      if (threadIdx.x == 0) {{ s_red[{k}] = v{k}_; s_m1_[{k}] = v{k}_ / {scale!r}; "
                          f"s_m2_[{k}] = m{k}_; }}")
                    else:
                        w(f"      float t{k}_ = gm::acc8({op}, gm::acc_identity({op}), {x}, nvs);")
                        w(f"      const double v{k}_ = gm::cta_combine({op}, sok_ ? (double)t{k}_ : "
                          f"gm::red_identity({op}), s_w_);")
                        w(f"      if (threadIdx.x == 0) s_red[{k}] = v{k}_;")
                w("      if (threadIdx.x == 0) {")
                for r in reds:
                    w("        " + self._finish_reduction(r, self.red_index[r.uid]))
                for n in self.scalars:
                    if self.avail[n.uid] == p + 1 and n.op not in REDUCE:
                        w("        " + self._scalar_code(n))
                w("      }")
                w("      __syncthreads();")
                w("    }")
        finally:
            self._tail = False
        # Per-launch certification: a decision `red ⋈ c` is certain when the
        # sample estimate is more than 4 standard errors from c (sums, means,
        # counts, norms), or when the sample max / min already decides it.
        # Every decision certain -> speculate; otherwise the exact entry.
        nsmp = float(nsamp * nat.VEC)
        # a sample that covers the whole iteration space has no sampling error
        exact_sample = nsamp == self.vfull and self.n == self.vfull * nat.VEC
        w("    if (threadIdx.x == 0) {")
        w("      int cert_ = 1;")
        for j, d in enumerate(self.decisions):
            w(f"      s_pred[{j}] = s_scal[{self.slot[d.uid]}] != 0.0 ? 1 : 0;")
            form = self._simple_decision(d)
            if form is None:
                continue
            r, cmp, c, red_left = form
            k = self.red_index[r.uid]
            est = f"s_scal[{self.slot[r.uid]}]"
            cv = self._sv(c)
            if r.op in self.SAMPLE_SCALED:
                w("      {")
                w(f"        const double mu_ = s_m1_[{k}] / {nsmp!r}, var_ = fmax(s_m2_[{k}] / {nsmp!r} - mu_ * mu_, 0.0);")
                w(f"        double se_ = {'0.0 * ' if exact_sample else ''}sqrt(var_ / {nsmp!r});")
                if r.op in ("sum", "count_nonzero"):
                    w(f"        se_ *= {float(self.n)!r};")
                elif r.op == "norm":
                    w(f"        se_ = se_ * {float(self.n)!r} / (2.0 * fmax({est}, 1e-30));")
                w(f"        if (!(fabs({est} - ({cv})) > 4.0 * se_ + 1e-12 * fabs({cv}))) cert_ = 0;")
                w("      }")
            # max / min / any / all: a sample's extreme bounds the true one
            # from one side only, so `max > c` is certain once the sample
            # exceeds c but `max <= c` never is.  Such decisions are taken
            # from the sample without certification (a miss then clears the
            # confidence counter); requiring it would leave every chain with
            # a `c.min() < 0` that holds false unspeculated (phi4_like).
        w("      s_cert_ = cert_;")
        w("    }")
        w("    __syncthreads();")
        w("  }")

    # -- launch layout and staging ---------------------------------------------------
    def _plan_layout(self) -> None:
        """Grid, vectors per thread and staging, decided from the shape and
        the device so the kernel source is a function of the plan key.

        Every region runs 2 CTAs x 512 threads per SM (co-resident, so the
        grid barrier is safe) over a grid-stride vector map: vector v is the
        k = v // T-th vector of thread v % T (T = grid x 512), so at every
        moment the whole grid sweeps one contiguous stretch of HBM.  A thread
        issues the loads of all its vectors of a register block before any
        arithmetic (K x 16-32 B in flight per input).

        Exact multi-pass kernels keep an input a later pass re-reads in
        registers across the grid barrier when the whole pass is one block
        and the budget allows, else in its thread-private shared-memory slots
        (stashed by the first pass, or prefetched with cp.async at kernel
        start when only later passes read it).  Speculative kernels stage
        nothing: their exact fallback re-reads (from L2 in practice)."""
        sms, smem_optin = self.device_info
        self.vfull = self.n // nat.VEC
        # 2 CTAs x 512 threads per SM (64 registers a thread).  A region with
        # 8-register (fp32) vectors and >= 3 reductions keeps more live
        # values than that allows (phi4's chain spilled and ran 1.5x slower,
        # tools/ab_regions.py): one CTA per SM, 128 registers a thread.
        wide = any(VEC_REGS.get(ip.dtype, 4) == 8 for ip in self.inputs if ip.mode == MODE_FULL) \
            and len(self.reductions) >= 3
        self.threads = int(os.environ.get("GM_CTA_THREADS", str(nat.THREADS)))
        per_sm = 1024 // self.threads     # 2 x 512 or 1 x 1024 threads per SM
        self.minb = int(os.environ.get("GM_CTAS_PER_SM", str(max(1, per_sm // 2) if wide else per_sm)))
        self.grid = max(1, min(self.minb * sms, -(-max(self.vfull, 1) // self.threads)))
        self.T = self.grid * self.threads
        self.K = -(-self.vfull // self.T) if self.vfull else 0
        self.stage = {ip.slot: "none" for ip in self.inputs}
        self.load_pass: dict[int, int] = {}
        self.prefetch: set[int] = set()
        self.smem_off: dict[int, int] = {}
        self.smem_bytes = 0
        self.decisions = self._decisions()
        self.spec = self._spec_ok()
        # exact entry of a speculative region: inputs a later pass reads
        # first are prefetched into L2 during pass 0 (prefetch.global.L2),
        # so the pass after the grid barrier reads only L2 and writes HBM.
        # Nothing is staged in shared memory: on B200 the 126 MB L2 holds
        # these inputs, and the 96 KB-per-CTA stash measured slower on both
        # entries (bigbird fp32: speculative hit 12.7 -> 15.2 us, exact
        # 17.9 -> 18.9 us; tools/ab_spec.sh).
        self.l2_prefetch: list[InputPlan] = []
        self.cta_pred = self.spec and self._cta_ok()
        self.sampled = self.spec and not self.cta_pred and self._sample_ok()
        if self.spec:
            self.l2_prefetch = [ip for ip in self.inputs if ip.mode == MODE_FULL and ip.passes
                                and min(ip.passes) > 0 and self._unguarded_in(ip, min(ip.passes))]
            return
        if not self.reductions or self.npass < 2 or not self.K \
                or os.environ.get("GM_STAGING", "1") == "0":
            return
        full = [ip for ip in self.inputs if ip.mode == MODE_FULL and ip.passes]
        multi = [ip for ip in full if len(ip.passes) >= 2 and self._unguarded_in(ip, min(ip.passes))]
        # prefetch only inputs a later pass reads unconditionally: an input
        # that only an untaken arm reads must cost no HBM traffic at all
        later = [ip for ip in full if len(ip.passes) == 1 and min(ip.passes) > 0
                 and self._unguarded_in(ip, min(ip.passes))]

        def fits_regs(staged: list[InputPlan]) -> bool:
            live = sum(self.K * VEC_REGS[ip.dtype] for ip in staged)
            for p in range(self.npass):
                tmp = sum(VEC_REGS[ip.dtype] for ip in self._preload_inputs(p) if ip not in staged)
                if live + self.K * tmp > _data_regs():
                    return False
            return True

        staged: list[InputPlan] = []
        if fits_regs([]):
            for ip in multi + later:
                if fits_regs(staged + [ip]):
                    staged.append(ip)
        for ip in staged:
            self.stage[ip.slot] = "reg"
            self.load_pass[ip.slot] = 0 if ip in later else min(ip.passes)
        budget = SMEM_PER_SM // self.minb - STATIC_SMEM_RESERVE
        used = 0
        for ip in multi + later:
            if ip in staged or DT_SIZE[ip.dtype] < 2:
                continue
            b = (self.K * self.threads * nat.VEC * DT_SIZE[ip.dtype] + 127) // 128 * 128
            if used + b <= min(budget, smem_optin - STATIC_SMEM_RESERVE):
                self.stage[ip.slot] = "smem"
                self.smem_off[ip.slot] = used
                used += b
                if ip in later:
                    self.prefetch.add(ip.slot)
        self.smem_bytes = used

    def _preload_inputs(self, ctx) -> list[InputPlan]:
        """Full-size inputs a context reads unconditionally (loaded at the
        top of each register block)."""
        roots = self._ctx_roots(ctx)
        nodes = self._nodes(roots)
        guards = self._guards_roots(roots)
        out = []
        for n in nodes:
            if n.op == "free" and n.kind == "elem":
                ip = self.in_by_uid[n.uid]
                if ip.mode == MODE_FULL and not self._guard_expr(guards.get(n.uid, frozenset({frozenset()}))):
                    out.append(ip)
        return out

    def _block_loads(self, ctx) -> list[tuple[InputPlan, str]]:
        """(input, action) issued at the top of each register block of `ctx`:
        'rs' = load into the kernel-scope register stage, 'ld' = load,
        'ldst' = load and stash to shared memory after use, 'lds' = read the
        stash."""
        acts = []
        for ip in self._preload_inputs(ctx):
            st = self.stage[ip.slot]
            if st == "reg":
                if ctx == self.load_pass[ip.slot]:
                    acts.append((ip, "rs"))
            elif st == "smem":
                if ip.slot in self.prefetch or ctx != min(ip.passes):
                    acts.append((ip, "lds"))
                else:
                    acts.append((ip, "ldst"))
            else:
                acts.append((ip, "ld"))
        if ctx == 0:
            for ip in self.inputs:
                if self.stage[ip.slot] == "reg" and self.load_pass[ip.slot] == 0 and min(ip.passes) > 0:
                    acts.append((ip, "rs"))
        return acts

    def _raw_for(self, ip: InputPlan, u: int) -> tuple[list[str], str]:
        """Statements + name of the raw vector `u` of input `ip` in the
        current block (preloaded, register-staged, or loaded here)."""
        k = ip.slot
        dt = DT_CODE[ip.dtype]
        if k in self._preloaded:
            return [], self._preloaded[k].format(u=u)
        if self.stage[k] == "reg":
            return [], f"rs{k}_{u}"
        name = f"rl{k}_{u}"
        if self.stage[k] == "smem":
            return [f"gm::Raw<{dt}> {name};",
                    f"gm::rlds<{dt}>(sres{k} + (u32)(le{u} * {DT_SIZE[ip.dtype]}), {name});"], name
        return [f"gm::Raw<{dt}> {name};", f"gm::rload<{dt}>(P.in[{k}], e{u}, {name});"], name

    # -- emission ---------------------------------------------------------------------
    def _emit(self) -> str:
        out: list[str] = []
        w = out.append
        nscal = max(1, len(self.scalars))
        self._plan_layout()
        self._tail = False
        self._preloaded: dict[int, str] = {}
        prof = bool(os.environ.get("GM_PROFILE"))
        self.profiled = prof
        if prof:
            w("#define GM_PROF 1")
        if self.threads != nat.THREADS:
            w(f"#define GM_THREADS {self.threads}")
        if os.environ.get("GM_ARRIVE_RED"):
            w(f"#define GM_ARRIVE_RED {int(os.environ['GM_ARRIVE_RED'])}")
        if os.environ.get("GM_ARRIVE_SPLIT"):
            w(f"#define GM_ARRIVE_SPLIT {int(os.environ['GM_ARRIVE_SPLIT'])}")
        w('#include "gm_region.cuh"')
        w("#define gm_bool(x) (((x) != 0.0) ? 1.0 : 0.0)")
        w("#define gm_trunc(x) ((double)(long long)(x))")
        w("#define GM_LIVE_EXIT() do { if (threadIdx.x == 0 && s_live_) gm::live_exit(P); } while (0)")
        w(f"// region {self.name}: shape {list(self.shape)}, {self.npass} pass(es), "
          f"{len(self.reductions)} reduction(s), {len(self.inputs)} input(s); grid {self.grid} x {self.threads}, "
          f"{self.K} vector(s)/thread{', speculative' if self.spec else ''}")
        w(f'extern "C" __global__ void __launch_bounds__(GM_THREADS, {self.minb})')
        w("GM_KERNEL_NAME(const __grid_constant__ gm::Params P) {")
        w("  using namespace gm;")
        w("  extern __shared__ __align__(128) unsigned char smem[];")
        w("  __shared__ double s_warp[GM_WARPS * GM_MAX_RED];")
        w("  __shared__ double s_red[GM_MAX_RED];")
        w(f"  __shared__ double s_scal[{nscal}];")
        w("  (void)s_warp; (void)s_red; (void)smem;")
        if prof:
            w("  u64* prof_ = (u64*)P.scal_out + 64;")
            w("  if (threadIdx.x == 0) atomicMin(&prof_[0], gm::globaltimer());")
        w(f"  const i64 T_ = {self.T}ll;  // grid threads: vector v belongs to thread v % T_")
        w(f"  const i64 VF_ = {self.vfull}ll;  // full 8-element vectors")
        w("  const i64 t0_ = (i64)blockIdx.x * GM_THREADS + threadIdx.x;")
        w("  (void)T_; (void)VF_; (void)t0_;")
        # programmatic dependent launch: wait for the previous kernel's
        # results before the first global read (a no-op without PDL)
        w('  asm volatile("griddepcontrol.wait;" ::: "memory");')
        w("  __shared__ int s_live_;  // live timer on (diagnostics word, bench.py)")
        w("  if (threadIdx.x == 0) {")
        w("    int f_; asm volatile(\"ld.global.u32 %0, [%1];\" : \"=r\"(f_) : \"l\"((int*)(P.barrier + GM_SCRATCH_FORCE)));")
        w("    s_live_ = (f_ & GM_LIVE_BIT) != 0;")
        w("    if (s_live_) gm::live_start(P);")
        w("  }")
        w("  u64 ep_ = gm::grid_epoch_begin(P); (void)ep_;  // arrival epoch (thread 0)")
        w("  __shared__ int s_epi_;  // does this CTA write the scalar outputs / mirror")
        w("  if (threadIdx.x == 0) s_epi_ = blockIdx.x == 0;")
        for ip in self.inputs:
            if ip.mode == MODE_FULL and self.stage[ip.slot] == "smem":
                w(f"  const u32 sres{ip.slot} = smem_u32(smem + {self.smem_off[ip.slot]});")
        for ip in self.inputs:
            if self.stage[ip.slot] == "reg":
                for u in range(self.K):
                    w(f"  gm::Raw<{DT_CODE[ip.dtype]}> rs{ip.slot}_{u};")
        def prefetch():
            if not self.prefetch:
                return
            # cp.async of every vector a later pass reads into its stash slot
            for slot in sorted(self.prefetch):
                ip = self.inputs[slot]
                dt = DT_CODE[ip.dtype]
                w(f"  for (int k = 0; k < {self.K}; ++k) {{")
                w("    const i64 v = t0_ + (i64)k * T_;")
                w(f"    if (v < VF_) gm::rprefetch<{dt}>(sres{slot} + (u32)(((i64)k * GM_THREADS + threadIdx.x) * "
                  f"GM_VEC * {DT_SIZE[ip.dtype]}), P.in[{slot}], v * GM_VEC);")
                w("  }")
            w("  gm::cp_async_commit();")

        self.red_index = {r.uid: i for i, r in enumerate(self.reductions)}
        if not self.spec:
            prefetch()
            self._emit_scalar_level(w, 0)
        else:
            # Adaptive speculation.  A confidence counter in the scratch
            # (+56) picks the entry: >= 2 speculates; below, the exact passes
            # run and the counter grows while launches confirm the predictor.
            # A hit keeps the counter, a miss resets it.  Sampled regions
            # predict from this launch's own data and speculate only when the
            # sample certifies the decisions; the others predict the last
            # launch's decisions, so inputs whose decisions alternate settle
            # on the exact entry instead of paying a sweep plus a restart.
            nd = len(self.decisions)
            w(f"  __shared__ int s_pred[{nd}];")
            w("  __shared__ int s_miss;")
            w("  __shared__ int s_mode;  // 1: speculate on the predicted decisions")
            w("  int* pred_ = (int*)(P.barrier + GM_SCRATCH_PRED);  // last launch's decisions")
            w("  int* conf_ = (int*)(P.barrier + GM_SCRATCH_CONF);  // prediction confidence")
            w("  __shared__ int s_force_;  // diagnostics word (GM_SCRATCH_FORCE)")
            w("  if (threadIdx.x == 0) {")
            w("    int c_; asm volatile(\"ld.global.u32 %0, [%1];\" : \"=r\"(c_) : \"l\"(conf_));")
            w("    int f_; asm volatile(\"ld.global.u32 %0, [%1];\" : \"=r\"(f_) : \"l\"((int*)(P.barrier + GM_SCRATCH_FORCE)));")
            w(f"    s_mode = c_ >= {SPEC_CONFIDENT} ? 1 : 0;")
            w("    s_force_ = f_;")
            w("  }")
            if self.cta_pred:
                w("  __shared__ int s_cert_;")
                w("  __shared__ double s_w_[2 * GM_WARPS + 2], s_m1_[GM_MAX_RED], s_m2_[GM_MAX_RED];")
            self._emit_scalar_level(w, 0)
            if self.sampled:
                # sampled regions: the sample certifies (or not) THIS launch's
                # decisions; the counter only guards against a predictor that
                # keeps missing (a miss clears it, certified launches raise it)
                w("  __shared__ int s_cert_;")
                self._emit_sample(w)
                w("  if (threadIdx.x == 0) s_mode = (s_cert_ && s_mode) ? 1 : 0;")
            w("  if (threadIdx.x == 0) {  // diagnostics: forced entry / flipped predictions")
            w("    if (s_force_ & (1 << 30)) s_mode = 0;")
            w("    if (s_force_ & (int)0x80000000u) s_mode = 1;")
            if self.sampled:
                for j in range(nd):
                    w(f"    s_pred[{j}] ^= (s_force_ >> {j}) & 1;")
            w("  }")
            w("  __syncthreads();")
            w("  if (s_mode) {")
            saved = (self.stage, self.prefetch)
            self.stage = {k: "none" for k in self.stage}
            self.prefetch = set()
            self._emit_ctx(w, "spec")
            w("  if (!s_miss) {")
            self._emit_epilogue(w, "    ", mode="hit")
            w("    GM_LIVE_EXIT();")
            w("    return;")
            w("  }")
            w("  // misprediction: the exact passes from the first mispredicted level (inputs re-read)")
            for p in range(1, self.npass):
                # decisions have level >= 1, so pass 0 never reruns
                w(f"  if (s_miss <= {p}) {{")
                self._emit_ctx(w, p)
                w("  }")
            self._emit_epilogue(w, "  ", mode="miss")
            w("  GM_LIVE_EXIT();")
            w("  return;")
            w("  }")
            self.stage, self.prefetch = saved
            w("  // exact entry: every pass; inputs first read after a grid barrier are pulled into L2 now")
            for ip in self.l2_prefetch:
                w(f"  for (int k = 0; k < {self.K}; ++k) {{")
                w("    const i64 v = t0_ + (i64)k * T_;")
                w(f"    if (v < VF_) gm::prefetch_l2((const char*)P.in[{ip.slot}].ptr + v * GM_VEC * "
                  f"{DT_SIZE[ip.dtype]}, {nat.VEC * DT_SIZE[ip.dtype]});")
                w("  }")
            prefetch()
        for p in range(self.npass):
            if p in self.hoisted and not self.spec:
                self._emit_hoist_guard(w, p)
                w(f"  if (!s_hoist{p}) {{  // hoisting guard failed: the exact sweep")
                self._emit_ctx(w, p, scalar_level=False)
                w("  }")
                self._emit_scalar_level(w, p + 1)
            else:
                self._emit_ctx(w, p)
        if prof:
            w("  __syncthreads();")
            w("  if (threadIdx.x == 0) atomicMax(&prof_[63], gm::globaltimer());")
        self._emit_epilogue(w, "  ", mode="exact" if self.spec else "plain")
        w("  GM_LIVE_EXIT();")
        w("}")
        return "\n".join(out) + "\n"

    def _emit_epilogue(self, w, ind: str, mode: str) -> None:
        """Scalar outputs, the debug mirror and (speculative kernels) the
        prediction and confidence update + launch / miss / exact-entry
        counters, by one thread.  `mode`: "plain" (no speculation), "hit",
        "miss" (after the restart) or "exact" (the exact entry)."""
        w(f"{ind}if (s_epi_ && threadIdx.x == 0) {{")
        for j, o in enumerate(self.outputs):
            if o.kind == "dscalar":
                k = self._out_slot(j)
                val = self._sv(o)
                if o.dtype == torch.int64:
                    w(f"{ind}  *(long long*)P.out[{k}].ptr = (long long){val};")
                elif o.dtype == torch.int32:
                    w(f"{ind}  *(int*)P.out[{k}].ptr = (int){val};")
                else:
                    w(f"{ind}  gm::store_scalar<{DT_CODE[o.dtype]}>(P.out[{k}], {val});")
        w(f"{ind}  if (P.scal_out) {{")
        w(f"{ind}    for (int i = 0; i < {len(self.scalars)}; ++i) ((double*)P.scal_out)[i] = s_scal[i];")
        w(f"{ind}  }}")
        if self.spec:
            w(f"{ind}  u64* st_ = (u64*)(P.barrier + GM_SCRATCH_STATS);  // [launches, mispredictions, exact entries]")
            w(f"{ind}  st_[0] += 1;")
            if mode == "hit":
                w(f"{ind}  *conf_ = min(*conf_ + 1, {SPEC_CONF_MAX});")
            elif mode == "miss":
                w(f"{ind}  st_[1] += 1;")
                # per-CTA prediction: an uncertified launch was expected to
                # risk a miss; only a certified miss indicts the predictor
                w(f"{ind}  if (s_cert_) *conf_ = 0;" if self.cta_pred else f"{ind}  *conf_ = 0;")
            elif self.cta_pred:
                w(f"{ind}  st_[2] += 1;")
                w(f"{ind}  *conf_ = min(*conf_ + 1, {SPEC_CONF_MAX});  // no prediction on this entry")
            else:
                w(f"{ind}  st_[2] += 1;")
                w(f"{ind}  int same_ = 1;")
                ref = "s_pred" if self.sampled else "pred_"
                for j, d in enumerate(self.decisions):
                    w(f"{ind}  same_ &= ((s_scal[{self.slot[d.uid]}] != 0.0) == ({ref}[{j}] != 0)) ? 1 : 0;")
                if self.sampled:
                    # an uncertified launch says nothing about the predictor
                    w(f"{ind}  if (s_cert_) *conf_ = same_ ? min(*conf_ + 1, {SPEC_CONF_MAX}) : 0;")
                else:
                    w(f"{ind}  *conf_ = same_ ? min(*conf_ + 1, {SPEC_CONF_MAX}) : 0;")
            if mode in ("miss", "exact"):
                for j, d in enumerate(self.decisions):
                    w(f"{ind}  pred_[{j}] = (s_scal[{self.slot[d.uid]}] != 0.0) ? 1 : 0;")
        w(f"{ind}}}")

    def _emit_ctx(self, w, ctx, scalar_level: bool = True) -> None:
        spec = ctx == "spec"
        roots = self._ctx_roots(ctx)
        elem_nodes = self._nodes(roots)
        guards = self._guards_roots(roots)
        if spec:
            reds = list(self.reductions)
            outs = [jo for p in range(self.npass) for jo in self.pass_outputs[p]]
        else:
            reds = self.pass_reds[ctx]
            outs = self.pass_outputs[ctx]
        if not elem_nodes and not reds and not outs:
            return
        w(f"  {{ // ---- {'speculative pass (every pass under predicted decisions)' if spec else f'pass {ctx}'}")
        # values read from global memory are loaded after the first block's
        # data loads are issued (`late`), so their round trip overlaps them
        late: list[str] = []
        for s in self._used_scalars(elem_nodes, guards):
            if spec and self.avail.get(s.uid, 0) >= 1 and self.cta_pred:
                w(f"    float sf{s.uid} = 0.f; bool sb{s.uid} = false; (void)sf{s.uid}; (void)sb{s.uid};")
            elif spec and self.avail.get(s.uid, 0) >= 1 and self.sampled:
                j = self.decisions.index(s)
                w(f"    const bool sb{s.uid} = s_pred[{j}] != 0; const float sf{s.uid} = sb{s.uid} ? 1.f : 0.f; "
                  f"(void)sf{s.uid};")
            elif spec and self.avail.get(s.uid, 0) >= 1:
                j = self.decisions.index(s)
                w(f"    float sf{s.uid} = 0.f; bool sb{s.uid} = false; (void)sf{s.uid}; (void)sb{s.uid};")
                late.append(f"{{ int pd_; asm volatile(\"ld.global.u32 %0, [%1];\" : \"=r\"(pd_) : \"l\"(pred_ + {j})); "
                            f"pd_ = (pd_ != 0) ^ ((s_force_ >> {j}) & 1); "
                            f"sf{s.uid} = pd_ ? 1.f : 0.f; sb{s.uid} = pd_ != 0; if (threadIdx.x == 0) s_pred[{j}] = pd_; }}")
            else:
                w(f"    const float sf{s.uid} = (float)s_scal[{self.slot[s.uid]}]; (void)sf{s.uid};")
                w(f"    const bool sb{s.uid} = s_scal[{self.slot[s.uid]}] != 0.0; (void)sb{s.uid};")
            if (s.op == "free" and s.kind == "host") or (s.kind == "dscalar" and s.dtype == torch.bfloat16):
                w(f"    u32 spk{s.uid} = gm::f2bf2(sf{s.uid}, sf{s.uid}); (void)spk{s.uid};")
        for ip in self.inputs:
            if ip.mode == MODE_SCALAR and ip.node.kind == "elem" and ip.node in elem_nodes:
                w(f"    float sin{ip.slot} = 0.f;")
                late.append(f"sin{ip.slot} = gm::load_scalar<{DT_CODE[ip.dtype]}>(P.in[{ip.slot}]);")
        self._late = late
        self._cta_predict_here = spec and self.cta_pred
        for k, r in enumerate(reds):
            if r.op in ("argmax", "argmin"):
                w(f"    u64 acc{k} = 0ull;")
            elif self._exact_acc(r):
                w(f"    double acc{k} = 0.0;")
            else:
                w(f"    float acc{k} = gm::acc_identity({RED_OP[r.op]});")
        if self.prefetch and not spec and ctx == min(min(self.inputs[s].passes) for s in self.prefetch):
            w("    gm::cp_async_wait_all();  // this thread's prefetched stash slots")
        loads = self._block_loads(ctx)
        prof = self.profiled
        nr = len(reds)
        pidx = self.npass if spec else ctx
        pargs = f", prof_ + 40 + 4 * {pidx}" if prof else ""
        nx = self.extra_slots() if spec else 0
        if reds:
            ops = [str(RED_OP[r.op]) for r in reds]
            slots = [str(self.red_index[r.uid]) for r in reds]
            for j in range(len(self.decisions) if nx else 0):
                ops += [str(RED_OP["amin"]), str(RED_OP["amax"])]
                slots += [str(len(self.reductions) + 2 * j), str(len(self.reductions) + 2 * j + 1)]
            if nx:
                ops.append(str(RED_OP["amin"]))
                slots.append(str(len(self.reductions) + 2 * len(self.decisions)))
            w(f"    const int ops_[{nr + nx}] = {{{', '.join(ops)}}};")
            w(f"    const int slots_[{nr + nx}] = {{{', '.join(slots)}}};")
            w("    u64 tgt_ = 0; (void)tgt_;")

        def stamp_loop_end():
            if prof:
                idx = 1 + 2 * pidx
                w("    __syncthreads();")
                w(f"    if (threadIdx.x == 0) {{ const u64 t_ = gm::globaltimer(); atomicMax(&prof_[{idx}], t_); "
                  f"atomicMin(&prof_[{32 + idx}], t_); }}")

        def arrive():
            vals = [f"__longlong_as_double((long long)acc{k})" if r.op in ("argmax", "argmin")
                    else f"(double)acc{k}" for k, r in enumerate(reds)]
            for j in range(len(self.decisions) if nx else 0):
                vals += [f"(double)s_pred[{j}]", f"(double)s_pred[{j}]"]
            if nx:
                vals.append("(double)s_cert_")
            w(f"    {{ double vals_[{nr + nx}] = {{{', '.join(vals)}}};")
            w(f"      tgt_ = grid_arrive(P, {nr + nx}, ops_, slots_, vals_, s_warp, s_red, ep_{pargs}); }}")

        deferred = False
        if self.K:
            tmp = sum(VEC_REGS[ip.dtype] for ip, a in loads if a != "rs")
            if any(st == "reg" for st in self.stage.values()):
                kb = self.K                      # register staging: one block by construction
            else:
                kb = self.K if self.K * tmp <= _data_regs() else max(1, _data_regs() // max(1, tmp))
                nblk = -(-self.K // kb)
                kb = -(-self.K // nblk)
            pref = None
            if not os.environ.get("GM_NO_PACKED"):
                pp = self._packed_plan(elem_nodes)
                if any(v == "P" for v in pp.values()):
                    pref = pp
            if kb >= self.K:
                # one block: optionally (GM_DEFER_STORES=1) the block's output
                # stores are held in registers and issued after the grid
                # arrival; measured neutral on B200 (tools/ab_regions.py)
                deferred = bool(reds) and bool(outs) and os.environ.get("GM_DEFER_STORES", "0") == "1"
                w("    {")
                self._emit_block(w, "0", self.K, elem_nodes, reds, outs, guards, loads, pref, defer=deferred)
                if deferred:
                    if self.n % nat.VEC:
                        w("    {")
                        self._emit_tail(w, elem_nodes, reds, outs, guards)
                        w("    }")
                    stamp_loop_end()
                    arrive()
                    self._emit_deferred_stores(w, "      ", outs, self.K, pref)
                w("    }")
            else:
                w(f"    for (int kb = 0; kb < {self.K}; kb += {kb}) {{")
                self._emit_block(w, "kb", kb, elem_nodes, reds, outs, guards, loads, pref)
                w("    }")
        # the launch's last reduction (exact path, results feed only scalar
        # outputs): the completing CTA combines alone, the others exit
        last_arriver = (bool(reds) and not spec and ctx == self.npass - 1 and not deferred
                        and os.environ.get("GM_LAST_ARRIVER", "1") != "0")
        if not deferred:
            if self.n % nat.VEC:
                for line in self._late:
                    w("    " + line)
                self._emit_tail(w, elem_nodes, reds, outs, guards)
            stamp_loop_end()
            if reds and not last_arriver:
                arrive()
        if last_arriver:
            vals = ", ".join(f"__longlong_as_double((long long)acc{k})" if r.op in ("argmax", "argmin")
                             else f"(double)acc{k}" for k, r in enumerate(reds))
            w(f"    {{ double vals_[{nr}] = {{{vals}}};")
            w(f"      if (!gm::grid_reduce_last(P, {nr}, ops_, slots_, vals_, s_warp, s_red, ep_{pargs})) "
              f"{{ GM_LIVE_EXIT(); return; }} }}")
            w("    if (threadIdx.x == 0) s_epi_ = 1;  // this CTA writes the scalar outputs")
        elif reds:
            w(f"    grid_wait(P, {nr + nx}, ops_, slots_, tgt_, s_red{pargs});")
        if reds:
            if prof:
                idx = 2 + 2 * pidx
                w(f"    if (threadIdx.x == 0) atomicMax(&prof_[{idx}], gm::globaltimer());")
            if spec:
                # replay the scalar levels in order with the exact statistics
                # and compare every predicted decision
                w("    if (threadIdx.x == 0) {")
                for p in range(self.npass):
                    for r in self.pass_reds[p]:
                        w("      " + self._finish_reduction(r, self.red_index[r.uid]))
                    for n in self.scalars:
                        if self.avail[n.uid] == p + 1 and n.op not in REDUCE:
                            w("      " + self._scalar_code(n))
                # s_miss = the lowest scalar level holding a mispredicted
                # decision (0: every prediction held).  Passes below it ran
                # under correct decisions, so their reductions and outputs
                # are exact and the miss path restarts at that pass.
                w("      int miss_ = 0x7fffffff;")
                if self.cta_pred:
                    # every CTA predicted for itself: a decision holds when
                    # all CTAs predicted it (min == max) and it was right
                    base = len(self.reductions)
                    for j, d in enumerate(self.decisions):
                        lo, hi = f"s_red[{base + 2 * j}]", f"s_red[{base + 2 * j + 1}]"
                        w(f"      if (!({lo} == {hi} && (({lo} != 0.0) == (s_scal[{self.slot[d.uid]}] != 0.0)))) "
                          f"miss_ = min(miss_, {self.avail[d.uid]});")
                    w(f"      s_cert_ = s_red[{base + 2 * len(self.decisions)}] != 0.0 ? 1 : 0;  // all CTAs certified")
                else:
                    for j, d in enumerate(self.decisions):
                        w(f"      if ((s_scal[{self.slot[d.uid]}] != 0.0) != (s_pred[{j}] != 0)) "
                          f"miss_ = min(miss_, {self.avail[d.uid]});")
                w("      s_miss = miss_ == 0x7fffffff ? 0 : miss_;")
                w("    }")
                w("    __syncthreads();")
            else:
                w("    if (threadIdx.x == 0) {")
                for k, r in enumerate(reds):
                    w("      " + self._finish_reduction(r, k))
                w("    }")
                w("    __syncthreads();")
                if scalar_level:
                    self._emit_scalar_level(w, ctx + 1)
        w("  }")

    def _emit_block(self, w, kb: str, U: int, elem_nodes, reds, outs, guards, loads, pref, defer=False) -> None:
        """One register block: U vectors per thread, every load issued first.
        With `defer`, outputs are kept in registers (ho*) for stores issued by
        the caller after the grid arrival."""
        ind = "      "
        for u in range(U):
            k = f"({kb} + {u})" if kb != "0" else f"{u}"
            w(f"{ind}const i64 v{u} = t0_ + (i64){k} * T_;")
            if kb == "0" and (u + 1) * self.T <= self.vfull:
                w(f"{ind}const bool ok{u} = true;  // t0_ < T_: every thread has its vector {u}")
            else:
                w(f"{ind}const bool ok{u} = v{u} < VF_;")
            w(f"{ind}const i64 e{u} = v{u} * GM_VEC;")
            w(f"{ind}const int nv{u} = GM_VEC; (void)nv{u};")
            w(f"{ind}const i64 le{u} = ((i64){k} * GM_THREADS + threadIdx.x) * GM_VEC; (void)le{u};")
        self._preloaded = {}
        for ip, act in loads:
            dt = DT_CODE[ip.dtype]
            k = ip.slot
            if act == "rs":
                self._preloaded[k] = f"rs{k}_{{u}}"
                continue
            self._preloaded[k] = f"r{k}_{{u}}"
            for u in range(U):
                w(f"{ind}gm::Raw<{dt}> r{k}_{u};")
        for u in range(U):
            for ip, act in loads:
                dt = DT_CODE[ip.dtype]
                k = ip.slot
                if act in ("rs", "ld", "ldst"):
                    dst = f"rs{k}_{u}" if act == "rs" else f"r{k}_{u}"
                    w(f"{ind}if (ok{u}) gm::rload<{dt}>(P.in[{k}], e{u}, {dst});")
                else:
                    w(f"{ind}if (ok{u}) gm::rlds<{dt}>(sres{k} + (u32)(le{u} * {DT_SIZE[ip.dtype]}), r{k}_{u});")
        for line in self._late:
            w(ind + line)
        if getattr(self, "_cta_predict_here", False):
            w(ind + (f"if ({kb} == 0) " if kb != "0" else "") + "{")
            for line in self._cta_predict_lines():
                w(ind + "  " + line)
            w(ind + "}")
        if pref is None:
            pref = {n.uid: "F" for n in elem_nodes}
        needs: dict[int, set] = {n.uid: {pref[n.uid]} for n in elem_nodes}
        for n in elem_nodes:
            for a in n.args:
                if a.kind == "elem":
                    needs[a.uid].add(pref[n.uid] if (pref[n.uid] == "P" and not (n.op == "where" and a is n.args[0]))
                                     else "F")
        for r in reds:
            x = r.args[0]
            packed_red = r.op in ("amax", "amin") and pref.get(x.uid) == "P"
            needs[x.uid].add("P" if packed_red else "F")
        for _, o in outs:
            needs[o.uid].add(pref[o.uid])
        # nodes some consumer reads unpacked (float lanes)
        self._f_consumers = {}
        for n in elem_nodes:
            for a in n.args:
                if a.kind == "elem" and (pref[n.uid] == "F" or (n.op == "where" and a is n.args[0])):
                    self._f_consumers[a.uid] = True
        for r in reds:
            if not (r.op in ("amax", "amin") and pref.get(r.args[0].uid) == "P"):
                self._f_consumers[r.args[0].uid] = True
        for _, o in outs:
            if pref[o.uid] == "F":
                self._f_consumers[o.uid] = True
        if defer:
            for u in range(U):
                for j, o in outs:
                    if pref.get(o.uid) == "P":
                        w(f"{ind}u32 ho{j}_{u}[4];")
                    else:
                        w(f"{ind}float ho{j}_{u}[GM_VEC];")
        alias = self._arm_aliases(elem_nodes, reds, outs, pref, needs)
        root_reds: dict[int, list] = {}
        root_red_k: dict[int, int] = {}
        for k, r in enumerate(reds):
            root_reds.setdefault(r.args[0].uid, []).append(r)
            root_red_k[r.uid] = k
        root_outs: dict[int, list] = {}
        for j, o in outs:
            root_outs.setdefault(o.uid, []).append((j, o))
        w_outer = w
        for u in range(U):
            body: list[str] = []
            w = body.append
            w(f"{ind}if (ok{u}) {{")
            for n in elem_nodes:
                if n.uid in alias:
                    continue
                if "F" in needs[n.uid]:
                    w(f"{ind}  float n{n.uid}_{u}[GM_VEC];")
                if "P" in needs[n.uid]:
                    w(f"{ind}  u32 p{n.uid}_{u}[4];")
            cur_guard = None
            open_block = False
            for n in elem_nodes:
                g = self._guard_expr(guards.get(n.uid, frozenset({frozenset()})))
                if g != cur_guard:
                    if open_block:
                        w(f"{ind}  }}")
                        open_block = False
                    if g:
                        w(f"{ind}  if ({g}) {{")
                        open_block = True
                    cur_guard = g
                for line in self._node_code(n, u, pref, needs):
                    w(ind + "    " + line.replace("\n", "\n" + ind + "    "))
                # reductions and stores of a root right after it is computed
                # (roots are unguarded), so its registers die early
                if n.uid in root_reds or n.uid in root_outs:
                    if open_block:
                        w(f"{ind}  }}")
                        open_block = False
                        cur_guard = None
                    self._emit_reds_outs(w, ind + "  ", root_reds.get(n.uid, []), root_outs.get(n.uid, []), u,
                                         pref, hold=defer, red_index=root_red_k)
            if open_block:
                w(f"{ind}  }}")
            for ip, act in loads:
                if act == "ldst":
                    w(f"{ind}  gm::rstash<{DT_CODE[ip.dtype]}>(sres{ip.slot} + (u32)(le{u} * {DT_SIZE[ip.dtype]}), "
                      f"r{ip.slot}_{u});")
            w(f"{ind}}}")
            text = "\n".join(body)
            for a_uid, w_uid in alias.items():
                text = re.sub(rf"\b([np]){a_uid}_{u}\b", rf"\g<1>{w_uid}_{u}", text)
            w_outer(text)
        self._preloaded = {}

    def _arm_aliases(self, elem_nodes, reds, outs, pref, needs) -> dict[int, int]:
        """Arms of a uniform select computed only for it write straight into
        the select's registers (`where(p, A, B)`: A under `if (p)`, B under
        `else`), so the select is a no-op and the two arms never hold
        registers at the same time — the phi4 chain keeps ~3 live vectors
        instead of ~10.  Returns {arm uid: select uid} (resolved through
        chains of selects)."""
        cons: dict[int, list] = {n.uid: [] for n in elem_nodes}
        for n in elem_nodes:
            for a in n.args:
                if a.kind == "elem" and a.uid in cons:
                    cons[a.uid].append(n)
        for r in reds:
            cons.setdefault(r.args[0].uid, []).append(r)
        for _, o in outs:
            cons.setdefault(o.uid, []).append(None)
        alias: dict[int, int] = {}
        for n in elem_nodes:
            if n.op != "where" or n.args[0].kind == "elem":
                continue
            for arm in n.args[1:]:
                if arm.kind != "elem" or arm.op == "free" or arm.uid in alias or arm is n.args[0]:
                    continue
                if any(c is not n for c in cons.get(arm.uid, [])):
                    continue
                if arm.dtype != n.dtype or pref[arm.uid] != pref[n.uid] or not needs[arm.uid] <= needs[n.uid]:
                    continue
                alias[arm.uid] = n.uid
        # resolve chains (an arm aliased to a select that is itself an arm)
        for a in list(alias):
            t = alias[a]
            while t in alias:
                t = alias[t]
            alias[a] = t
        return alias

    def _emit_tail(self, w, elem_nodes, reds, outs, guards) -> None:
        """The partial last vector (n % 8 lanes), owned by thread VF_ % T_;
        per-lane global loads and stores."""
        ind = "      "
        w("    if (t0_ == VF_ % T_) {")
        w(f"{ind}const i64 e0 = VF_ * GM_VEC;")
        w(f"{ind}const int nv0 = (int)({self.n}ll - e0);")
        w(f"{ind}const i64 le0 = 0; (void)le0;")
        self._tail = True
        for n in elem_nodes:
            w(f"{ind}float n{n.uid}_0[GM_VEC];")
        cur_guard = None
        open_block = False
        for n in elem_nodes:
            g = self._guard_expr(guards.get(n.uid, frozenset({frozenset()})))
            if g != cur_guard:
                if open_block:
                    w(f"{ind}}}")
                    open_block = False
                if g:
                    w(f"{ind}if ({g}) {{")
                    open_block = True
                cur_guard = g
            for line in self._elem_code(n, 0):
                w(ind + "  " + line.replace("\n", "\n" + ind + "  "))
        if open_block:
            w(f"{ind}}}")
        self._emit_reds_outs(w, ind, reds, outs, 0)
        self._tail = False
        w("    }")

    def _node_code(self, n: Node, u: int, pref: dict, needs: dict) -> list[str]:
        def convert() -> list[str]:
            out = []
            if pref[n.uid] == "P" and "F" in needs[n.uid]:
                out.append(f"gm::unpack8(p{n.uid}_{u}, n{n.uid}_{u});")
            if pref[n.uid] == "F" and "P" in needs[n.uid]:
                out.append(f"gm::pack8(n{n.uid}_{u}, p{n.uid}_{u});")
            return out

        if pref[n.uid] == "F":
            # a bf16 node only read packed: pack8's RN conversion is its rounding
            self._no_round = (n.dtype == torch.bfloat16 and "P" in needs[n.uid]
                              and not self._f_consumers.get(n.uid))
            try:
                return self._elem_code(n, u) + convert()
            finally:
                self._no_round = False
        dst = f"p{n.uid}_{u}"
        if n.op == "free":
            pre, raw = self._raw_for(self.in_by_uid[n.uid], u)
            return pre + [f"#pragma unroll\nfor (int j = 0; j < 4; ++j) {dst}[j] = {raw}.w[j];"] + convert()

        def pv(a: Node) -> str:
            return f"p{a.uid}_{u}[j]" if a.kind == "elem" else self._packed_scalar(a)

        a = n.args
        if n.op in ("add", "sub", "mul"):
            fn = {"add": "gm::hadd2", "sub": "gm::hsub2", "mul": "gm::hmul2"}[n.op]
            body = f"{fn}({pv(a[0])}, {pv(a[1])})"
        elif n.op == "div":
            rb = self._bf16_bits(self._pow2_recip(a[1].value))
            body = f"gm::hmul2({pv(a[0])}, 0x{(rb << 16) | rb:08x}u)"
        elif n.op == "relu":
            body = f"gm::hmax2({pv(a[0])}, 0u)"
        elif n.op == "neg":
            body = f"({pv(a[0])} ^ 0x80008000u)"
        elif n.op == "abs":
            body = f"({pv(a[0])} & 0x7fff7fffu)"
        elif n.op == "pos":
            body = pv(a[0])
        elif n.op == "where":
            c = a[0]
            return [f"if (sb{c.uid}) {{\n#pragma unroll\nfor (int j = 0; j < 4; ++j) {dst}[j] = p{a[1].uid}_{u}[j];\n}} "
                    f"else {{\n#pragma unroll\nfor (int j = 0; j < 4; ++j) {dst}[j] = p{a[2].uid}_{u}[j];\n}}"] + convert()
        else:
            raise AssertionError(n.op)
        return [f"#pragma unroll\nfor (int j = 0; j < 4; ++j) {dst}[j] = {body};"] + convert()


    # -- packed bf16x2 path ------------------------------------------------------
    @staticmethod
    def _pow2_recip(v):
        """1/v when v is a power of two whose reciprocal is a normal float32
        (then x / v == x * (1/v) bit for bit), else None."""
        try:
            f = float(v)
        except (TypeError, ValueError):
            return None
        if f == 0.0 or f != f or abs(f) == float("inf"):
            return None
        m, e = math.frexp(abs(f))
        if m != 0.5 or not (-125 <= e - 1 <= 125):
            return None
        return 1.0 / f

    @staticmethod
    def _bf16_exact(v) -> bool:
        f = torch.tensor(float(v), dtype=torch.float32)
        return bool(f.to(torch.bfloat16).to(torch.float32) == f)

    @staticmethod
    def _bf16_bits(v) -> int:
        return int(torch.tensor(float(v), dtype=torch.float32).to(torch.bfloat16).view(torch.int16).item()) & 0xFFFF

    def _scalar_packable(self, s: Node, op: str) -> bool:
        """May scalar `s` enter a packed bf16 op `op` without changing the
        result?  add/sub/compare round the scalar to bf16 in torch anyway;
        mul keeps it in fp32, so it must be bf16-exact."""
        if s.op == "const":
            return op in ("add", "sub") or self._bf16_exact(s.value)
        if s.op == "free" and s.kind == "host":
            return op in ("add", "sub") or self.host_exact.get(s.uid, False)
        if s.kind == "dscalar" and s.dtype == torch.bfloat16:
            # a 0-d bf16 tensor holds a bf16 value: the packed op is exact
            return op in ("add", "sub", "mul")
        return False

    def _packed_plan(self, elem_nodes: list[Node]) -> dict[int, str]:
        pref: dict[int, str] = {}
        bf = torch.bfloat16
        for n in elem_nodes:
            r = "F"
            if n.dtype == bf:
                if n.op == "free":
                    ip = self.in_by_uid[n.uid]
                    if ip.mode == MODE_FULL and ip.dtype == bf:
                        r = "P"
                elif n.op in ("add", "sub", "mul"):
                    ok = True
                    for a in n.args:
                        if a.kind == "elem":
                            ok &= a.dtype == bf
                        else:
                            ok &= self._scalar_packable(a, n.op)
                    if ok and any(a.kind == "elem" for a in n.args):
                        r = "P"
                elif n.op == "div" and n.args[0].kind == "elem" and n.args[0].dtype == bf \
                        and n.args[1].op == "const" and self._pow2_recip(n.args[1].value) is not None:
                    r = "P"   # x / 2^k == x * 2^-k (bf16-exact), one rounding either way
                elif n.op in ("neg", "pos", "abs", "relu"):
                    if n.args[0].kind == "elem" and n.args[0].dtype == bf:
                        r = "P"
                elif n.op == "where" and n.args[0].kind != "elem":
                    if all(a.kind == "elem" and a.dtype == bf for a in n.args[1:]):
                        r = "P"
            pref[n.uid] = r
        return pref

    def _packed_scalar(self, s: Node) -> str:
        if s.op == "const":
            b = self._bf16_bits(s.value)
            return f"0x{(b << 16) | b:08x}u"
        return f"spk{s.uid}"

    def _emit_deferred_stores(self, w, ind, outs, U, pref) -> None:
        for u in range(U):
            w(f"{ind}if (ok{u}) {{")
            for j, o in outs:
                k = self._out_slot(j)
                if pref is not None and pref.get(o.uid) == "P":
                    w(f"{ind}  gm::stg_raw(P.out[{k}], e{u}, ho{j}_{u});")
                else:
                    w(f"{ind}  gm::store8<{DT_CODE[o.dtype]}>(P.out[{k}], e{u}, nv{u}, ho{j}_{u});")
            w(f"{ind}}}")

    def _emit_reds_outs(self, w, ind, reds, outs, u, pref=None, hold=False, red_index=None):
        for k0, r in enumerate(reds):
            k = red_index[r.uid] if red_index is not None else k0
            x = r.args[0]
            src = f"n{x.uid}_{u}"
            if r.op in ("amax", "amin") and pref is not None and pref.get(x.uid) == "P":
                # bf16 max/min on the packed words: 3 max.NaN.bf16x2, then 2 lanes
                w(f"{ind}acc{k} = gm::acc_minmax_p<{1 if r.op == 'amax' else 0}>(acc{k}, p{x.uid}_{u});")
            elif r.op in ("sum", "mean", "norm") and pref is not None and pref.get(x.uid) == "P" \
                    and x.dtype == torch.bfloat16 and os.environ.get("GM_PACKED_SUM", "1") != "0":
                w(f"{ind}acc{k} = gm::acc_sum_p<{'true' if r.op == 'norm' else 'false'}>(acc{k}, p{x.uid}_{u}, nv{u});")
            elif r.op in ("argmax", "argmin"):
                w(f"{ind}acc{k} = gm::argkey8(acc{k}, {src}, e{u}, nv{u}, {'true' if r.op == 'argmin' else 'false'});")
            elif r.op == NZSUM:
                w(f"{ind}{{ double t_ = 0.0;\n#pragma unroll\n{ind}for (int l = 0; l < GM_VEC; ++l) "
                  f"if (l < nv{u} && {src}[l] != 0.f) t_ += (double)({self._coordsum(f'(e{u} + l)')});\n"
                  f"{ind}acc{k} += t_; }}")
            elif self._exact_acc(r):
                w(f"{ind}{{ double t_ = 0.0;\n#pragma unroll\n{ind}for (int l = 0; l < GM_VEC; ++l) "
                  f"if (l < nv{u}) t_ += (double)({'(' + src + '[l] != 0.f ? 1.f : 0.f)' if r.op == 'count_nonzero' else src + '[l]'});\n"
                  f"{ind}acc{k} += t_; }}")
            elif r.op == "norm":
                w(f"{ind}{{ float t_[GM_VEC];\n#pragma unroll\n{ind}for (int l = 0; l < GM_VEC; ++l) t_[l] = gm::mul({src}[l], {src}[l]);\n{ind}acc{k} = gm::acc8({RED_OP[r.op]}, acc{k}, t_, nv{u}); }}")
            else:
                w(f"{ind}acc{k} = gm::acc8({RED_OP[r.op]}, acc{k}, {src}, nv{u});")
        for j, o in outs:
            k = self._out_slot(j)
            if hold:
                if pref is not None and pref.get(o.uid) == "P":
                    w(f"{ind}#pragma unroll\n{ind}for (int j_ = 0; j_ < 4; ++j_) ho{j}_{u}[j_] = p{o.uid}_{u}[j_];")
                else:
                    w(f"{ind}#pragma unroll\n{ind}for (int l = 0; l < GM_VEC; ++l) ho{j}_{u}[l] = n{o.uid}_{u}[l];")
                continue
            if pref is not None and pref.get(o.uid) == "P":
                w(f"{ind}gm::stg_raw(P.out[{k}], e{u}, p{o.uid}_{u});")
            else:
                w(f"{ind}gm::store8<{DT_CODE[o.dtype]}>(P.out[{k}], e{u}, nv{u}, n{o.uid}_{u});")

    def _unguarded_in(self, ip: InputPlan, p: int) -> bool:
        dnf = self._guards(p).get(ip.node.uid, frozenset({frozenset()}))
        return any(len(c) == 0 for c in dnf)

    def _exact_acc(self, r: Node) -> bool:
        """Integer-valued reductions accumulate in fp64 (exact to 2^53)."""
        return r.op in INT_REDUCE or (r.op == "sum" and not r.args[0].dtype.is_floating_point)

    def _coordsum(self, idx: str) -> str:
        """Sum of the coordinates of flat index `idx` in the iteration space."""
        S = list(self.shape)
        terms = []
        stride = 1
        for d in range(len(S) - 1, -1, -1):
            t = f"({idx} / {stride}ll)" if stride != 1 else f"({idx})"
            if d > 0:
                t = f"({t} % {S[d]}ll)"
            terms.append(t)
            stride *= S[d]
        return " + ".join(terms) if terms else "0"

    def _emit_scalar_level(self, w, level: int) -> None:
        nodes = [n for n in self.scalars if self.avail[n.uid] == level and n.op not in REDUCE]
        if not nodes:
            if level == 0:
                w("  __syncthreads();")
            return
        w("  if (threadIdx.x == 0) {")
        for n in nodes:
            w("    " + self._scalar_code(n))
        w("  }")
        w("  __syncthreads();")

    def _out_slot(self, j: int) -> int:
        k = 0
        for i, o in enumerate(self.outputs):
            if o.kind == "elem" and o.op == "free":
                continue
            if o.kind == "host":
                continue
            if i == j:
                return k
            k += 1
        raise AssertionError(j)

"""Row regions: fused kernels for arms that reduce along the innermost dim.

The purity gate admits `softmax` (data/pure_ops.cfg:18) and any torch.* call
in an arm (transform.py:265-289), and the attr_table reductions
(sum/mean/max/min, attr_table.cfg:4-7) are also written with a `dim`
(`x - x.amax(-1, keepdim=True)`, `x / x.sum(-1, keepdim=True)`).  The
grid-stride region kernel (codegen.Plan) cannot express those: its vectors
are spread over the whole grid, not over rows.  A row region is a run of
statements whose row operators (ir.ROW_OPS) all reduce the innermost dim of
one iteration space S = [..., C]:

  * a group of TPR threads owns one row (TPR a power of two, the smallest
    that keeps U = ceil(C / 8 / TPR) <= 4 vectors per thread); thread t of
    the group holds the row's vectors u*TPR + t, so the group's loads of one
    u are one contiguous stretch of the row (coalesced 128-bit accesses);
  * the whole row stays in registers: a row statistic is a per-thread
    partial, an xor-shuffle tree inside the warp and, for TPR > 32, a fixed
    order combine of the group's warps through shared memory — every thread
    of the group ends with the same value, and the elementwise code after
    it reads the row from registers (one HBM read and one write per element
    for `softmax(x * s)`, against eager's five passes);
  * values with one element per row (`x.sum(-1, keepdim=True)`, a [..., 1]
    input) are one register per thread (`rs<uid>`);
  * scalar predicates of `torch.where` (0-d tensors computed by a preceding
    grid region, host numbers) are uniform: the untaken arm's row operators
    and loads are skipped by a branch, as in the grid kernel.

A row region holds no grid-wide reduction (the lowering splits the
statements, lowering._row_mixing): the predicate statistic runs in a grid
region before it, whose 0-d output the row kernel reads.

Numerics follow torch's CPU kernels for the last dim (aten/src/ATen/native/
cpu/SoftMaxKernel.cpp `_vec_softmax_lastdim` / `_vec_log_softmax_lastdim`,
ReduceOps): max, then exp(x - max) in the input's float type (accurate expf
for fp32 outputs; for 16-bit outputs one MUFU.EX2 of x·log2 e - max·log2 e,
relative error <= 2e-6, far below their rounding — accurate expf made the
bf16 kernel ALU-bound), its sum, then
x * (1 / sum) (softmax) or x - max - log(sum) (log_softmax); sums accumulate
in fp32 per thread and fp64 across threads, rounded once to the dtype; mean
= (float)sum / C rounded once.
"""

from __future__ import annotations

import hashlib
import math
import os

import torch

from .codegen import B200_DEVICE, DT_CODE, MODE_FULL, MODE_PERIODIC, MODE_SCALAR, MODE_STRIDED, Plan, _round_f
from . import _native as nat
from .ir import ROW_NORM, ROW_OPS, ROW_RED, Graph, Node, Unsupported, infer, is_fusable_dtype, topo

MODE_ROWIN = "row"        # one value per row ([..., 1]-shaped input)


def _bcast_to(a: tuple, target: tuple) -> bool:
    try:
        return tuple(torch.broadcast_shapes(a, target)) == tuple(target)
    except RuntimeError:
        return False
UMAX = 4                  # vectors per thread (registers: U x 8 floats per live node)
MAX_TPR = 1024
CTA_THREADS = 128        # threads per row-kernel CTA (GM_ROW_CTA; 128 vs 256: softmax bf16 62.6 -> 59.6 us, fp32 neutral)


def has_row_ops(outputs: list[Node]) -> bool:
    return any(n.op in ROW_OPS for n in topo(outputs))


class RowPlan(Plan):
    """One specialisation of a row region (same interface as codegen.Plan:
    source, kernel, grid, threads, smem_bytes, inputs, outputs, scalars)."""

    def __init__(self, graph: Graph, outputs: list[Node], args: list, name: str = "region",
                 device_info: tuple[int, int] = B200_DEVICE, allow_cpu: bool = False):
        self.device_info = device_info
        self.allow_cpu = allow_cpu
        self.graph = graph
        self.outputs = outputs
        self.name = name
        infer(graph, args, outputs)
        self.order = topo(outputs)
        self.host_exact = {n.uid: self._bf16_exact(args[n.value]) for n in self.order
                           if n.op == "free" and n.kind == "host"}
        self._classify_rows(args)
        self._scalars_rows()
        self._inputs(args)
        self.hoisted = {}
        self.decisions = []
        self.spec = False
        self.stage = {ip.slot: "none" for ip in self.inputs}
        self._preloaded = {}
        self._tail = False
        self.source = self._emit_rows()
        digest = hashlib.sha1(self.source.encode()).hexdigest()[:16]
        self.kernel = f"gm_row_{digest}"
        self.source = self.source.replace("GM_KERNEL_NAME", self.kernel)

    # -- classification -----------------------------------------------------------
    def _classify_rows(self, args) -> None:
        rowops = [n for n in self.order if n.op in ROW_OPS]
        if not rowops:
            raise Unsupported("row region without a row operator")
        shapes = {tuple(n.args[0].shape) for n in rowops}
        if len(shapes) != 1:
            raise Unsupported(f"row operators over different shapes {shapes}")
        S = next(iter(shapes))
        if len(S) < 1 or math.prod(S) == 0:
            raise Unsupported("empty or 0-d row operand")
        self.shape = S
        self.C = S[-1]
        self.R = math.prod(S[:-1]) if len(S) > 1 else 1
        self.n = self.R * self.C
        keep = S[:-1] + (1,)
        nokeep = S[:-1]
        # rowval: one value per row; full: one value per element of S
        self.rowval: set[int] = set()
        read = {a.uid for n in self.order for a in n.args}
        for node in self.order:
            if node.op == "free" and node.uid not in read:
                continue  # only passed through as an output alias
            if node.kind == "elem":
                if not is_fusable_dtype(node.dtype):
                    raise Unsupported(f"elementwise dtype {node.dtype}")
                shp = tuple(node.shape)
                if node.op in ROW_RED:
                    if tuple(node.args[0].shape) != S:
                        raise Unsupported("row reduction of a non-full operand")
                    if shp == nokeep and len(S) < 2:
                        raise Unsupported("row reduction of a 1-d tensor to a 0-d one")
                    self.rowval.add(node.uid)
                    continue
                if node.op in ROW_NORM:
                    continue
                if node.op == "free":
                    t = args[node.value]
                    if t.device.type != "cuda" and not self.allow_cpu:
                        raise Unsupported("tensor not on a CUDA device")
                    if not _bcast_to(shp, S):
                        raise Unsupported("input does not broadcast to the row space")
                    if t.numel() == 1 or (len(shp) >= 1 and shp[-1] == 1 and self.C != 1):
                        self.rowval.add(node.uid)
                    continue
                elem_args = [a for a in node.args if a.kind == "elem"]
                if elem_args and all(a.uid in self.rowval for a in elem_args):
                    # computed from row values (and scalars) only
                    if shp not in (keep, nokeep) and not _bcast_to(shp, keep):
                        raise Unsupported(f"row value of shape {shp}")
                    self.rowval.add(node.uid)
                    continue
                if not _bcast_to(shp, S):
                    raise Unsupported("node does not broadcast to the row space")
                for a in elem_args:
                    if a.uid in self.rowval and tuple(a.shape) == nokeep and nokeep != keep and len(S) >= 2:
                        raise Unsupported("a keepdim=False row value broadcast against the full rows")
            elif node.kind == "dscalar":
                if any(a.kind == "elem" for a in node.args):
                    raise Unsupported("grid reduction inside a row region")
                if node.dtype not in (torch.float32, torch.bfloat16, torch.float16, torch.bool, torch.int64,
                                      torch.int32):
                    raise Unsupported(f"scalar dtype {node.dtype}")
        for o in self.outputs:
            if o.kind == "host":
                raise Unsupported("host-only output")
            if o.kind == "elem" and o.op != "free":
                if o.uid in self.rowval:
                    if tuple(o.shape) not in (keep, nokeep):
                        raise Unsupported(f"row output of shape {tuple(o.shape)}")
                elif tuple(o.shape) != S:
                    raise Unsupported("output shape differs from the row space")
        if self.n >= 2 ** 62:
            raise Unsupported("row space too large")
        # geometry
        self.vec8 = self.C % nat.VEC == 0
        nv_row = -(-self.C // nat.VEC)
        tpr = 1
        while -(-nv_row // tpr) > UMAX and tpr < MAX_TPR:
            tpr *= 2
        if -(-nv_row // tpr) > UMAX:
            raise Unsupported(f"row of {self.C} elements exceeds the on-chip row ({MAX_TPR * UMAX * 8})")
        want_u = int(os.environ.get("GM_ROW_U", "0"))
        if want_u and self.vec8 and nv_row % want_u == 0:
            # a whole number of warps per row (any multiple of 32, combined
            # through shared memory) holding want_u full vectors per thread
            t = nv_row // want_u
            if (t % 32 == 0 and t <= MAX_TPR) or (t <= 32 and t & (t - 1) == 0):
                tpr = t
        self.TPR = tpr
        self.U = -(-nv_row // tpr)
        self.full_vecs = self.vec8 and nv_row % tpr == 0
        cta = int(os.environ.get("GM_ROW_CTA", CTA_THREADS))
        self.threads = max(cta // tpr, 1) * tpr
        self.RPC = self.threads // tpr
        self.grid = -(-self.R // self.RPC)
        if self.grid >= 2 ** 31:
            raise Unsupported("too many rows")
        self.K = self.U
        # persistent CTAs looping over row groups (GM_ROW_PERSIST=1); the
        # launch clamps the grid to the co-resident CTAs
        self.persist = bool(int(os.environ.get("GM_ROW_PERSIST", "0")))
        self.smem_bytes = 0
        self.smem_off = {}
        self.minb = 1

    def _scalars_rows(self) -> None:
        self.reductions = []
        self.npass = 1
        self.avail = {}
        self.need = {}
        for node in self.order:
            if node.kind in ("host", "dscalar"):
                self.avail[node.uid] = 0
            elif node.kind == "elem":
                self.need[node.uid] = 0
        self.pass_outputs = {0: [(j, o) for j, o in enumerate(self.outputs) if o.kind == "elem" and o.op != "free"]}
        self.pass_reds = {0: []}
        self.scalars = [n for n in self.order if n.kind in ("host", "dscalar") and n.op != "const"]
        self.slot = {n.uid: i for i, n in enumerate(self.scalars)}

    def _mode(self, t: torch.Tensor) -> str:
        S = tuple(self.shape)
        if t.numel() == 1:
            return MODE_SCALAR
        shp = tuple(t.shape)
        if shp[-1:] == (1,) and S[-1] != 1:
            return MODE_ROWIN
        if shp == S and t.is_contiguous() and t.data_ptr() % 16 == 0:
            return MODE_FULL
        trail = list(shp)
        while trail and trail[0] == 1:
            trail.pop(0)
        if t.is_contiguous() and trail and tuple(trail) == S[len(S) - len(trail):] and t.data_ptr() % 16 == 0:
            return MODE_PERIODIC
        return MODE_STRIDED

    def row_offsets(self, t: torch.Tensor) -> list[tuple[int, int]]:
        """(size, element stride) of the leading dims of a [..., 1] input
        expanded to S (stride 0 where it broadcasts), outer..inner."""
        S = tuple(self.shape)
        ex = t.expand(S[:-1] + (1,)) if len(S) > 1 else t.reshape(1)
        return list(zip(S[:-1], ex.stride()[:-1])) if len(S) > 1 else []

    # -- emission ---------------------------------------------------------------------
    def _ev(self, node: Node, lane: str, u) -> str:
        if node.kind == "elem" and node.uid in self.rowval:
            return f"rs{node.uid}"
        return super()._ev(node, lane, u)

    def _uniform_select(self, node: Node, u) -> list[str]:
        c, ta, ea = node.args
        R = _round_f(node.dtype) if node.dtype != torch.bool else ""

        def val(x: Node) -> str:
            if x.kind == "elem":
                s = self._ev(x, "l", u)
                return f"{R}({s})" if (R and x.dtype != node.dtype) else s
            s = self._sf(x)
            return f"{R}({s})" if R else s

        return [
            f"if (sb{c.uid}) {{\n#pragma unroll\nfor (int l = 0; l < GM_VEC; ++l) n{node.uid}_{u}[l] = {val(ta)};\n}} "
            f"else {{\n#pragma unroll\nfor (int l = 0; l < GM_VEC; ++l) n{node.uid}_{u}[l] = {val(ea)};\n}}"
        ]

    def _free_full(self, node: Node, u: int) -> str:
        ip = self.in_by_uid[node.uid]
        dt, k = DT_CODE[ip.dtype], ip.slot
        dst = f"n{node.uid}_{u}"
        if ip.mode == MODE_FULL:
            fn = "load8_gmem" if self.vec8 else "load8_elems"
        elif ip.mode == MODE_PERIODIC:
            fn = "load8_gmem" if self.vec8 else "load8_elems"
            return f"gm::{fn}<{dt}>(P.in[{k}], pb{k} + c{u}, nv{u}, {dst});"
        else:
            fn = "load8_strided"
        return f"gm::{fn}<{dt}>(P.in[{k}], e{u}, nv{u}, {dst});"

    def _emit_rows(self) -> str:
        out: list[str] = []
        w = out.append
        U, TPR = self.U, self.TPR
        nscal = max(1, len(self.scalars))
        if self.threads != nat.THREADS:
            w(f"#define GM_THREADS {self.threads}")
        w('#include "gm_region.cuh"')
        w("#define gm_bool(x) (((x) != 0.0) ? 1.0 : 0.0)")
        w("#define gm_trunc(x) ((double)(long long)(x))")
        w(f"// row region {self.name}: rows {self.R} x {self.C}, {TPR} thread(s)/row, {U} vector(s)/thread, "
          f"{self.RPC} row(s)/CTA, grid {self.grid} x {self.threads}{'' if self.vec8 else ', per-lane access'}")
        minb = int(os.environ.get("GM_ROW_MINB", "0"))
        w(f'extern "C" __global__ void __launch_bounds__({self.threads}{", " + str(minb) if minb else ""})')
        w("GM_KERNEL_NAME(const __grid_constant__ gm::Params P) {")
        w("  using namespace gm;")
        w(f"  __shared__ double s_scal[{nscal}];")
        w(f"  __shared__ double s_rw[{max(1, self.threads // 32)}];")
        w("  (void)s_rw;")
        w('  asm volatile("griddepcontrol.wait;" ::: "memory");')
        # LayerNorm weight / bias ([C] inputs read once per row after the row
        # statistics): one cp.async copy into shared memory per CTA at kernel
        # start, in flight together with the rows' own loads, read back from
        # shared memory after the statistics — no second global round trip
        # on each row's critical path, no registers held across it
        self._smem_wb = {}
        if self.full_vecs and not os.environ.get("GM_ROW_NO_SMEM_WB"):
            per = {ip.node.uid: ip for ip in self.inputs if ip.mode == MODE_PERIODIC and ip.node.kind == "elem"
                   and self._periods.get(ip.slot) == self.C}
            users: dict = {}
            for n in self.order:
                for j, a in enumerate(n.args):
                    if a.uid in per:
                        users.setdefault(a.uid, []).append((n.op, j))
            total = 0
            for uid, us in users.items():
                ip = per[uid]
                nb = self.C * torch.empty((), dtype=ip.dtype).element_size()
                if all(op == "layer_norm" and j in (1, 2) for op, j in us) and nb % 16 == 0 and total + nb <= 32768:
                    self._smem_wb[uid] = ip
                    total += nb
            for uid, ip in self._smem_wb.items():
                nb = self.C * torch.empty((), dtype=ip.dtype).element_size()
                w(f"  __shared__ __align__(16) unsigned char swb{ip.slot}[{nb}];")
                w(f"  for (int i = threadIdx.x; i < {nb // 16}; i += {self.threads}) "
                  f"gm::cp_async16(gm::smem_u32(swb{ip.slot} + 16 * i), (const char*)P.in[{ip.slot}].ptr + 16 * i);")
            if self._smem_wb:
                w("  gm::cp_async_commit();")
        # live timer (diagnostics word bit 29, bench.py's timed loop): CTA 0
        # stamps the start, every CTA counts its exit (gm::live_exit) — the
        # kernel's own duration inside the forward's graph, no event nodes
        w("  __shared__ int s_live_;")
        w("  if (threadIdx.x == 0) {")
        w("    int f_; asm volatile(\"ld.global.u32 %0, [%1];\" : \"=r\"(f_) : \"l\"((int*)(P.barrier + GM_SCRATCH_FORCE)));")
        w("    s_live_ = (f_ & GM_LIVE_BIT) != 0;")
        w("    if (s_live_) gm::live_start(P);")
        w("  }")
        self._emit_scalar_level(w, 0)  # ends with __syncthreads: s_live_ is visible
        roots = [o for _, o in self.pass_outputs[0]]
        nodes = self._nodes(roots)
        guards = self._guards_roots(roots)
        for s in self._used_scalars(nodes, guards):
            w(f"  const float sf{s.uid} = (float)s_scal[{self.slot[s.uid]}]; (void)sf{s.uid};")
            w(f"  const bool sb{s.uid} = s_scal[{self.slot[s.uid]}] != 0.0; (void)sb{s.uid};")
            if (s.op == "free" and s.kind == "host") or (s.kind == "dscalar" and s.dtype == torch.bfloat16):
                w(f"  const u32 spk{s.uid} = gm::f2bf2(sf{s.uid}, sf{s.uid}); (void)spk{s.uid};")
        w(f"  const int tr_ = threadIdx.x % {TPR};")
        if self.persist:
            # persistent: each CTA walks row groups g_ = blockIdx.x + k·gridDim.x
            # (grid = the co-resident CTAs, region._Spec), and asks L2 for
            # its next group's rows before working on this one
            ng = self.grid
            w(f"  for (i64 g_ = blockIdx.x; g_ < {ng}ll; g_ += gridDim.x) {{")
            w(f"  {{ const i64 rn_ = (g_ + gridDim.x) * {self.RPC} + threadIdx.x / {TPR};")
            w(f"    if (rn_ < {self.R}ll) {{")
            for ip in self.inputs:
                if ip.mode == MODE_FULL and ip.node.kind == "elem" and not os.environ.get("GM_ROW_NOPF"):
                    es = torch.empty((), dtype=ip.dtype).element_size()
                    for u in range(U):
                        w(f"      asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"((const char*)P.in[{ip.slot}].ptr + "
                          f"(rn_ * {self.C}ll + ((i64){u} * {TPR} + tr_) * GM_VEC) * {es}ll));")
            w("  } }")
            blk = "g_"
        else:
            blk = "(i64)blockIdx.x"
        if os.environ.get("GM_ROW_REVERSE"):
            # last rows first: the tail of an input the previous kernel
            # swept in address order is still in L2 when the first CTAs run
            w(f"  const i64 ri_ = {blk} * {self.RPC} + threadIdx.x / {TPR};")
            w(f"  const bool rok_ = ri_ < {self.R}ll;")
            w(f"  const i64 row_ = rok_ ? {self.R - 1}ll - ri_ : 0ll;")
        else:
            w(f"  const i64 row_ = {blk} * {self.RPC} + threadIdx.x / {TPR};")
            w(f"  const bool rok_ = row_ < {self.R}ll;")
        w(f"  const i64 rb_ = row_ * {self.C}ll;")
        w("  (void)tr_; (void)rok_;")
        for u in range(U):
            w(f"  const i64 c{u} = ((i64){u} * {TPR} + tr_) * GM_VEC;")
            if self.full_vecs:
                # every vector of a row is full: lanes are valid iff the row is
                w(f"  const int nv{u} = rok_ ? GM_VEC : 0;")
            else:
                w(f"  const int nv{u} = rok_ ? (int)max(0ll, min((i64)GM_VEC, {self.C}ll - c{u})) : 0;")
            w(f"  const i64 e{u} = rb_ + c{u}; (void)e{u}; (void)nv{u};")
        # periodic inputs (a [.., C] tensor broadcast over the leading dims):
        # the row's offset into the period, once per row
        for ip in self.inputs:
            if ip.mode == MODE_PERIODIC and ip.node.kind == "elem" and ip.node in nodes:
                reps = self._periods[ip.slot] // self.C
                w(f"  const i64 pb{ip.slot} = (row_ % {reps}ll) * {self.C}ll;")
        # inputs read once per row / once per launch
        for ip in self.inputs:
            if ip.node.kind != "elem" or ip.node not in nodes:
                continue
            dt = DT_CODE[ip.dtype]
            if ip.mode == MODE_SCALAR:
                w(f"  const float rs{ip.node.uid} = gm::load_scalar<{dt}>(P.in[{ip.slot}]);")
            elif ip.mode == MODE_ROWIN:
                terms = []
                idx = "row_"
                div = 1
                for size, stride in reversed(self._row_layout[ip.slot]):
                    if stride:
                        t = f"(({idx} / {div}ll) % {size}ll) * {stride}ll" if div != 1 else f"({idx} % {size}ll) * {stride}ll"
                        terms.append(t)
                    div *= size
                off = " + ".join(terms) if terms else "0ll"
                w(f"  const float rs{ip.node.uid} = rok_ ? gm::load_at<{dt}>(P.in[{ip.slot}], {off}) : 0.f;")
        # every unguarded full-size input's vectors are loaded first
        TRUE = frozenset({frozenset()})
        first = [n for n in nodes if n.op == "free" and n.uid not in self.rowval
                 and not self._guard_expr(guards.get(n.uid, TRUE))]
        # ...except periodic inputs (a [C] weight / bias broadcast over the
        # rows: L1/L2-resident after the first rows) read only after a row
        # statistic: they load at their first consumer, so their registers
        # are not live across the row reductions (LayerNorm's weight and
        # bias: 102 -> 70 registers, 2 -> 3 CTAs per SM)
        periodic = {ip.node.uid for ip in self.inputs if ip.mode == MODE_PERIODIC and ip.node.kind == "elem"}
        late = {}
        if not os.environ.get("GM_ROW_EARLY_PERIODIC"):
            before_rowop = set()
            for n in nodes:
                if n.op in ROW_OPS:
                    break
                before_rowop.update(a.uid for a in n.args)
            late = {n.uid: n for n in first if n.uid in periodic and n.uid not in before_rowop}
            first = [n for n in first if n.uid not in late]
        self._plan_packing(nodes, roots)
        pref, needs = self._pref, self._needs
        # every value is declared here: guarded blocks only assign
        for n in nodes:
            if n.uid in self.rowval:
                if n.op != "free":
                    w(f"  float rs{n.uid} = 0.f;")
                continue
            if "F" in needs[n.uid]:
                w(f"  float {', '.join(f'n{n.uid}_{u}[GM_VEC]' for u in range(U))};")
            if "P" in needs[n.uid]:
                w(f"  u32 {', '.join(f'p{n.uid}_{u}[4]' for u in range(U))};")
        for n in first:
            self._emit_node(w, n)
        rest = [n for n in nodes if n not in first and n.uid not in late]
        cur = None
        for n in rest:
            g = self._guard_expr(guards.get(n.uid, TRUE))
            if g != cur:
                if cur:
                    w("  }")
                if g:
                    w(f"  if ({g}) {{")
                cur = g
            # a LayerNorm loads its own weight / bias after its statistics
            for a in (n.args[:1] if n.op == "layer_norm" else n.args):
                if a.uid in late:
                    self._emit_node(w, late.pop(a.uid))
            self._late = late
            self._emit_node(w, n)
        if cur:
            w("  }")
        # stores
        for j, o in self.pass_outputs[0]:
            k = self._out_slot(j)
            dt = DT_CODE[o.dtype]
            if o.uid in self.rowval:
                w(f"  if (rok_ && tr_ == 0) gm::store_at<{dt}>(P.out[{k}], row_, rs{o.uid});")
            elif pref.get(o.uid) == "P":
                for u in range(U):
                    w(f"  if (nv{u}) gm::stg_raw(P.out[{k}], e{u}, p{o.uid}_{u});")
            else:
                fn = "store8" if self.vec8 else "store8_elems"
                for u in range(U):
                    w(f"  if (nv{u}) gm::{fn}<{dt}>(P.out[{k}], e{u}, nv{u}, n{o.uid}_{u});")
        if self.persist:
            w("  }  // row groups")
        # scalar outputs and the scalar mirror (CTA 0)
        w("  if (blockIdx.x == 0 && threadIdx.x == 0) {")
        for j, o in enumerate(self.outputs):
            if o.kind == "dscalar":
                k = self._out_slot(j)
                val = self._sv(o)
                if o.dtype == torch.int64:
                    w(f"    *(long long*)P.out[{k}].ptr = (long long){val};")
                elif o.dtype == torch.int32:
                    w(f"    *(int*)P.out[{k}].ptr = (int){val};")
                else:
                    w(f"    gm::store_scalar<{DT_CODE[o.dtype]}>(P.out[{k}], {val});")
        w(f"    if (P.scal_out) for (int i = 0; i < {len(self.scalars)}; ++i) ((double*)P.scal_out)[i] = s_scal[i];")
        w("  }")
        w("  if (s_live_) {")
        w("    __syncthreads();")
        w("    if (threadIdx.x == 0) gm::live_exit(P);")
        w("  }")
        w("}")
        return "\n".join(out) + "\n"

    def _inputs(self, args) -> None:
        super()._inputs(args)
        self._row_layout = {}
        self._periods = {}
        for ip in self.inputs:
            if ip.mode == MODE_PERIODIC:
                self._periods[ip.slot] = args[ip.free_index].numel()
            if ip.mode == MODE_ROWIN:
                t = args[ip.free_index]
                self._row_layout[ip.slot] = self.row_offsets(t)

    def _plan_packing(self, nodes: list[Node], roots: list[Node]) -> None:
        """bf16 chains before / after the row operators stay packed (the
        grid kernel's bf16x2 path, codegen.Plan._packed_plan / _node_code):
        `scores * 0.125 + mask` is two `bf16x2` ops per element pair instead
        of an unpack, two fp32 ops and two roundings per element.  Values
        with one element per row stay fp32 registers.  A bf16 value that
        only a packed consumer or a store reads skips its own rounding: the
        pack (cvt.rn.bf16x2) is that rounding."""
        full = [n for n in nodes if n.uid not in self.rowval]
        pref = {n.uid: "F" for n in full}
        if self.full_vecs and not os.environ.get("GM_NO_PACKED"):
            cand = [n for n in full if n.op not in ROW_OPS]
            pp = self._packed_plan(cand)
            for n in cand:
                if n.op == "free" and n.dtype == torch.bfloat16 and self._raw_ok(n):
                    pp[n.uid] = "P"   # periodic inputs too: their vectors are aligned per row
            for n in full:
                if pp.get(n.uid) == "P" and not any(a.uid in self.rowval for a in n.args if a.kind == "elem"):
                    pref[n.uid] = "P"
        needs: dict[int, set] = {n.uid: {pref[n.uid]} for n in full}
        f_cons: dict[int, bool] = {}
        for n in nodes:
            for a in n.args:
                if a.kind != "elem" or a.uid in self.rowval:
                    continue
                if n.uid in self.rowval or n.op in ROW_OPS:
                    needs[a.uid].add("F")
                    f_cons[a.uid] = True
                elif pref[n.uid] == "P" and not (n.op == "where" and a is n.args[0]):
                    needs[a.uid].add("P")
                else:
                    needs[a.uid].add("F")
                    f_cons[a.uid] = True
        self._pref, self._needs, self._f_consumers = pref, needs, f_cons
        # stores of a bf16 / f16 F value round it themselves (cvt.rn)
        self._store_rounds = {o.uid for o in roots if o.uid not in self.rowval and pref[o.uid] == "F"
                              and o.dtype in (torch.bfloat16, torch.float16)}

    def _raw_ok(self, n: Node) -> bool:
        """A full-size / periodic input read as raw aligned vectors."""
        ip = self.in_by_uid.get(n.uid)
        return (ip is not None and self.full_vecs and ip.mode in (MODE_FULL, MODE_PERIODIC)
                and ip.dtype in (torch.float32, torch.bfloat16, torch.float16))

    def _skip_round(self, n: Node) -> bool:
        """`n`'s own rounding is redundant: every reader packs it (RN) or a
        store of the same dtype converts it (RN) — and nothing reads the
        fp32 lanes."""
        if n.dtype not in (torch.bfloat16, torch.float16) or self._f_consumers.get(n.uid):
            return False
        return "P" in self._needs[n.uid] or n.uid in self._store_rounds

    def _emit_node(self, w, n: Node) -> None:
        U = self.U
        pref, needs = self._pref, self._needs
        if n.op == "free":
            if n.uid in self.rowval:
                return  # loaded above (rs<uid>)
            ip = self.in_by_uid[n.uid]
            if self._raw_ok(n):
                # raw 16/32-byte vectors (no per-lane masking: a row is
                # either valid, every vector full, or skipped)
                dt, k = DT_CODE[ip.dtype], ip.slot
                addr = "pb{k} + c{u}" if ip.mode == MODE_PERIODIC else "e{u}"
                for u in range(U):
                    a = addr.format(k=k, u=u)
                    w(f"  gm::Raw<{dt}> rl{k}_{u} = {{}}; if (rok_) gm::rload<{dt}>(P.in[{k}], {a}, rl{k}_{u});")
                for u in range(U):
                    if "P" in needs[n.uid]:
                        w(f"#pragma unroll\n  for (int j = 0; j < 4; ++j) p{n.uid}_{u}[j] = rl{k}_{u}.w[j];")
                    if "F" in needs[n.uid]:
                        w(f"  gm::rcvt<{dt}>(rl{k}_{u}, n{n.uid}_{u});")
                return
            for u in range(U):
                w("  " + self._free_full(n, u))
                if "P" in needs[n.uid]:
                    w(f"  gm::pack8(n{n.uid}_{u}, p{n.uid}_{u});")
            return
        if n.op in ROW_RED:
            self._emit_row_reduce(w, n)
            return
        if n.op in ROW_NORM:
            self._emit_row_norm(w, n)
            if "P" in needs[n.uid]:
                for u in range(U):
                    w(f"  gm::pack8(n{n.uid}_{u}, p{n.uid}_{u});")
            return
        if n.uid in self.rowval:
            # one value per row: computed once per thread
            w("  {")
            w(f"  float n{n.uid}_r[GM_VEC];")
            for line in self._elem_code(n, "r"):
                w("  " + line.replace("\n", "\n  "))
            w(f"  rs{n.uid} = n{n.uid}_r[0];")
            w("  }")
            return
        for u in range(U):
            if pref[n.uid] == "F":
                self._no_round = self._skip_round(n)
                try:
                    lines = self._elem_code(n, u)
                finally:
                    self._no_round = False
                if "P" in needs[n.uid]:
                    lines.append(f"gm::pack8(n{n.uid}_{u}, p{n.uid}_{u});")
            else:
                lines = self._node_code(n, u, pref, needs)
            for line in lines:
                w("  " + line.replace("\n", "\n  "))

    def _row_stat(self, w, name: str, x: Node, op: str, expr=None) -> None:
        """float `name` = the row's max/min (NaN-propagating) or sum of
        expr(x lane) over its valid lanes; sums: fp32 per thread, fp64 across
        threads, rounded once to fp32."""
        U, TPR = self.U, self.TPR
        ident = {"max": "__int_as_float(0xff800000)", "fmax": "__int_as_float(0xff800000)",
                 "min": "__int_as_float(0x7f800000)", "sum": "0.f"}[op]
        w(f"  float {name}_t = {ident}; (void){name}_t;")
        for u in range(U):
            v = f"n{x.uid}_{u}[l]" if expr is None else expr(u)
            if op == "sum":
                upd = f"{name}_t = gm::add({name}_t, {v});"
            elif op == "fmax":
                upd = f"{name}_t = fmaxf({name}_t, {v});"
            else:
                upd = f"{name}_t = gm::n{op}({name}_t, {v});"
            # full vectors: every lane of a valid row is valid, and an
            # invalid row (past R, loads read 0) is never stored
            mask = "" if self.full_vecs else f"if (l < nv{u}) "
            w(f"#pragma unroll\n  for (int l = 0; l < GM_VEC; ++l) {mask}{upd}")
        code = {"sum": "GM_R_SUM", "max": "GM_R_MAX", "fmax": "GM_R_MAX", "min": "GM_R_MIN"}[op]
        w(f"  const float {name} = (float)gm::row_combine<{TPR}, {code}>((double){name}_t, s_rw);")

    def _emit_row_reduce(self, w, n: Node) -> None:
        x = n.args[0]
        fn = ROW_RED[n.op]
        R = _round_f(n.dtype)
        if fn in ("amax", "amin"):
            self._row_stat(w, f"st{n.uid}", x, "max" if fn == "amax" else "min")
            w(f"  rs{n.uid} = st{n.uid};")
            return
        if x.dtype == torch.bool:
            raise Unsupported("row sum of a bool tensor")
        self._row_stat(w, f"st{n.uid}", x, "sum")
        if fn in ("var", "std"):
            # two passes over the row held in registers: mean, then the sum
            # of squared deviations (torch's CPU var is a Welford / two-pass
            # equivalent), divided by C - correction
            corr = n.value[2]
            w(f"  const float mu{n.uid} = __fdiv_rn(st{n.uid}, {float(self.C)!r}f);")
            self._row_stat(w, f"sq{n.uid}", x, "sum",
                           expr=lambda u: f"gm::mul(gm::sub(n{x.uid}_{u}[l], mu{n.uid}), gm::sub(n{x.uid}_{u}[l], mu{n.uid}))")
            den = float(max(self.C - corr, 0))
            val = f"__fdiv_rn(sq{n.uid}, {den!r}f)"
            if fn == "std":
                val = f"gm::fsqrt({val})"
        else:
            val = f"st{n.uid}" if fn == "sum" else f"__fdiv_rn(st{n.uid}, {float(self.C)!r}f)"
        w(f"  rs{n.uid} = {R}({val});" if R else f"  rs{n.uid} = {val};")

    def _emit_row_norm(self, w, n: Node) -> None:
        x = n.args[0]
        U = self.U
        R = _round_f(n.dtype)
        if n.op == "layer_norm":
            # torch's CPU LayerNorm: mean, rstd = 1 / sqrt(var + eps), then
            # (x * rstd + (-rstd * mean)) * weight + bias, in fp32
            if self._skip_round(n):
                R = ""
            wt, bs = n.args[1], n.args[2]
            self._row_stat(w, f"ls{n.uid}", x, "sum")
            w(f"  const float mu{n.uid} = __fdiv_rn(ls{n.uid}, {float(self.C)!r}f);")
            self._row_stat(w, f"lq{n.uid}", x, "sum",
                           expr=lambda u: f"gm::mul(gm::sub(n{x.uid}_{u}[l], mu{n.uid}), gm::sub(n{x.uid}_{u}[l], mu{n.uid}))")
            w(f"  const float rstd{n.uid} = __frcp_rn(gm::fsqrt(gm::add(__fdiv_rn(lq{n.uid}, {float(self.C)!r}f), "
              f"{float(n.value[2])!r}f)));")
            w(f"  const float bia{n.uid} = gm::mul(-rstd{n.uid}, mu{n.uid});")
            late = getattr(self, "_late", {})
            staged = [a for a in (wt, bs) if a.uid in late and a.uid in self._smem_wb]
            if staged:
                w("  gm::cp_async_wait_all();")
                w("  __syncthreads();")
            for a in (wt, bs):
                if a.uid in late:
                    if a.uid in self._smem_wb:
                        late.pop(a.uid)
                        ip = self._smem_wb[a.uid]
                        dt, es = DT_CODE[ip.dtype], torch.empty((), dtype=ip.dtype).element_size()
                        for u in range(U):
                            w(f"  gm::Raw<{dt}> rl{ip.slot}_{u} = *(const gm::Raw<{dt}>*)(swb{ip.slot} + c{u} * {es});")
                            w(f"  gm::rcvt<{dt}>(rl{ip.slot}_{u}, n{a.uid}_{u});")
                    else:
                        self._emit_node(w, late.pop(a.uid))
            for u in range(U):
                wv = self._ev(wt, "l", u) if wt.kind == "elem" else self._sf(wt)
                bv = self._ev(bs, "l", u) if bs.kind == "elem" else self._sf(bs)
                body = (f"gm::add(gm::mul(gm::add(gm::mul(n{x.uid}_{u}[l], rstd{n.uid}), bia{n.uid}), {wv}), {bv})")
                w(f"#pragma unroll\n  for (int l = 0; l < GM_VEC; ++l) n{n.uid}_{u}[l] = {R}({body});" if R else
                  f"#pragma unroll\n  for (int l = 0; l < GM_VEC; ++l) n{n.uid}_{u}[l] = {body};")
            return
        if self._skip_round(n):
            R = ""
        m = f"mx{n.uid}"
        # the shift needs no NaN propagation: a NaN lane makes exp(x - m) and
        # so the row's sum NaN, and every output NaN, as torch's propagating
        # max does (one FMNMX per element instead of a compare and select)
        self._row_stat(w, m, x, "fmax")
        if n.op == "softmax" and n.dtype != torch.float32:
            # 16-bit outputs: exp(x - max) = 2^(x·log2 e - max·log2 e), one
            # FFMA + one MUFU.EX2 (the bf16 rounding dwarfs its ~2e-6 error;
            # accurate expf made the bf16 kernel ALU-bound).  fp32 keeps
            # torch's own sequence, x - max then an accurate expf: the fp32
            # kernel is HBM-bound either way, and programs that threshold or
            # deduplicate softmax outputs (moe_minicpm_like's nonzero /
            # unique of x > 0.05) flip far fewer decisions
            w(f"  const float ml{n.uid} = gm::mul({m}, 1.4426950408889634f);")
            for u in range(U):
                w(f"#pragma unroll\n  for (int l = 0; l < GM_VEC; ++l) n{n.uid}_{u}[l] = "
                  f"gm::ex2(__fmaf_rn(n{x.uid}_{u}[l], 1.4426950408889634f, -ml{n.uid}));")
        else:
            ex = "expf" if n.dtype == torch.float32 else "gm::fexp"
            for u in range(U):
                w(f"#pragma unroll\n  for (int l = 0; l < GM_VEC; ++l) n{n.uid}_{u}[l] = "
                  f"{ex}(gm::sub(n{x.uid}_{u}[l], {m}));")
        s = f"sm{n.uid}"
        self._row_stat(w, s, n, "sum")
        if n.op == "softmax":
            w(f"  const float iv{n.uid} = gm::div(1.f, {s});")
            body = f"gm::mul(n{n.uid}_{{u}}[l], iv{n.uid})"
        else:
            w(f"  const float ls{n.uid} = logf({s});")
            body = f"gm::sub(gm::sub(n{x.uid}_{{u}}[l], {m}), ls{n.uid})"
        for u in range(U):
            b = body.format(u=u)
            w(f"#pragma unroll\n  for (int l = 0; l < GM_VEC; ++l) n{n.uid}_{u}[l] = {R}({b});" if R else
              f"#pragma unroll\n  for (int l = 0; l < GM_VEC; ++l) n{n.uid}_{u}[l] = {b};")

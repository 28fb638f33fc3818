"""Source-level lowering of a GraphMend-transformed program for B200.

Input: the text `fix_file` returns (transform.py:822-936) — the reference
transform API is unchanged and is not re-implemented here.  Output: the same
program where

  * every maximal run of fusable straight-line assignments (predicate
    bindings `__gm_pred_k = ...`, arm temporaries `__gm_then_T_k` /
    `__gm_else_T_k`, the `T = torch.where(...)` selects, return hoists
    `__gm_ret_k = ...` and ordinary elementwise statements around them)
    becomes ONE call of a fused region (region.py): the predicate reduction,
    the selected arm and the select run in one sm_100a kernel and only the
    names read later are materialised;
  * every deferred replay `callee(*__gm_defer_k)` (transform.py:707-708,
    :729-731) becomes `__gm_rt.replay(site, callee, __gm_defer_k)`, which
    hands tensor arguments to the device log ring (logring.py) instead of
    formatting (and synchronising on) them inside the forward;
  * capture tuples `__gm_defer_k = (...)` whose elements do not depend on the
    current region are hoisted above it, so deferral sites do not split
    regions (the tuple holds references, transform.py:748-753).

Statements outside the fusable subset are left untouched and run as
PyTorch ops on the device (cuBLAS for Linear/matmul, per `north_star`).
"""

from __future__ import annotations

import ast
import copy
import itertools
import linecache
import types
from dataclasses import dataclass, field

from .ir import ITEM, NZSUM, REDUCE, ROW_OPS, Builder, Graph, Unsupported, attr_chain
from .region import Region

GM_RT = "__gm_rt__"  # dunder suffix: exempt from private-name mangling in class bodies
_module_ids = itertools.count()


@dataclass
class ReplaySite:
    site: int
    callee_src: str
    capture_name: str
    function: str
    lineno: int


@dataclass
class Lowered:
    original: str
    source: str
    regions: list[Region] = field(default_factory=list)
    sites: list[ReplaySite] = field(default_factory=list)
    region_sources: list[str] = field(default_factory=list)
    dynamic_shape_lowered: list = field(default_factory=list)
    gemm_arms: list = field(default_factory=list)


def _torch_aliases(tree: ast.Module) -> tuple[set[str], set[str]]:
    torch_names: set[str] = set()
    functional: set[str] = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            for a in node.names:
                if a.name == "torch":
                    torch_names.add(a.asname or "torch")
                elif a.name == "torch.nn.functional" and a.asname:
                    functional.add(a.asname)
                elif a.name.startswith("torch.") and not a.asname:
                    torch_names.add("torch")
        elif isinstance(node, ast.ImportFrom) and node.module in ("torch.nn", "torch.nn.functional"):
            for a in node.names:
                if node.module == "torch.nn" and a.name == "functional":
                    functional.add(a.asname or "functional")
    return torch_names or {"torch"}, functional


def _layer_norm_attrs(cls: ast.ClassDef, torch_names: set[str], nn_names: set[str]) -> dict[str, float]:
    """`self.X = torch.nn.LayerNorm(n[, eps=c])` at the top level of the
    class's `__init__`, X assigned nowhere else in the class and the shape a
    single dimension (an int, or a one-element tuple / list): {X: eps}."""
    stores: dict[str, int] = {}
    for node in ast.walk(cls):
        if isinstance(node, (ast.Assign, ast.AnnAssign, ast.AugAssign, ast.Delete)):
            targets = node.targets if isinstance(node, (ast.Assign, ast.Delete)) else [node.target]
            for t in targets:
                for sub in ast.walk(t):
                    if isinstance(sub, ast.Attribute) and isinstance(sub.value, ast.Name) and sub.value.id == "self":
                        stores[sub.attr] = stores.get(sub.attr, 0) + 1
        if isinstance(node, ast.Call) and isinstance(node.func, ast.Name) and node.func.id in ("setattr", "delattr"):
            return {}
    init = next((f for f in cls.body if isinstance(f, ast.FunctionDef) and f.name == "__init__"), None)
    if init is None:
        return {}
    found: dict[str, float] = {}
    for st in init.body:
        if not (isinstance(st, ast.Assign) and len(st.targets) == 1 and isinstance(st.targets[0], ast.Attribute)
                and isinstance(st.targets[0].value, ast.Name) and st.targets[0].value.id == "self"
                and isinstance(st.value, ast.Call)):
            continue
        chain = attr_chain(st.value.func)
        if not (chain and chain[-1] == "LayerNorm"
                and ((len(chain) == 3 and chain[0] in torch_names and chain[1] == "nn")
                     or (len(chain) == 2 and chain[0] in nn_names))):
            continue
        c = st.value
        if len(c.args) != 1 or isinstance(c.args[0], ast.Starred):
            continue
        a0 = c.args[0]
        if isinstance(a0, (ast.Tuple, ast.List)) and len(a0.elts) != 1:
            continue
        eps, ok = 1e-5, True
        for k in c.keywords:
            v = k.value
            if k.arg == "eps" and isinstance(v, ast.Constant) and isinstance(v.value, (int, float)) \
                    and not isinstance(v.value, bool):
                eps = float(v.value)
            elif k.arg in ("elementwise_affine", "bias") and isinstance(v, ast.Constant) and v.value is True:
                pass
            elif k.arg not in ("device", "dtype"):
                ok = False
        if ok:
            found[st.targets[0].attr] = eps
    return {x: e for x, e in found.items() if stores.get(x) == 1}


def _inline_layer_norms(tree: ast.Module, torch_names: set[str]) -> list[str]:
    """`self.X(e)` with X an nn.LayerNorm the class builds in `__init__`
    becomes `F.layer_norm(e, self.X.normalized_shape, self.X.weight,
    self.X.bias, eps)` in the class's other methods — the form Dynamo's FX
    graph has — so a residual add before a post-LayerNorm fuses with it into
    one row region (`self.norm(self.out(h) + x)`: GEMM, then ONE kernel).  A
    guard at the top of each rewritten method (ModuleRuntime.
    inlined_layer_norms) raises if such an attribute is later replaced or
    given hooks.  Returns the rewritten `Class.X` names."""
    nn_names = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.ImportFrom) and node.module == "torch":
            nn_names |= {a.asname or a.name for a in node.names if a.name == "nn"}
        if isinstance(node, ast.Import):
            nn_names |= {a.asname for a in node.names if a.name == "torch.nn" and a.asname}
    tname = "torch" if "torch" in torch_names else sorted(torch_names)[0]
    done = []
    for cls in [n for n in ast.walk(tree) if isinstance(n, ast.ClassDef)]:
        attrs = _layer_norm_attrs(cls, torch_names, nn_names)
        if not attrs:
            continue

        class _Sub(ast.NodeTransformer):
            used: set = set()

            def visit_Call(self, node):
                self.generic_visit(node)
                f = node.func
                if (isinstance(f, ast.Attribute) and isinstance(f.value, ast.Name) and f.value.id == "self"
                        and f.attr in attrs and len(node.args) == 1 and not node.keywords
                        and not isinstance(node.args[0], ast.Starred)):
                    self.used.add(f.attr)
                    me = lambda a: ast.Attribute(ast.Attribute(ast.Name("self", ast.Load()), f.attr, ast.Load()),  # noqa: E731
                                                 a, ast.Load())
                    fn = ast.Attribute(ast.Attribute(ast.Attribute(ast.Name(tname, ast.Load()), "nn", ast.Load()),
                                                     "functional", ast.Load()), "layer_norm", ast.Load())
                    return ast.copy_location(ast.Call(fn, [node.args[0], me("normalized_shape"), me("weight"),
                                                           me("bias"), ast.Constant(attrs[f.attr])], []), node)
                return node

        for fn in cls.body:
            if not isinstance(fn, ast.FunctionDef) or fn.name == "__init__":
                continue
            sub = _Sub()
            sub.used = set()
            fn.body = [sub.visit(st) for st in fn.body]
            if sub.used:
                names = sorted(sub.used)
                guard = ast.Expr(ast.Call(ast.Attribute(ast.Name(GM_RT, ast.Load()), "inlined_layer_norms",
                                                        ast.Load()),
                                          [ast.Name("self", ast.Load()),
                                           ast.Tuple([ast.Constant(n) for n in names], ast.Load())], []))
                fn.body.insert(0, ast.copy_location(guard, fn.body[0]))
                done += [f"{cls.name}.{n}" for n in names]
    ast.fix_missing_locations(tree)
    return done


def _is_capture(stmt: ast.stmt) -> str | None:
    if (
        isinstance(stmt, ast.Assign)
        and len(stmt.targets) == 1
        and isinstance(stmt.targets[0], ast.Name)
        and stmt.targets[0].id.startswith("__gm_defer_")
        and isinstance(stmt.value, ast.Tuple)
    ):
        return stmt.targets[0].id
    return None


def _is_replay(stmt: ast.stmt) -> tuple[ast.expr, str] | None:
    if not (isinstance(stmt, ast.Expr) and isinstance(stmt.value, ast.Call)):
        return None
    call = stmt.value
    if call.keywords or len(call.args) != 1 or not isinstance(call.args[0], ast.Starred):
        return None
    inner = call.args[0].value
    if isinstance(inner, ast.Name) and inner.id.startswith("__gm_defer_"):
        return call.func, inner.id
    return None


_DYN_OPS = {"nonzero", "unique", "masked_select"}   # data/dynamic_shape_ops.cfg


def _dyn_def(stmt: ast.stmt, torch_names: set[str]):
    """`V = torch.nonzero(M)` / `M.nonzero()` / `X.unique()` / `torch.unique(X)` /
    `torch.masked_select(X, M)` / `X.masked_select(M)` -> (V, op, operand exprs)."""
    if not (isinstance(stmt, ast.Assign) and len(stmt.targets) == 1 and isinstance(stmt.targets[0], ast.Name)
            and isinstance(stmt.value, ast.Call) and not stmt.value.keywords):
        return None
    call = stmt.value
    f = call.func
    if not isinstance(f, ast.Attribute) or f.attr not in _DYN_OPS:
        return None
    if isinstance(f.value, ast.Name) and f.value.id in torch_names:
        operands = list(call.args)
    else:
        operands = [f.value] + list(call.args)
    want = {"nonzero": 1, "unique": 1, "masked_select": 2}[f.attr]
    if len(operands) != want:
        return None
    return stmt.targets[0].id, f.attr, operands


def _row_mixing(g: Graph) -> bool:
    """A run may hold grid-wide reductions (one grid region, codegen.Plan) or
    row operators (one row region, rowgen.RowPlan), not both: a predicated
    block `p = x.sum() > 0; t = softmax(x, -1); y = where(p, t, x)` becomes a
    grid region for `p` followed by a row region that reads it."""
    ops = {n.op for n in g.nodes}
    return bool(ops & ROW_OPS) and bool(ops & (REDUCE | {NZSUM}))


def _names_read(node: ast.AST) -> set[str]:
    return {n.id for n in ast.walk(node) if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Load)}


class _FunctionLowerer:
    def __init__(self, owner: "_Lowerer", fn: ast.FunctionDef):
        self.owner = owner
        self.fn = fn
        # every Name load of the function with its position (for liveness)
        self.loads: list[tuple[tuple[int, int], str]] = [
            ((n.lineno, n.col_offset), n.id)
            for n in ast.walk(fn)
            if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Load)
        ]
        # names a deferred scope may read whenever it runs (a lambda / nested
        # def / class body defined anywhere in the function, or a name
        # declared global / nonlocal): never dead, whatever their position
        self.always_live: set[str] = set()
        for n in ast.walk(fn):
            if n is fn:
                continue
            if isinstance(n, (ast.Lambda, ast.FunctionDef, ast.AsyncFunctionDef, ast.ClassDef)):
                self.always_live |= {m.id for m in ast.walk(n) if isinstance(m, ast.Name)}
            elif isinstance(n, (ast.Global, ast.Nonlocal)):
                self.always_live |= set(n.names)

    def read_after(self, name: str, pos: tuple[int, int]) -> bool:
        return name in self.always_live or any(p > pos and n == name for p, n in self.loads)

    # -- region formation -------------------------------------------------------
    def _build(self, stmts: list[ast.stmt]) -> tuple[Graph, Builder]:
        g = Graph()
        b = Builder(g, self.owner.torch_names, self.owner.functional_names)
        for s in stmts:
            node = b.expr(s.value)
            b.env[s.targets[0].id] = node
        return g, b

    def _eligible(self, stmt: ast.stmt) -> bool:
        return (
            isinstance(stmt, ast.Assign)
            and len(stmt.targets) == 1
            and isinstance(stmt.targets[0], ast.Name)
            and not stmt.targets[0].id.startswith("__gm_defer_")
        )

    def _try_extend(self, run: list[ast.stmt], stmt: ast.stmt) -> bool:
        if not self._eligible(stmt):
            return False
        try:
            g, _ = self._build(run + [stmt])
        except Unsupported:
            return False
        return not _row_mixing(g)

    def _lower_dynamic_shape(self, stmts: list[ast.stmt]) -> list[ast.stmt]:
        """a dynamic-shape op whose only consumer is a full
        `.sum()` is replaced by a fixed-shape reduction, so no host sync is
        needed to size its output (the reference reports these sites
        unfixable, data/dynamic_shape_ops.cfg; the counts stay the reference's):
          nonzero(M).sum()          -> __gm_rt__.nonzero_sum(M)   (fused coordinate sum)
          masked_select(X, M).sum() -> torch.where(M, X, 0).sum() (fused)
          X.unique().sum()          -> __gm_rt__.unique_sum(X)    (distinct-value sum kernels)
        The replacement is evaluated AT THE DEFINITION SITE (`V = op(X)` becomes
        `__gm_s_k = <fixed-shape sum>`) and the use `V.sum()` reads
        `__gm_s_k`, so names of X rebound or mutated between the definition
        and the use cannot change the result."""
        torch_name = sorted(self.owner.torch_names)[0]
        out = list(stmts)
        i = 0
        while i < len(out):
            d = _dyn_def(out[i], self.owner.torch_names)
            if d is None:
                i += 1
                continue
            var, op, operands = d
            loads = [n for n in ast.walk(self.fn) if isinstance(n, ast.Name) and n.id == var]
            stores = [n for n in loads if isinstance(n.ctx, ast.Store)]
            uses = [n for n in loads if isinstance(n.ctx, ast.Load)]
            if len(stores) != 1 or len(uses) != 1:
                i += 1
                continue
            if op == "nonzero":
                repl = ast.Call(ast.Attribute(ast.Name(GM_RT, ast.Load()), "nonzero_sum", ast.Load()),
                                [operands[0]], [])
            elif op == "unique":
                repl = ast.Call(ast.Attribute(ast.Name(GM_RT, ast.Load()), "unique_sum", ast.Load()),
                                [operands[0]], [])
            else:
                where = ast.Call(ast.Attribute(ast.Name(torch_name, ast.Load()), "where", ast.Load()),
                                 [operands[1], operands[0], ast.Constant(0)], [])
                repl = ast.Call(ast.Attribute(where, "sum", ast.Load()), [], [])
            target = uses[0]
            sname = f"__gm_s_{self.owner.next_tmp()}"

            class _Sub(ast.NodeTransformer):
                done = 0

                def visit_Call(self, node):
                    f = node.func
                    if (isinstance(f, ast.Attribute) and f.attr == "sum" and f.value is target
                            and not node.args and not node.keywords):
                        _Sub.done += 1
                        return ast.copy_location(ast.Name(sname, ast.Load()), node)
                    return self.generic_visit(node)

            new_tail = [_Sub().visit(s) for s in out[i + 1:]]
            if _Sub.done != 1:
                i += 1
                continue
            self.owner.dyn_lowered.append((var, op))
            defn = ast.copy_location(ast.Assign(targets=[ast.Name(sname, ast.Store())], value=repl), out[i])
            defn.end_lineno, defn.end_col_offset = out[i].end_lineno, out[i].end_col_offset
            self.loads.append(((target.lineno, target.col_offset), sname))
            out = out[:i] + [defn] + new_tail
            ast.fix_missing_locations(self.fn)
            i += 1
        return out

    def _rematerialise(self, stmts: list[ast.stmt]) -> list[ast.stmt]:
        """A cheap elementwise value read both by a grid reduction and by a
        row operator (`scores = t / 8.0; p = scores.abs().mean() > c;
        probs = softmax(scores + bias, -1)`) would be written to HBM by the
        grid region and read back by the row region that follows it
        (lowering._row_mixing splits them).  It is substituted into its uses
        instead — each region recomputes it from its inputs, with the same
        operators in the same order (identical values), and the full-size
        intermediate is never materialised.  Only single-assignment names
        whose every read is in a later top-level statement of this block,
        with inputs not rebound before the last read."""
        out = list(stmts)
        i = 0
        while i < len(out):
            s = out[i]
            if not self._eligible(s) or s.targets[0].id in self.always_live:
                i += 1
                continue
            V = s.targets[0].id
            try:
                g, _ = self._build([s])
            except Unsupported:
                i += 1
                continue
            ops = [n.op for n in g.nodes if n.op not in ("free", "const")]
            if not ops or len(ops) > 8 or set(ops) & (REDUCE | ROW_OPS | {NZSUM, ITEM}) \
                    or any("[" in fv.text for fv in g.frees):
                i += 1
                continue
            names = [n for n in ast.walk(self.fn) if isinstance(n, ast.Name) and n.id == V]
            if sum(isinstance(n.ctx, ast.Store) for n in names) != 1:
                i += 1
                continue
            uses = [j for j in range(i + 1, len(out)) if V in _names_read(out[j])]
            n_loads = sum(isinstance(n.ctx, ast.Load) for n in names)
            if not uses or sum(sum(1 for n in ast.walk(out[j]) if isinstance(n, ast.Name) and n.id == V
                                   and isinstance(n.ctx, ast.Load)) for j in uses) != n_loads:
                i += 1
                continue
            roots = {fv.text.split(".")[0] for fv in g.frees}
            rebound = {n.id for t in out[i + 1:max(uses) + 1] for n in ast.walk(t)
                       if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Store)}
            if roots & rebound:
                i += 1
                continue
            kinds, direct = self._use_kinds(out, i, V, 0)
            # read (through cheap elementwise statements) by both a grid
            # reduction and a row operator; or an elementwise producer whose
            # every read is a row operator's statement (`add = scores + bias;
            # p = softmax(add, -1)`, the FX graph's one-op-per-line form):
            # the row region computes it instead of the region before it
            # writing it out
            if "other" in direct or not ({"row", "grid"} <= kinds or direct == {"row"}):
                i += 1
                continue
            expr = s.value

            class _Sub(ast.NodeTransformer):
                def visit_Name(self, node):
                    if node.id == V and isinstance(node.ctx, ast.Load):
                        e = copy.deepcopy(expr)
                        for sub in ast.walk(e):
                            if hasattr(sub, "lineno"):
                                ast.copy_location(sub, node)
                        return e
                    return node

            for j in uses:
                out[j] = _Sub().visit(out[j])
                pos = (out[j].lineno, out[j].col_offset + 1)
                self.loads.extend((pos, r) for r in _names_read(expr))
            self.owner.rematerialised.append(V)
            del out[i]
        return out

    def _use_kinds(self, out: list[ast.stmt], i: int, V: str, depth: int) -> tuple[set, set]:
        """What reads the value `V` assigned by out[i]: ({"row", "grid",
        "other"} over its reads, followed through single-target elementwise
        statements, {...} over its direct reads only)."""
        kinds, direct = set(), set()
        for j in range(i + 1, len(out)):
            if V not in _names_read(out[j]):
                continue
            if not self._eligible(out[j]):
                kinds.add("other")
                direct.add("other")
                continue
            try:
                gj, _ = self._build([out[j]])
            except Unsupported:
                kinds.add("other")
                direct.add("other")
                continue
            oj = {n.op for n in gj.nodes}
            k = set()
            if oj & ROW_OPS:
                k.add("row")
            if oj & (REDUCE | {NZSUM, ITEM}):
                k.add("grid")
            direct |= k or {"elem"}
            kinds |= k
            W = out[j].targets[0].id
            if not k and depth < 8 and W not in self.always_live:
                kinds |= self._use_kinds(out, j, W, depth + 1)[0]
            if isinstance(out[j], ast.Assign) and V in {t.id for t in out[j].targets if isinstance(t, ast.Name)}:
                break                                       # V rebound: later reads are another value
        return kinds, direct

    def _fusable(self, e: ast.expr) -> bool:
        try:
            Builder(Graph(), self.owner.torch_names, self.owner.functional_names).expr(e)
        except Unsupported:
            return False
        return True

    def _split_calls(self, stmts: list[ast.stmt]) -> list[ast.stmt]:
        """`x = f(g(y)) + z` with g non-fusable (a module or library call,
        e.g. a Linear on cuBLAS) and the rest elementwise becomes
        `__gm_t_k = g(y); x = f(__gm_t_k) + z`, so the elementwise remainder
        joins a fused region instead of running as separate PyTorch ops.
        Hoisted calls keep their left-to-right order; what is left around
        them is pure (fusable), so evaluation order is unchanged."""
        out: list[ast.stmt] = []
        for s in stmts:
            if not self._eligible(s) or self._fusable(s.value):
                out.append(s)
                continue
            temps: list[ast.stmt] = []

            def split(e: ast.expr) -> ast.expr:
                if self._fusable(e):
                    return e
                lr = self._linear_relu(e)
                if lr is not None:
                    e = lr
                if isinstance(e, ast.BinOp) and not isinstance(e.op, ast.MatMult):
                    return ast.BinOp(split(e.left), e.op, split(e.right))
                if isinstance(e, ast.UnaryOp):
                    return ast.UnaryOp(e.op, split(e.operand))
                if isinstance(e, ast.Call) and not e.keywords and not any(isinstance(a, ast.Starred) for a in e.args):
                    n_temps = len(temps)
                    args = [split(a) for a in e.args]
                    cand = ast.Call(e.func, args, [])
                    if self._fusable(cand):
                        return cand
                    if attr_chain(e.func) is not None and attr_chain(e.func)[0] == "self":
                        # a module call `self.m(<fusable expr>)`: the argument
                        # becomes its own statement (a fused region: e.g. the
                        # residual add before a LayerNorm) and the call reads it
                        hoisted = []
                        for a in args:
                            if self._fusable(a) and not isinstance(a, (ast.Name, ast.Constant)):
                                tn = f"__gm_t_{self.owner.next_tmp()}"
                                temps.append(ast.copy_location(ast.Assign(targets=[ast.Name(tn, ast.Store())],
                                                                          value=a), s))
                                # read by the call, which follows the temp's statement
                                self.loads.append(((s.end_lineno, s.end_col_offset + 1), tn))
                                hoisted.append(ast.Name(tn, ast.Load()))
                            else:
                                hoisted.append(a)
                        e = ast.Call(e.func, hoisted, [])
                    else:
                        # the call itself is hoisted: its arguments as written
                        # (temporaries made for them would be dead)
                        del temps[n_temps:]
                name = f"__gm_t_{self.owner.next_tmp()}"
                temps.append(ast.copy_location(ast.Assign(targets=[ast.Name(name, ast.Store())], value=e), s))
                self.loads.append(((s.lineno, s.col_offset + 1), name))
                return ast.Name(name, ast.Load())

            new_value = split(s.value)
            if len(temps) == 1 and isinstance(new_value, ast.Name) and isinstance(temps[0].value, ast.Call) \
                    and ast.unparse(temps[0].value.func) == f"{GM_RT}.linear_relu":
                # the whole statement was relu(Linear(x))
                res = ast.copy_location(ast.Assign(targets=s.targets, value=temps[0].value), s)
                res.end_lineno, res.end_col_offset = s.end_lineno, s.end_col_offset
                out.append(res)
                continue
            if (isinstance(new_value, ast.Name) and len(temps) > 1 and isinstance(temps[-1].targets[0], ast.Name)
                    and temps[-1].targets[0].id == new_value.id):
                # the statement is a call whose arguments were hoisted (a
                # module call on a fusable expression): the argument
                # statements, then the call assigned to the original target
                res = ast.copy_location(ast.Assign(targets=s.targets, value=temps[-1].value), s)
                res.end_lineno, res.end_col_offset = s.end_lineno, s.end_col_offset
                ast.fix_missing_locations(res)
                out.extend(temps[:-1] + [res])
                continue
            if not temps or isinstance(new_value, ast.Name) or not self._fusable(new_value):
                out.append(s)
                continue
            res = ast.copy_location(ast.Assign(targets=s.targets, value=new_value), s)
            res.end_lineno, res.end_col_offset = s.end_lineno, s.end_col_offset
            ast.fix_missing_locations(res)
            out.extend(temps + [res])
        return out

    def _linear_relu(self, e: ast.expr) -> ast.expr | None:
        """`relu(m(x))` with m a module call -> `__gm_rt__.linear_relu(m, x)`:
        for an nn.Linear on CUDA one cuBLASLt GEMM with the RELU_BIAS
        epilogue (relu commutes with the output rounding, so the value is
        relu(Linear(x))); otherwise the runtime falls back to relu(m(x))."""
        mods = self.owner.torch_names | self.owner.functional_names
        if not (isinstance(e, ast.Call) and isinstance(e.func, ast.Attribute) and e.func.attr == "relu"
                and isinstance(e.func.value, ast.Name) and e.func.value.id in mods
                and len(e.args) == 1 and not e.keywords):
            return None
        inner = e.args[0]
        if not (isinstance(inner, ast.Call) and len(inner.args) == 1 and not inner.keywords
                and not isinstance(inner.args[0], ast.Starred) and attr_chain(inner.func) is not None
                and attr_chain(inner.func)[0] not in mods and not self._fusable(inner)):
            return None
        return ast.Call(ast.Attribute(ast.Name(GM_RT, ast.Load()), "linear_relu", ast.Load()),
                        [inner.func, inner.args[0]], [])

    # -- dense contractions -----------------------------------------------------
    def _gemm_call(self, e: ast.expr) -> ast.expr | None:
        """`a @ b`, `torch.matmul(a, b)`, `torch.nn.functional.linear(x, w[, b])`
        and `self.<sub>(x)` -> the module runtime's GEMM entry points (gemm.py:
        fp32 on cuBLASLt BF16x9; everything else as written)."""
        rt = lambda name: ast.Attribute(ast.Name(GM_RT, ast.Load()), name, ast.Load())  # noqa: E731
        if isinstance(e, ast.BinOp) and isinstance(e.op, ast.MatMult):
            return ast.Call(rt("matmul"), [e.left, e.right], [])
        if not isinstance(e, ast.Call) or e.keywords or any(isinstance(a, ast.Starred) for a in e.args):
            return None
        chain = attr_chain(e.func)
        if chain is None:
            return None
        tn, fn = self.owner.torch_names, self.owner.functional_names
        if len(chain) == 2 and chain[0] in tn and chain[1] == "matmul" and len(e.args) == 2:
            return ast.Call(rt("matmul"), list(e.args), [])
        is_f = (len(chain) == 2 and chain[0] in fn) or (len(chain) == 4 and chain[0] in tn
                                                        and chain[1:3] == ["nn", "functional"])
        is_c = len(chain) == 4 and chain[0] in tn and chain[1:3] == ["_C", "_nn"]   # Dynamo's FX spelling
        if (is_f or is_c) and chain[-1] == "linear" and len(e.args) in (2, 3):
            return ast.Call(rt("linear"), list(e.args), [])
        if chain[0] == "self" and len(chain) >= 2 and len(e.args) == 1:
            return ast.Call(rt("call"), [e.func, e.args[0]], [])
        return None

    def _copy_call(self, e: ast.expr) -> ast.expr | None:
        """`X.reshape(*shape)` / `X.contiguous()` (X a computed value, e.g.
        attention's `matmul(p, v).transpose(1, 2).reshape(b, n, h)`) -> the
        module runtime's reshape / contiguous (gm_copy_strided when a copy is
        needed)."""
        if not (isinstance(e, ast.Call) and isinstance(e.func, ast.Attribute) and not e.keywords
                and not any(isinstance(a, ast.Starred) for a in e.args)):
            return None
        f = e.func
        if attr_chain(f.value) is not None and attr_chain(f.value)[0] in (self.owner.torch_names
                                                                       | self.owner.functional_names):
            return None   # torch.reshape(...) itself: left as written
        rt = lambda name: ast.Attribute(ast.Name(GM_RT, ast.Load()), name, ast.Load())  # noqa: E731
        if f.attr == "reshape" and e.args:
            return ast.Call(rt("reshape"), [f.value] + list(e.args), [])
        if f.attr == "contiguous" and not e.args:
            return ast.Call(rt("contiguous"), [f.value], [])
        return None

    def _route_gemms(self, stmts: list[ast.stmt]) -> list[ast.stmt]:
        outer = self

        class _Route(ast.NodeTransformer):
            def visit_Lambda(self, node):
                return node

            def generic_visit(self, node):
                node = super().generic_visit(node)
                if isinstance(node, ast.expr):
                    r = outer._gemm_call(node)
                    if r is None:
                        r = outer._copy_call(node)
                    if r is not None:
                        return ast.copy_location(r, node)
                return node

        out = []
        for s in stmts:
            if isinstance(s, (ast.Assign, ast.AugAssign, ast.AnnAssign, ast.Return)) and s.value is not None \
                    and _is_replay(s) is None:
                s.value = _Route().visit(s.value)
                ast.fix_missing_locations(s)
            out.append(s)
        return out

    def _select_gemm_arms(self, stmts: list[ast.stmt]) -> list[ast.stmt]:
        """SURVEY §8f rank 3.  A predicated block whose arms each hold one
        GEMM (transform.py:272 admits torch-rooted calls; :404-412 evaluates
        both arms):
            __gm_t_a = __gm_rt__.matmul(A1, B1)     # then arm
            __gm_then_Y_k = __gm_t_a + c1
            __gm_t_b = __gm_rt__.matmul(A2, B2)     # else arm
            __gm_else_Y_k = __gm_t_b + c2
            Y = torch.where(P, __gm_then_Y_k, __gm_else_Y_k)
        becomes ONE contraction of the operands the predicate selects on the
        device (gemm.select_gemm), read by both arms:
            __gm_mm_j = __gm_rt__.select_gemm(P, 'matmul', (A1, B1), (A2, B2))
            __gm_then_Y_k = __gm_mm_j + c1 ; __gm_else_Y_k = __gm_mm_j + c2
        Under the `where` only the selected arm's value survives, and in that
        arm __gm_mm_j is its own GEMM; arms are pure (the purity gate), so
        the dropped GEMM had no effect."""
        tn = self.owner.torch_names
        out = list(stmts)

        def gemm_of(s):
            if not (isinstance(s, ast.Assign) and len(s.targets) == 1 and isinstance(s.targets[0], ast.Name)
                    and isinstance(s.value, ast.Call) and not s.value.keywords):
                return None
            ch = attr_chain(s.value.func)
            if ch in ([GM_RT, "matmul"], [GM_RT, "linear"]):
                return s.targets[0].id, ch[1], s.value.args
            return None

        def def_index(name, before):
            for j in range(before - 1, -1, -1):
                t = out[j]
                if isinstance(t, ast.Assign) and any(isinstance(x, ast.Name) and x.id == name
                                                     for tg in t.targets for x in ast.walk(tg)):
                    return j
            return None

        def stores(j0, j1):
            names = set()
            for t in out[j0:j1 + 1]:
                names |= {n.id for n in ast.walk(t) if isinstance(n, ast.Name) and isinstance(n.ctx, ast.Store)}
            return names

        def reads(name):
            # generated names only (hoisted temps, arm temporaries): all their
            # reads are in this block
            if not name.startswith("__gm_"):
                return [None, None]
            return [n for t in out for n in ast.walk(t) if isinstance(n, ast.Name) and n.id == name
                    and isinstance(n.ctx, ast.Load)]

        i = 0
        while i < len(out):
            s = out[i]
            w = s.value if isinstance(s, ast.Assign) else None
            ch = attr_chain(w.func) if isinstance(w, ast.Call) else None
            if not (ch and len(ch) == 2 and ch[0] in tn and ch[1] == "where" and len(w.args) == 3
                    and not w.keywords and all(isinstance(a, ast.Name) for a in w.args)):
                i += 1
                continue
            P, TT, TE = (a.id for a in w.args)
            found = []
            for arm in (TT, TE):
                ja = def_index(arm, i)
                g = None
                if ja is not None:
                    g = gemm_of(out[ja])
                    if g is None:   # the GEMM is a hoisted temp read once by the arm statement
                        cands = [n.id for n in ast.walk(out[ja].value) if isinstance(n, ast.Name)]
                        for c in cands:
                            jc = def_index(c, ja)
                            if jc is not None and gemm_of(out[jc]) is not None and len(reads(c)) == 1:
                                g, ja = gemm_of(out[jc]), jc
                                break
                    elif len(reads(arm)) != 1:
                        g = None
                found.append((ja, g))
            (j1, g1), (j2, g2) = found
            if g1 is None or g2 is None or j1 == j2 or g1[1] != g2[1] or len(g1[2]) != len(g2[2]):
                i += 1
                continue
            lo, hi = min(j1, j2), max(j1, j2)
            jp = def_index(P, lo + 1)
            operand_names = {n.id for a in list(g1[2]) + list(g2[2]) for n in ast.walk(a) if isinstance(n, ast.Name)}
            if (jp is None and P in stores(0, i)) or (jp is not None and jp >= lo) \
                    or (operand_names | {P}) & stores(lo, hi) - {g1[0], g2[0]}:
                i += 1
                continue
            name = f"__gm_mm_{self.owner.next_tmp()}"
            call = ast.Call(ast.Attribute(ast.Name(GM_RT, ast.Load()), "select_gemm", ast.Load()),
                            [ast.Name(P, ast.Load()), ast.Constant(g1[1]),
                             ast.Tuple(list(g1[2]), ast.Load()), ast.Tuple(list(g2[2]), ast.Load())], [])
            new = ast.copy_location(ast.Assign(targets=[ast.Name(name, ast.Store())], value=call), out[lo])
            new.end_lineno, new.end_col_offset = out[lo].end_lineno, out[lo].end_col_offset
            for old in (g1[0], g2[0]):
                for n in reads(old):
                    n.id = name
                    self.loads.append(((n.lineno, n.col_offset), name))
            out = out[:lo] + [new] + out[lo + 1:hi] + out[hi + 1:]
            ast.fix_missing_locations(new)
            self.owner.gemm_arms.append((P, g1[1]))
            i = lo + 1
        return out

    def lower_block(self, stmts: list[ast.stmt], in_loop: bool) -> list[ast.stmt]:
        out: list[ast.stmt] = []
        run: list[ast.stmt] = []
        hoist: list[ast.stmt] = []
        stmts = self._select_gemm_arms(self._route_gemms(self._split_calls(self._lower_dynamic_shape(stmts))))
        stmts = self._rematerialise(stmts)
        for stmt in self._split_returns(stmts):
            cap = _is_capture(stmt)
            if cap is not None and run:
                assigned = {s.targets[0].id for s in run}
                if not (_names_read(stmt.value) & assigned):
                    hoist.append(stmt)
                    continue
            if self._try_extend(run, stmt):
                run.append(stmt)
                continue
            out.extend(self.flush(run, hoist, in_loop))
            run, hoist = [], []
            if self._try_extend([], stmt):
                run.append(stmt)
                continue
            out.append(self.lower_stmt(stmt, in_loop))
        out.extend(self.flush(run, hoist, in_loop))
        return out

    def _split_returns(self, stmts: list[ast.stmt]) -> list[ast.stmt]:
        """`return <fusable expr>` -> `__gm_retv_k = <expr>; return __gm_retv_k`
        so the returned expression can join the preceding region."""
        out: list[ast.stmt] = []
        for s in stmts:
            if isinstance(s, ast.Return) and s.value is not None and not isinstance(s.value, (ast.Name, ast.Constant)):
                try:
                    Builder(Graph(), self.owner.torch_names, self.owner.functional_names).expr(s.value)
                except Unsupported:
                    out.append(s)
                    continue
                name = f"__gm_retv_{self.owner.next_ret()}"
                a = ast.copy_location(ast.Assign(targets=[ast.Name(name, ast.Store())], value=s.value), s)
                r = ast.copy_location(ast.Return(ast.Name(name, ast.Load())), s)
                r.end_lineno, r.end_col_offset = s.end_lineno, s.end_col_offset
                self.loads.append(((s.end_lineno, s.end_col_offset + 1), name))
                out.extend([a, r])
            else:
                out.append(s)
        return out

    def lower_stmt(self, stmt: ast.stmt, in_loop: bool) -> ast.stmt:
        rep = _is_replay(stmt)
        if rep is not None:
            func, cap = rep
            site = self.owner.new_site(ast.unparse(func), cap, self.fn.name, stmt.lineno)
            call = ast.Call(
                func=ast.Attribute(ast.Name(GM_RT, ast.Load()), "replay", ast.Load()),
                args=[ast.Constant(site), func, ast.Name(cap, ast.Load())],
                keywords=[],
            )
            return ast.copy_location(ast.Expr(call), stmt)
        loop = in_loop or isinstance(stmt, (ast.For, ast.AsyncFor, ast.While))
        for attr in ("body", "orelse", "finalbody"):
            block = getattr(stmt, attr, None)
            if isinstance(block, list) and block and isinstance(block[0], ast.stmt):
                setattr(stmt, attr, self.lower_block(block, loop))
        if isinstance(stmt, ast.Try):
            for h in stmt.handlers:
                h.body = self.lower_block(h.body, loop)
        return stmt

    def flush(self, run: list[ast.stmt], hoist: list[ast.stmt], in_loop: bool) -> list[ast.stmt]:
        if not run:
            return list(hoist)
        graph, b = self._build(run)
        assigned: list[str] = []
        for s in run:
            name = s.targets[0].id
            if name in assigned:
                assigned.remove(name)
            assigned.append(name)
        last = run[-1]
        end = (last.end_lineno, last.end_col_offset)
        live = [n for n in assigned if in_loop or self.read_after(n, end)]
        # a live-out whose final binding is a constant (`a = x.sum(); a = 3`,
        # the reference's taint_kill fixture) is assigned after the region
        consts = [ast.copy_location(ast.Assign(targets=[ast.Name(n, ast.Store())],
                                               value=ast.Constant(b.env[n].value)), last)
                  for n in live if b.env[n].op == "const"]
        live = [n for n in live if b.env[n].op != "const"]
        out_nodes = [b.env[n] for n in live]
        if not live or not any(n.op not in ("free", "const") for n in graph.nodes):
            if consts and not live:
                return list(hoist) + consts
            return list(hoist) + list(run)
        rid = len(self.owner.regions)
        src = "\n".join(ast.unparse(s) for s in run)
        fallback = self.owner.make_fallback(rid, run, graph, live)
        region = Region(rid, f"{self.fn.name}:{run[0].lineno}-{last.end_lineno}", graph, live, out_nodes,
                        fallback, src)
        self.owner.regions.append(region)
        self.owner.region_sources.append(src)
        args = [ast.parse(fv.text, mode="eval").body for fv in graph.frees]
        call = ast.Call(
            func=ast.Subscript(
                ast.Attribute(ast.Name(GM_RT, ast.Load()), "regions", ast.Load()), ast.Constant(rid), ast.Load()
            ),
            args=args,
            keywords=[],
        )
        if len(live) == 1:
            target: ast.expr = ast.Name(live[0], ast.Store())
        else:
            target = ast.Tuple([ast.Name(n, ast.Store()) for n in live], ast.Store())
        stmt = ast.Assign(targets=[target], value=call)
        ast.copy_location(stmt, run[0])
        return list(hoist) + [stmt] + consts


class _Lowerer:
    def __init__(self, text: str):
        self.text = text
        self.tree = ast.parse(text)
        self.torch_names, self.functional_names = _torch_aliases(self.tree)
        self.inlined_layer_norms = _inline_layer_norms(self.tree, self.torch_names)
        self.regions: list[Region] = []
        self.region_sources: list[str] = []
        self.sites: list[ReplaySite] = []
        self.fallback_defs: list[ast.FunctionDef] = []
        self.dyn_lowered: list[tuple[str, str]] = []
        self.gemm_arms: list[tuple[str, str]] = []
        self.rematerialised: list[str] = []

    def next_tmp(self) -> int:
        self._tmp = getattr(self, "_tmp", 0) + 1
        return self._tmp - 1

    def next_ret(self) -> int:
        self._ret = getattr(self, "_ret", -1) + 1
        return self._ret

    def new_site(self, callee_src: str, cap: str, fn: str, lineno: int) -> int:
        sid = len(self.sites)
        self.sites.append(ReplaySite(sid, callee_src, cap, fn, lineno))
        return sid

    def make_fallback(self, rid: int, run: list[ast.stmt], graph: Graph, live: list[str]):
        """The region's original statements as a function of its free values."""
        params = [f"__gm_a{i}" for i in range(len(graph.frees))]
        attr_frees = {fv.text: params[i] for i, fv in enumerate(graph.frees) if "." in fv.text}
        name_frees = [(fv.text, params[i]) for i, fv in enumerate(graph.frees) if "." not in fv.text]

        class _Sub(ast.NodeTransformer):
            def visit_Attribute(self, node):
                chain = attr_chain(node)
                if chain is not None and isinstance(node.ctx, ast.Load):
                    text = ".".join(chain)
                    if text in attr_frees:
                        return ast.copy_location(ast.Name(attr_frees[text], ast.Load()), node)
                return self.generic_visit(node)

        body: list[ast.stmt] = [
            ast.Assign(targets=[ast.Name(n, ast.Store())], value=ast.Name(p, ast.Load())) for n, p in name_frees
        ]
        body += [_Sub().visit(copy.deepcopy(s)) for s in run]
        ret = ast.Name(live[0], ast.Load()) if len(live) == 1 else ast.Tuple(
            [ast.Name(n, ast.Load()) for n in live], ast.Load())
        body.append(ast.Return(ret))
        fdef = ast.FunctionDef(
            name=f"__gm_fallback_{rid}",
            args=ast.arguments(posonlyargs=[], args=[ast.arg(p) for p in params], vararg=None, kwonlyargs=[],
                               kw_defaults=[], kwarg=None, defaults=[]),
            body=body,
            decorator_list=[],
            returns=None,
            type_params=[],
        )
        self.fallback_defs.append(fdef)
        holder = {"rid": rid}
        self._pending = getattr(self, "_pending", [])
        self._pending.append(holder)

        def call(*args, _holder=holder):
            return _holder["fn"](*args)

        return call

    def _is_compile_decorator(self, d: ast.expr) -> bool:
        target = d.func if isinstance(d, ast.Call) else d
        chain = attr_chain(target)
        return chain is not None and len(chain) == 2 and chain[0] in self.torch_names and chain[1] == "compile"

    def run(self) -> Lowered:
        fns = [n for n in ast.walk(self.tree) if isinstance(n, (ast.FunctionDef, ast.AsyncFunctionDef))]
        for fn in fns:
            if fn.name.startswith("__") and fn.name.endswith("__") and fn.name != "__call__":
                # constructors and other dunders run once on the host (module
                # set-up: buffers, masks), not on the forward's hot path
                continue
            # `@torch.compile` entry points (analysis.py entry mechanisms) are
            # executed by the B200 path itself: drop the Dynamo wrapper
            fn.decorator_list = [d for d in fn.decorator_list if not self._is_compile_decorator(d)]
            fl = _FunctionLowerer(self, fn)
            fn.body = fl.lower_block(fn.body, in_loop=False)
        ast.fix_missing_locations(self.tree)
        source = ast.unparse(self.tree)
        return Lowered(self.text, source, self.regions, self.sites, self.region_sources, list(self.dyn_lowered),
                       list(self.gemm_arms))


def lower(text: str) -> tuple[Lowered, "_Lowerer"]:
    lw = _Lowerer(text)
    return lw.run(), lw


def load(text: str, name: str | None = None, runtime=None, allow_eager: bool = False
         ) -> tuple[types.ModuleType, Lowered]:
    """Lower `text` and execute it as a fresh module whose `__gm_rt` is the
    module runtime (logring.ModuleRuntime).  With `allow_eager`, a region
    whose arguments leave the fused subset (e.g. CPU tensors) runs its
    original statements with PyTorch; by default it raises
    region.RegionUnsupported."""
    from .logring import ModuleRuntime

    lowered, lw = lower(text)
    for r in lowered.regions:
        r.allow_eager = allow_eager
    mod_name = name or f"_gm_b200_prog_{next(_module_ids)}"
    filename = f"<gm-b200:{mod_name}>"
    module = types.ModuleType(mod_name)
    module.__file__ = filename
    rt = runtime or ModuleRuntime(lowered)
    module.__dict__[GM_RT] = rt
    # fallbacks are compiled in the module namespace so globals resolve
    fb_mod = ast.Module(body=lw.fallback_defs, type_ignores=[])
    ast.fix_missing_locations(fb_mod)
    fb_src = ast.unparse(fb_mod)
    full = lowered.source + "\n\n" + fb_src + "\n"
    linecache.cache[filename] = (len(full), None, full.splitlines(True), filename)
    code = compile(full, filename, "exec")
    import sys

    sys.modules[mod_name] = module
    exec(code, module.__dict__)
    for holder in getattr(lw, "_pending", []):
        holder["fn"] = module.__dict__[f"__gm_fallback_{holder['rid']}"]
    lowered.source = full
    return module, lowered

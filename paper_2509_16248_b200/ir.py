"""Expression IR for fused regions of a GraphMend-transformed forward.

The transform emits straight-line Python (transform.py:359-444):
    __gm_pred_k = <cond>                       (transform.py:386-388)
    __gm_then_T_k = <pure expr> ...            (transform.py:404-412)
    T = torch.where(__gm_pred_k, then, else)   (transform.py:374-376, :420-422)
whose arms are restricted by the purity gate to names, constants,
`+ - * / // % ** @`, unary +/-, comparisons, subscripts, torch.* calls and the
allowlisted tensor methods (transform.py:225-289, data/pure_ops.cfg), and
whose predicates are reductions from attr_table.cfg (analysis.py:472-501).

This module parses such statements into a DAG of `Node`s.  Anything outside
the fusable subset (matmul, calls on modules, subscripts, reductions with a
`dim`, ...) raises `Unsupported`, and the lowering leaves that statement to
PyTorch.  Types and shapes are not guessed: `infer()` evaluates the DAG on
`meta` tensors, so promotion and broadcasting are torch's own.
"""

from __future__ import annotations

import ast
import math
from dataclasses import dataclass, field
from typing import Any

import torch


class Unsupported(Exception):
    """The expression leaves the fusable subset."""


# `.item()` (attr_table.cfg: dynamic) lowered to a device scalar with Python
# number semantics — SURVEY §8f rank 2 (corpus/longformer_like/original.py:18-26).
ITEM = "item"

UNARY = {
    "neg", "pos", "abs", "relu", "sigmoid", "tanh", "exp", "log", "sqrt", "rsqrt", "sin", "cos",
    "silu", "square", "reciprocal", "logical_not", "gelu", "gelu_tanh", "erf",
}
BINARY = {"add", "sub", "mul", "div", "pow", "maximum", "minimum", "gt", "ge", "lt", "le", "eq", "ne",
          "logical_and", "logical_or", "floordiv", "mod", "fmod"}
COMPARE = {"gt", "ge", "lt", "le", "eq", "ne"}
REDUCE = {"sum", "mean", "amax", "amin", "norm", "prod", "any", "all", "count_nonzero", "nzsum", "argmax", "argmin"}
# Row operators over the innermost dimension (pure_ops.cfg: softmax; the
# attr_table reductions sum/mean/max/min called with `dim`, transform.py:
# 265-289 admits any torch.* call in an arm).  They run in the row-region
# kernel (rowgen.py), one row per thread group, the row held on chip.
# Node.value = (dim, keepdim) as written; infer() checks dim is the last one.
ROW_RED = {"row_sum": "sum", "row_mean": "mean", "row_amax": "amax", "row_amin": "amin", "row_var": "var",
           "row_std": "std"}
ROW_NORM = {"softmax", "log_softmax", "layer_norm"}
ROW_OPS = set(ROW_RED) | ROW_NORM
# reductions whose result is an integer count/sum: accumulated exactly in fp64
INT_REDUCE = {"count_nonzero", "nzsum"}
# `torch.nonzero(m).sum()` lowered to a reduction: the sum over the positions
# where m holds of their coordinates (SURVEY §8f rank 1,
# corpus/moe_minicpm_like/original.py:14-15)
NZSUM = "nzsum"
GM_RT_NAME = "__gm_rt__"
BOOL_AND, BOOL_OR, BOOL_NOT = "bool_and", "bool_or", "bool_not"
# `v is None` / `v is not None`: the reference copies such predicates verbatim
# (transform.py:386-388; parameters are taint seeds, analysis.py:340-344), so
# the rewrite hands torch.where a Python bool.  They are resolved on the host
# when a region is specialised (fold_host_predicates): the original `if`.
IS_NONE, IS_NOT_NONE = "is_none", "is_not_none"

# torch.<name>(...) / torch.nn.functional.<name>(...) spellings
_TORCH_FUNCS = {
    "relu": "relu", "sigmoid": "sigmoid", "tanh": "tanh", "exp": "exp", "log": "log", "sqrt": "sqrt",
    "rsqrt": "rsqrt", "abs": "abs", "sin": "sin", "cos": "cos", "neg": "neg", "negative": "neg",
    "square": "square", "reciprocal": "reciprocal", "silu": "silu", "logical_not": "logical_not",
    "add": "add", "sub": "sub", "subtract": "sub", "mul": "mul", "multiply": "mul", "div": "div",
    "true_divide": "div", "divide": "div", "pow": "pow", "maximum": "maximum", "minimum": "minimum",
    "gt": "gt", "greater": "gt", "ge": "ge", "lt": "lt", "less": "lt", "le": "le", "eq": "eq", "ne": "ne",
    "logical_and": "logical_and", "logical_or": "logical_or", "where": "where", "clamp": "clamp",
    "clip": "clamp", "sum": "sum", "mean": "mean", "amax": "amax", "amin": "amin", "prod": "prod",
    "any": "any", "all": "all", "count_nonzero": "count_nonzero", "norm": "norm",
    "argmax": "argmax", "argmin": "argmin", "max": "max", "min": "min",
    "softmax": "softmax", "log_softmax": "log_softmax", "gelu": "gelu", "erf": "erf", "var": "var", "std": "std",
    "floor_divide": "floordiv", "remainder": "mod", "fmod": "fmod",
}
# Tensor.<name>(...) spellings (pure_ops.cfg plus the attr_table reductions)
_METHODS = dict(_TORCH_FUNCS)
_METHODS.update({"clamp_min": "clamp_min", "clamp_max": "clamp_max", "item": ITEM})

_BINOP = {ast.Add: "add", ast.Sub: "sub", ast.Mult: "mul", ast.Div: "div", ast.Pow: "pow",
          ast.FloorDiv: "floordiv", ast.Mod: "mod"}
_CMPOP = {ast.Gt: "gt", ast.GtE: "ge", ast.Lt: "lt", ast.LtE: "le", ast.Eq: "eq", ast.NotEq: "ne"}


@dataclass(eq=False)
class Node:
    op: str                      # "free", "const", or an op name above
    args: tuple = ()
    value: Any = None            # free: arg index; const: Python value; clamp: (has_lo, has_hi)
    # filled by infer()
    kind: str = ""               # "host" | "dscalar" | "elem"
    dtype: Any = None            # torch dtype (host: python type)
    shape: tuple = ()
    meta: Any = None
    uid: int = -1

    def __repr__(self) -> str:  # pragma: no cover - debugging aid
        return f"Node#{self.uid}({self.op}, {self.kind}, {self.dtype}, {self.shape})"


@dataclass
class FreeVar:
    """A value the region reads from the enclosing scope: a Name or an
    attribute chain rooted at a name not assigned in the region."""
    text: str
    node: Node


@dataclass
class Graph:
    frees: list[FreeVar] = field(default_factory=list)
    nodes: list[Node] = field(default_factory=list)

    def add(self, node: Node) -> Node:
        node.uid = len(self.nodes)
        self.nodes.append(node)
        return node


def attr_chain(expr: ast.expr) -> list[str] | None:
    parts: list[str] = []
    cur = expr
    while isinstance(cur, ast.Attribute):
        parts.append(cur.attr)
        cur = cur.value
    if isinstance(cur, ast.Name):
        parts.append(cur.id)
        return parts[::-1]
    return None


class Builder:
    """AST -> Node for one region.  `env` maps region-assigned names to the
    node of their current binding (SSA by construction)."""

    def __init__(self, graph: Graph, torch_names: set[str], functional_names: set[str]):
        self.g = graph
        self.env: dict[str, Node] = {}
        self.torch_names = torch_names          # aliases of the torch module
        self.functional_names = functional_names  # aliases of torch.nn.functional
        self._free_by_text: dict[str, Node] = {}
        self._consts: dict[tuple, Node] = {}

    # -- leaves -------------------------------------------------------------
    def free(self, text: str) -> Node:
        if text not in self._free_by_text:
            node = self.g.add(Node("free", value=len(self.g.frees)))
            self.g.frees.append(FreeVar(text, node))
            self._free_by_text[text] = node
        return self._free_by_text[text]

    def const(self, value) -> Node:
        key = (type(value), value)
        if key not in self._consts:
            self._consts[key] = self.g.add(Node("const", value=value))
        return self._consts[key]

    def op(self, name: str, *args: Node, value=None) -> Node:
        return self.g.add(Node(name, tuple(args), value=value))

    # -- row operators ------------------------------------------------------------
    def _const_int(self, e) -> int:
        """A literal int (possibly negated) from an AST argument or a const node."""
        if isinstance(e, Node):
            if e.op == "const" and isinstance(e.value, int) and not isinstance(e.value, bool):
                return e.value
            if e.op == "neg" and len(e.args) == 1:
                return -self._const_int(e.args[0])
            raise Unsupported("non-constant dim")
        if isinstance(e, ast.Constant) and isinstance(e.value, int) and not isinstance(e.value, bool):
            return e.value
        if isinstance(e, ast.UnaryOp) and isinstance(e.op, ast.USub):
            return -self._const_int(e.operand)
        if isinstance(e, (ast.Tuple, ast.List)) and len(e.elts) == 1:
            return self._const_int(e.elts[0])
        raise Unsupported("non-constant dim")

    def _dim_arg(self, pos: list, kw: dict, names: tuple) -> int:
        if pos:
            return self._const_int(pos[0])
        for k in names:
            if k in kw:
                return self._const_int(kw[k])
        raise Unsupported("missing dim")

    def layer_norm(self, c: ast.Call) -> Node:
        """F.layer_norm(x, (C,), weight=None, bias=None, eps=1e-5) over the
        innermost dim (a one-element normalized_shape): a row operator.
        Missing weight / bias are the constants 1 / 0 (exact: x * 1 and
        x + 0 change no bits but -0 + 0)."""
        pos = list(c.args)
        kw = {k.arg: k.value for k in c.keywords}
        if None in kw or any(isinstance(a, ast.Starred) for a in pos):
            raise Unsupported("layer_norm arguments")
        names = ["input", "normalized_shape", "weight", "bias", "eps"]
        vals = dict(zip(names, pos))
        for k, v in kw.items():
            if k not in names or k in vals:
                raise Unsupported(f"layer_norm keyword {k}")
            vals[k] = v
        if "input" not in vals or "normalized_shape" not in vals:
            raise Unsupported("layer_norm arguments")
        ns = vals["normalized_shape"]
        # `self.<ln>.normalized_shape`: written by lowering._inline_layer_norms
        # for an nn.LayerNorm built with a one-dimensional shape
        inlined = isinstance(ns, ast.Attribute) and ns.attr == "normalized_shape"
        if inlined:
            # a free value the kernel never reads (the region's eager
            # statements, lowering.make_fallback, do read it)
            self.free(ast.unparse(ns))
        if not inlined and not (isinstance(ns, (ast.Tuple, ast.List)) and len(ns.elts) == 1):
            raise Unsupported("layer_norm over more than the innermost dim")
        eps = 1e-5
        if "eps" in vals:
            e = vals["eps"]
            if not (isinstance(e, ast.Constant) and isinstance(e.value, (int, float))):
                raise Unsupported("non-constant eps")
            eps = float(e.value)
        x = self.expr(vals["input"])

        def opt(key, default):
            v = vals.get(key)
            if v is None or (isinstance(v, ast.Constant) and v.value is None):
                return self.const(default)
            return self.expr(v)

        return self.op("layer_norm", x, opt("weight", 1.0), opt("bias", 0.0), value=(-1, True, eps))

    def _row_reduce(self, name: str, args: list, kw: dict) -> Node:
        """x.sum(-1, keepdim=True) / x.mean(dim=-1) / x.amax(-1) / torch.sum(x, -1)."""
        extra = set(kw) - {"dim", "keepdim"}
        if extra or len(args) > 3:
            raise Unsupported(f"{name} arguments {sorted(extra)}")
        dim = self._dim_arg(args[1:2], kw, ("dim",))
        keep = False
        if len(args) == 3:
            kn = args[2]
            if kn.op != "const" or not isinstance(kn.value, bool):
                raise Unsupported("non-constant keepdim")
            keep = kn.value
        elif "keepdim" in kw:
            v = kw["keepdim"]
            if not (isinstance(v, ast.Constant) and isinstance(v.value, bool)):
                raise Unsupported("non-constant keepdim")
            keep = v.value
        return self.op("row_" + name, args[0], value=(dim, keep))

    # -- expressions ------------------------------------------------------------
    def expr(self, e: ast.expr) -> Node:
        if isinstance(e, ast.Name):
            if e.id in self.env:
                return self.env[e.id]
            if e.id in self.torch_names or e.id in self.functional_names:
                raise Unsupported("module used as a value")
            return self.free(e.id)
        if isinstance(e, ast.Constant):
            if isinstance(e.value, bool) or isinstance(e.value, (int, float)):
                return self.const(e.value)
            raise Unsupported(f"constant {e.value!r}")
        if isinstance(e, ast.Attribute):
            chain = attr_chain(e)
            if chain is None or chain[0] in self.env or chain[0] in self.torch_names:
                raise Unsupported("attribute of a region value")
            return self.free(".".join(chain))
        if isinstance(e, ast.BinOp):
            name = _BINOP.get(type(e.op))
            if name is None:
                raise Unsupported(f"operator {type(e.op).__name__}")
            return self.op(name, self.expr(e.left), self.expr(e.right))
        if isinstance(e, ast.UnaryOp):
            if isinstance(e.op, ast.USub):
                return self.op("neg", self.expr(e.operand))
            if isinstance(e.op, ast.UAdd):
                return self.op("pos", self.expr(e.operand))
            if isinstance(e.op, ast.Not):
                return self.op(BOOL_NOT, self.expr(e.operand))
            raise Unsupported(f"unary {type(e.op).__name__}")
        if isinstance(e, ast.BoolOp):
            # `p and q` / `p or q` / `not p` on 0-d bool
            # tensors (the reference copies predicates verbatim,
            # transform.py:386-388, so these reach the runtime and sync via
            # Tensor.__bool__ or, for `not`, hand torch.where a Python bool)
            name = BOOL_AND if isinstance(e.op, ast.And) else BOOL_OR
            node = self.expr(e.values[0])
            for v in e.values[1:]:
                node = self.op(name, node, self.expr(v))
            return node
        if isinstance(e, ast.Compare):
            if len(e.ops) != 1:
                raise Unsupported("chained comparison")
            if isinstance(e.ops[0], (ast.Is, ast.IsNot)):
                left, right = e.left, e.comparators[0]
                if isinstance(right, ast.Constant) and right.value is None:
                    operand = left
                elif isinstance(left, ast.Constant) and left.value is None:
                    operand = right
                else:
                    raise Unsupported("identity comparison with a value other than None")
                return self.op(IS_NONE if isinstance(e.ops[0], ast.Is) else IS_NOT_NONE, self.expr(operand))
            name = _CMPOP.get(type(e.ops[0]))
            if name is None:
                raise Unsupported(f"comparison {type(e.ops[0]).__name__}")
            return self.op(name, self.expr(e.left), self.expr(e.comparators[0]))
        if isinstance(e, ast.Call):
            return self.call(e)
        if isinstance(e, ast.Subscript):
            return self.subscript(e)
        raise Unsupported(type(e).__name__)

    def subscript(self, e: ast.Subscript) -> Node:
        """Basic indexing of a value read from the enclosing scope
        (`x[..., :k]`, `x[:, 0]`, `x[None]`; transform.py:245-254 admits
        subscripts in arms) is a view: the region reads it as a free value —
        the subscript is evaluated by the caller when the region is called
        (no copy, no kernel) and the kernel reads the view's strides.
        Subscripts of region values, tensor indices and names assigned in the
        region stay unfused."""
        chain = attr_chain(e.value)
        if chain is None or chain[0] in self.env or chain[0] in self.torch_names \
                or chain[0] in self.functional_names:
            raise Unsupported("subscript of a region value")

        def basic(x: ast.expr) -> bool:
            if isinstance(x, ast.Constant):
                return x.value is None or x.value is Ellipsis or (isinstance(x.value, int)
                                                                  and not isinstance(x.value, bool))
            if isinstance(x, ast.UnaryOp) and isinstance(x.op, ast.USub):
                return basic(x.operand)
            if isinstance(x, ast.Slice):
                return all(v is None or basic(v) for v in (x.lower, x.upper, x.step))
            if isinstance(x, ast.Tuple):
                return all(basic(v) for v in x.elts)
            return False

        if not basic(e.slice):
            raise Unsupported("subscript with a non-constant index")
        return self.free(ast.unparse(e))

    def call(self, c: ast.Call) -> Node:
        func = c.func
        if not isinstance(func, ast.Attribute):
            raise Unsupported("call of a plain name")
        chain = attr_chain(func)
        if chain == [GM_RT_NAME, "nonzero_sum"] and len(c.args) == 1 and not c.keywords:
            return self.op(NZSUM, self.expr(c.args[0]))
        is_torch = chain is not None and (
            (len(chain) == 2 and chain[0] in self.torch_names)
            or (len(chain) == 2 and chain[0] in self.functional_names)
            or (len(chain) == 4 and chain[0] in self.torch_names and chain[1:3] == ["nn", "functional"])
            # Dynamo's FX spelling of the functional ops (`torch._C._nn.gelu`)
            or (len(chain) == 4 and chain[0] in self.torch_names and chain[1:3] == ["_C", "_nn"])
        )
        if is_torch and chain[-1] == "layer_norm":
            return self.layer_norm(c)
        if is_torch:
            name = _TORCH_FUNCS.get(chain[-1])
            if name is None:
                raise Unsupported(f"torch.{chain[-1]}")
            args = [self.expr(a) for a in c.args]
            return self.apply(name, args, c.keywords, method=False)
        # method call on an expression (receiver may be a region value or free)
        name = _METHODS.get(func.attr)
        if name is None:
            raise Unsupported(f"method .{func.attr}")
        recv = self.expr(func.value)
        args = [recv] + [self.expr(a) for a in c.args]
        return self.apply(name, args, c.keywords, method=True)

    def apply(self, name: str, args: list[Node], keywords: list[ast.keyword], method: bool) -> Node:
        kw = {}
        for k in keywords:
            if k.arg is None:
                raise Unsupported("**kwargs")
            kw[k.arg] = k.value
        if any(isinstance(a, ast.Starred) for a in args):
            raise Unsupported("*args")
        if name in ("max", "min"):
            if len(args) == 1 and not kw:
                return self.op("amax" if name == "max" else "amin", args[0])
            if len(args) == 2 and not kw and args[1].op != "const":
                return self.op("maximum" if name == "max" else "minimum", args[0], args[1])
            # max(dim) / min(dim) return (values, indices): not a tensor
            raise Unsupported(f"{name} with dim")
        if name in ("var", "std"):
            corr = 1
            if "unbiased" in kw:
                u = kw.pop("unbiased")
                if not (isinstance(u, ast.Constant) and isinstance(u.value, bool)):
                    raise Unsupported("non-constant unbiased")
                corr = 1 if u.value else 0
            if "correction" in kw:
                cv = kw.pop("correction")
                corr = self._const_int(cv)
            node = self._row_reduce(name, args, kw)
            node.value = node.value + (corr,)
            return node
        if name in ("sum", "mean", "amax", "amin") and (len(args) > 1 or kw):
            return self._row_reduce(name, args, kw)
        if name in ("softmax", "log_softmax"):
            dim = self._dim_arg(args[1:], kw, ("dim",))
            if len(args) > 2:
                raise Unsupported(f"{name} arguments")
            return self.op(name, args[0], value=(dim, True))
        if name in REDUCE:
            if len(args) != 1 or kw:
                raise Unsupported(f"{name} with arguments")
            return self.op(name, args[0])
        if name == ITEM:
            if len(args) != 1 or kw or not method:
                raise Unsupported("item arguments")
            return self.op(ITEM, args[0])
        if name == "gelu" and "approximate" in kw:
            v = kw.pop("approximate")
            if not (isinstance(v, ast.Constant) and v.value in ("none", "tanh")):
                raise Unsupported("gelu approximate")
            if v.value == "tanh":
                name = "gelu_tanh"
        if name in UNARY:
            if len(args) != 1 or kw:
                raise Unsupported(f"{name} arguments")
            return self.op(name, args[0])
        if name in BINARY:
            if len(args) != 2 or kw:
                raise Unsupported(f"{name} arguments")
            return self.op(name, args[0], args[1])
        if name == "where":
            if len(args) != 3 or kw:
                raise Unsupported("where arguments")
            return self.op("where", *args)
        if name in ("clamp", "clamp_min", "clamp_max"):
            x = args[0]
            lo = hi = None
            rest = args[1:]
            if name == "clamp_min":
                lo = rest[0] if rest else None
            elif name == "clamp_max":
                hi = rest[0] if rest else None
            else:
                if len(rest) >= 1:
                    lo = rest[0]
                if len(rest) >= 2:
                    hi = rest[1]
            for k, v in kw.items():
                if k == "min":
                    lo = self.expr(v)
                elif k == "max":
                    hi = self.expr(v)
                else:
                    raise Unsupported(f"clamp keyword {k}")
            if lo is None and hi is None:
                raise Unsupported("clamp without bounds")
            ops = [x] + [n for n in (lo, hi) if n is not None]
            return self.op("clamp", *ops, value=(lo is not None, hi is not None))
        raise Unsupported(name)


# ---------------------------------------------------------------------------
# meta evaluation: torch decides dtypes and shapes
# ---------------------------------------------------------------------------

def _t(x):
    return x


META_FNS = {
    "neg": lambda a: -a,
    "pos": lambda a: +a,
    "abs": lambda a: a.abs() if torch.is_tensor(a) else abs(a),
    "relu": lambda a: torch.relu(a),
    "sigmoid": lambda a: torch.sigmoid(a),
    "tanh": lambda a: torch.tanh(a),
    "exp": lambda a: torch.exp(a),
    "log": lambda a: torch.log(a),
    "sqrt": lambda a: torch.sqrt(a),
    "rsqrt": lambda a: torch.rsqrt(a),
    "sin": lambda a: torch.sin(a),
    "cos": lambda a: torch.cos(a),
    "silu": lambda a: torch.nn.functional.silu(a),
    "gelu": lambda a: torch.nn.functional.gelu(a),
    "gelu_tanh": lambda a: torch.nn.functional.gelu(a, approximate="tanh"),
    "erf": lambda a: torch.erf(a),
    "square": lambda a: torch.square(a),
    "reciprocal": lambda a: torch.reciprocal(a),
    "logical_not": lambda a: torch.logical_not(a),
    "add": lambda a, b: a + b,
    "sub": lambda a, b: a - b,
    "mul": lambda a, b: a * b,
    "div": lambda a, b: a / b,
    "pow": lambda a, b: a ** b,
    "maximum": lambda a, b: torch.maximum(a, b),
    "minimum": lambda a, b: torch.minimum(a, b),
    "gt": lambda a, b: a > b,
    "ge": lambda a, b: a >= b,
    "lt": lambda a, b: a < b,
    "le": lambda a, b: a <= b,
    "eq": lambda a, b: a == b,
    "ne": lambda a, b: a != b,
    "logical_and": lambda a, b: torch.logical_and(a, b),
    "logical_or": lambda a, b: torch.logical_or(a, b),
    "where": lambda c, a, b: torch.where(c, a, b),
    "sum": lambda a: a.sum(),
    "mean": lambda a: a.mean(),
    "amax": lambda a: a.max(),
    "amin": lambda a: a.min(),
    "norm": lambda a: a.norm(),
    "prod": lambda a: a.prod(),
    "any": lambda a: a.any(),
    "all": lambda a: a.all(),
    "count_nonzero": lambda a: torch.count_nonzero(a),
    "argmax": lambda a: a.argmax(),
    "argmin": lambda a: a.argmin(),
    "nzsum": lambda a: torch.zeros((), dtype=torch.int64, device=a.device),
    "floordiv": lambda a, b: a // b,
    "mod": lambda a, b: a % b,
    "fmod": lambda a, b: torch.fmod(a, b),
}


def _meta_row(node: Node, a, rest=()):
    """Row operators: torch's own result; the dim must be the innermost."""
    dim, keep = node.value[:2]
    if not torch.is_tensor(a) or a.dim() == 0:
        raise Unsupported(f"{node.op} of a scalar")
    if dim not in (-1, a.dim() - 1):
        raise Unsupported(f"{node.op} over dim {dim} (only the innermost dim is fused)")
    if node.op == "layer_norm":
        w, b = rest
        for t in (w, b):
            if torch.is_tensor(t) and tuple(t.shape) != (a.shape[-1],):
                raise Unsupported("layer_norm weight / bias not of the row's length")
        w = w if torch.is_tensor(w) else None
        b = b if torch.is_tensor(b) else None
        return torch.nn.functional.layer_norm(a, (a.shape[-1],), w, b, node.value[2])
    if node.op in ROW_NORM:
        return getattr(torch, node.op)(a, -1)
    if node.op in ("row_var", "row_std"):
        return getattr(a, ROW_RED[node.op])(-1, keepdim=keep, correction=node.value[2])
    return getattr(a, ROW_RED[node.op])(-1, keepdim=keep)


def _meta_bool(op: str, vals):
    """Python and/or/not.  On host values: Python semantics.  On 0-d bool
    tensors (predicates): the value Python would return is the logical
    and/or/not, computed on the device instead of through __bool__."""
    if all(not torch.is_tensor(v) for v in vals):
        if op == BOOL_NOT:
            return not vals[0]
        return (vals[0] and vals[1]) if op == BOOL_AND else (vals[0] or vals[1])
    if not all(torch.is_tensor(v) and v.dim() == 0 and v.dtype == torch.bool for v in vals):
        raise Unsupported(f"{op} needs 0-d bool tensors")
    return torch.empty((), dtype=torch.bool, device=vals[0].device)


def _meta_item(a):
    """Python-number stand-in with the type `Tensor.item()` would return."""
    if not torch.is_tensor(a) or a.numel() != 1:
        raise Unsupported("item of a non-scalar")
    if a.dtype == torch.bool:
        return False
    if a.dtype.is_floating_point:
        return 0.0
    return 0


def _meta_clamp(node: Node, vals):
    has_lo, has_hi = node.value
    x = vals[0]
    i = 1
    lo = hi = None
    if has_lo:
        lo = vals[i]
        i += 1
    if has_hi:
        hi = vals[i]
    return torch.clamp(x, min=lo, max=hi)


def _as_meta(v):
    if torch.is_tensor(v):
        return torch.empty_strided(v.shape, v.stride(), dtype=v.dtype, device="meta")
    return v


def infer(graph: Graph, args: list, needed: list[Node]) -> None:
    """Evaluate the nodes `needed` depends on with meta tensors; set kind,
    dtype and shape.  Raises Unsupported on anything torch rejects."""
    order = topo(needed)
    for node in order:
        if node.op == "free":
            v = _as_meta(args[node.value])
            if not (torch.is_tensor(v) or isinstance(v, (bool, int, float))):
                raise Unsupported(f"free value of type {type(v).__name__}")
        elif node.op == "const":
            v = node.value
        else:
            vals = [a.meta for a in node.args]
            try:
                if node.op == "clamp":
                    v = _meta_clamp(node, vals)
                elif node.op == ITEM:
                    v = _meta_item(vals[0])
                elif node.op in (BOOL_AND, BOOL_OR, BOOL_NOT):
                    v = _meta_bool(node.op, vals)
                elif node.op in ROW_OPS:
                    v = _meta_row(node, vals[0], vals[1:])
                else:
                    if all(not torch.is_tensor(x) for x in vals) and node.op not in (
                        "add", "sub", "mul", "div", "pow", "neg", "pos", "abs", "gt", "ge", "lt", "le", "eq", "ne",
                        "floordiv", "mod",
                    ):
                        # torch functions on Python numbers: compute on a 0-d tensor
                        raise Unsupported(f"{node.op} of host scalars")
                    v = META_FNS[node.op](*vals)
            except Unsupported:
                raise
            except Exception as exc:  # torch rejected the combination
                raise Unsupported(f"{node.op}: {exc}") from exc
        node.meta = v
        if torch.is_tensor(v):
            node.kind = "dscalar" if v.dim() == 0 else "elem"
            node.dtype = v.dtype
            node.shape = tuple(v.shape)
        elif isinstance(v, (bool, int, float)):
            node.kind = "host"
            node.dtype = type(v)
            node.shape = ()
        else:
            raise Unsupported(f"value of type {type(v).__name__}")


def evaluate(roots: list[Node], args: list) -> dict[int, Any]:
    """Evaluate the DAG eagerly with PyTorch on the arguments' device — the
    same operators, in the same order and dtypes, that the transformed
    statements run in eager mode.  Test infrastructure: the parity tests
    evaluate a region's statistics and branch decisions on CPU (the oracle's
    arithmetic) to compare with the fused kernel's scalar slots.  Returns
    {node.uid: value}."""
    vals: dict[int, Any] = {}
    for node in topo(roots):
        if node.op == "free":
            v = args[node.value]
        elif node.op == "const":
            v = node.value
        else:
            a = [vals[x.uid] for x in node.args]
            if node.op == "clamp":
                v = _meta_clamp(node, a)
            elif node.op == ITEM:
                v = a[0].item()
            elif node.op == BOOL_NOT:
                v = torch.logical_not(a[0]) if torch.is_tensor(a[0]) else (not a[0])
            elif node.op in (BOOL_AND, BOOL_OR):
                if torch.is_tensor(a[0]) or torch.is_tensor(a[1]):
                    f = torch.logical_and if node.op == BOOL_AND else torch.logical_or
                    v = f(torch.as_tensor(a[0]), torch.as_tensor(a[1]))
                else:
                    v = (a[0] and a[1]) if node.op == BOOL_AND else (a[0] or a[1])
            elif node.op in (IS_NONE, IS_NOT_NONE):
                v = (a[0] is None) == (node.op == IS_NONE)
            elif node.op == NZSUM:
                v = torch.nonzero(a[0]).sum()
            elif node.op in ROW_OPS:
                v = _meta_row(node, a[0], a[1:])
            else:
                v = META_FNS[node.op](*a)
        vals[node.uid] = v
    return vals


def fold_host_predicates(graph: Graph, outputs: list[Node], args: list) -> tuple[Graph, list[Node]]:
    """Resolve `is None` / `is not None` of the region's free values for these
    arguments (the specialisation key includes each argument's type) and
    keep only the selected arm of a `where` whose condition becomes a host
    bool — the original `if` semantics (the reference's rewrite would hand
    torch.where a Python bool and evaluate an arm on None).  and/or/not with
    a resolved operand fold as Python does.  Graphs without identity tests
    are returned unchanged."""
    if not any(n.op in (IS_NONE, IS_NOT_NONE) for n in graph.nodes):
        return graph, outputs
    g = Graph()
    consts: dict = {}
    memo: dict[int, Node] = {}
    for fv in graph.frees:
        nn = g.add(Node("free", value=fv.node.value))
        g.frees.append(FreeVar(fv.text, nn))
        memo[id(fv.node)] = nn

    def const(v) -> Node:
        key = (type(v), v)
        if key not in consts:
            consts[key] = g.add(Node("const", value=v))
        return consts[key]

    def is_const_bool(n: Node) -> bool:
        return n.op == "const" and isinstance(n.value, bool)

    def fold(n: Node) -> Node:
        if id(n) in memo:
            return memo[id(n)]
        if n.op == "const":
            r = const(n.value)
        elif n.op in (IS_NONE, IS_NOT_NONE):
            a = n.args[0]
            if a.op != "free":
                raise Unsupported("identity test of a computed value")
            none = args[a.value] is None
            r = const(none if n.op == IS_NONE else not none)
        elif n.op == "where" and is_const_bool(fold(n.args[0])):
            r = fold(n.args[1] if fold(n.args[0]).value else n.args[2])
        elif n.op == BOOL_NOT and is_const_bool(fold(n.args[0])):
            r = const(not fold(n.args[0]).value)
        elif n.op in (BOOL_AND, BOOL_OR) and is_const_bool(fold(n.args[0])):
            v = fold(n.args[0]).value
            short = (not v) if n.op == BOOL_AND else v
            r = const(v) if short else fold(n.args[1])
        else:
            r = g.add(Node(n.op, tuple(fold(a) for a in n.args), value=n.value))
        memo[id(n)] = r
        return r

    outs = [fold(o) for o in outputs]
    return g, outs


def topo(roots: list[Node]) -> list[Node]:
    seen: set[int] = set()
    order: list[Node] = []
    stack = [(r, False) for r in reversed(roots)]
    while stack:
        node, done = stack.pop()
        if done:
            order.append(node)
            continue
        if id(node) in seen:
            continue
        seen.add(id(node))
        stack.append((node, True))
        for a in reversed(node.args):
            if id(a) not in seen:
                stack.append((a, False))
    return order


def is_fusable_dtype(dt) -> bool:
    return dt in (torch.float32, torch.bfloat16, torch.float16, torch.bool)


def host_value_repr(v) -> str:
    if isinstance(v, bool):
        return "1.0" if v else "0.0"
    f = float(v)
    if math.isnan(f):
        return "(0.0/0.0)"
    if math.isinf(f):
        return "(1.0/0.0)" if f > 0 else "(-1.0/0.0)"
    return repr(f)

"""Randomised differential test of the B200 path: seeded random programs in
the transform's output form (predicated blocks `__gm_pred_k = <expr>.<red>()
⋈ c`, arm temporaries, `torch.where` selects; elementwise statements around
them; row operators; broadcast inputs; `//`, `%`) are lowered, run through
the fused kernels on the GPU and compared with CPU eager execution of the
same text (the oracle), in fp32 and bf16.

Thresholds are placed where the decision is unambiguous (the statistic of a
bounded expression against a constant outside its range, or a sum of a
strictly positive expression against 0), so a decision never hinges on the
last bit; both outcomes occur across the programs.
"""

import random

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import compile_program, harness
from parity import assert_parity, rowop_fp64_reference

UNARY = ["torch.sigmoid({})", "torch.tanh({})", "torch.relu({})", "({}).abs()", "-({})",
         "torch.sqrt(({}).abs() + 1.0)", "torch.exp(torch.tanh({}))", "torch.clamp({}, -2.0, 2.0)"]
BINARY = ["({} + {})", "({} - {})", "({} * {})", "({} / (({}).abs() + 1.0))", "torch.maximum({}, {})",
          "torch.minimum({}, {})", "torch.where({} > 0, {}, {})"]
BOUNDED = ["torch.sigmoid({})", "torch.tanh({})"]          # range (0,1) / (-1,1)
POSITIVE = ["torch.sigmoid({})", "(({}).abs() + 0.5)", "torch.exp(torch.tanh({}))"]
REDS = ["sum", "mean", "amax", "amin", "norm"]


def _expr(rng, names, depth):
    if depth == 0 or rng.random() < 0.3:
        v = rng.choice(names)
        return v if rng.random() < 0.8 else f"({v} * {rng.choice([0.5, 2.0, -1.5, 0.125])})"
    if rng.random() < 0.4:
        return rng.choice(UNARY).format(_expr(rng, names, depth - 1))
    op = rng.choice(BINARY)
    args = [_expr(rng, names, depth - 1) for _ in range(op.count("{}"))]
    if "where" in op:
        args = [args[0], args[1], args[2]]
    elif "abs()" in op:
        args = [args[0], args[1]]
    return op.format(*args)


def _predicate(rng, names):
    """One more predicate form (prod / argmax / any / all / count_nonzero
    reductions of attr_table.cfg, logical and / or / not of 0-d predicates)
    with an unambiguous outcome.  (Python `and` / `not` / `.item()` in a
    predicate make the reference's own rewrite raise in eager torch —
    tests/test_gpu_hardening.py covers those.)"""
    e = _expr(rng, names, 1)
    form = rng.randrange(6)
    if form == 0:
        return f"torch.sigmoid({e}).prod() > 2.0"                 # product of (0,1) values: always False
    if form == 1:
        return f"torch.logical_and(torch.sigmoid({e}).argmax() >= 0, ({e}).abs().sum() >= 0)"
    if form == 2:
        return f"torch.logical_not(torch.tanh({e}).amax() > 1.5)"
    if form == 3:
        return f"torch.sigmoid({e}).amin() > {rng.choice([1.5, -0.5])}"
    if form == 4:
        return f"torch.logical_or((torch.sigmoid({e}) > 2.0).any(), (({e}).abs() >= 0).all())"
    return f"torch.count_nonzero(torch.relu({e}) + 1.0) > 0"


def _program(seed: int, rows: bool) -> str:
    rng = random.Random(seed)
    names = ["x", "y"]
    lines = ["import torch", "", "def f(x, y, b):"]
    k = 0
    for s in range(rng.randint(2, 4)):
        kind = rng.random()
        if kind < 0.15:
            t = f"v{s}"
            lines.append(f"    __gm_pred_{k} = {_predicate(rng, names)}")
            lines.append(f"    __gm_then_{t}_{k} = {_expr(rng, names, 2)}")
            lines.append(f"    __gm_else_{t}_{k} = {_expr(rng, names, 2)}")
            lines.append(f"    {t} = torch.where(__gm_pred_{k}, __gm_then_{t}_{k}, __gm_else_{t}_{k})")
            k += 1
            names.append(t)
            continue
        if kind < 0.5:
            # a predicated block in the transform's emitted form
            red = rng.choice(REDS)
            if rng.random() < 0.5:
                stat = rng.choice(BOUNDED).format(_expr(rng, names, 2))
                thr, cmp = rng.choice([(1.5, ">"), (-1.5, ">"), (1.5, "<"), (-1.5, "<")]), None
                thr, cmp = thr
                if red in ("sum", "norm"):
                    thr = thr * 1e9           # outside the range of any sum of bounded values
            else:
                stat = rng.choice(POSITIVE).format(_expr(rng, names, 2))
                red = rng.choice(["sum", "mean", "amin"])
                thr, cmp = 0.0, rng.choice([">", "<"])
            t = f"v{s}"
            lines.append(f"    __gm_pred_{k} = ({stat}).{red}() {cmp} {thr!r}")
            lines.append(f"    __gm_then_{t}_{k} = {_expr(rng, names, 2)}")
            lines.append(f"    __gm_else_{t}_{k} = {_expr(rng, names, 2)}")
            lines.append(f"    {t} = torch.where(__gm_pred_{k}, __gm_then_{t}_{k}, __gm_else_{t}_{k})")
            k += 1
        elif rows and kind < 0.75:
            t = f"v{s}"
            e = _expr(rng, names, 1)
            form = rng.choice([f"torch.softmax({e} + b, dim=-1)", f"torch.log_softmax({e}, -1)",
                               f"({e}) - ({e}).amax(-1, keepdim=True)",
                               f"({e}) / (({e}).abs().sum(-1, keepdim=True) + 1.0)",
                               f"({e}) - ({e}).mean(-1, keepdim=True)",
                               f"torch.nn.functional.layer_norm({e}, (b.shape[-1],), b, None, 1e-5)",
                               f"torch.nn.functional.gelu({e}) * ({e}).std(-1, keepdim=True)",
                               f"({e}) / torch.sqrt(({e}).var(-1, keepdim=True, unbiased=False) + 1.0)"])
            lines.append(f"    {t} = {form}")
        else:
            t = f"v{s}"
            e = _expr(rng, names, 2)
            if rng.random() < 0.3:
                e = f"({e}) + (x // 0.75) * 0.01 + (y % 1.5)"
            lines.append(f"    {t} = {e}")
        names.append(t)
    lines.append(f"    return {names[-1]} * 1.0 + {names[-2]}")
    return "\n".join(lines) + "\n"


SHAPES32 = [(4, 37, 24), (8, 1024, 768), (33, 100), (6, 2, 3, 10)]
SHAPES16 = [(5, 13, 40), (4, 2048, 64), (7, 24)]
CASES = [(seed, dtype, shape) for seed in range(64)
         for dtype, shape in ((torch.float32, SHAPES32[seed % len(SHAPES32)]),
                              (torch.bfloat16, SHAPES16[seed % len(SHAPES16)]))]


def _fp64_reference(text, args):
    """The program evaluated in fp64 and rounded to its dtype: the noise
    yardstick for row reductions (their accumulation order is unspecified)."""
    ref64, _ = orc.call_captured(orc.reference_callable(text, "f"), [a.double() for a in args])
    return ref64.to(args[0].dtype)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,dtype,shape", CASES, ids=[f"s{c[0]}-{str(c[1])[6:]}-{'x'.join(map(str, c[2]))}"
                                                         for c in CASES])
def test_random_program(seed, dtype, shape):
    text = _program(seed, rows=True)
    torch.manual_seed(seed)
    x = torch.randn(shape).to(dtype)
    y = torch.randn(shape[-1]).to(dtype) if seed % 2 else torch.randn(shape).to(dtype)
    b = torch.randn(shape[-1]).to(dtype)
    args = [x, y, b]
    ref, _ = orc.call_captured(orc.reference_callable(text, "f"), list(args))
    noise = rowop_fp64_reference(text, "f", list(args)) if "softmax(" in text else None
    if noise is None and any(k in text for k in ("layer_norm(", ".std(", ".var(", ".sum(-1", ".mean(-1")):
        noise = _fp64_reference(text, args)
    ex, mod, low = compile_program(text, "f")
    dev_args = [a.cuda() for a in args]
    out, _ = harness.call_captured(ex, dev_args)
    torch.cuda.synchronize()
    info = ex.info()[0]
    assert info.mode == "graph" and info.host_syncs == 0, (text, info)
    for r in low.regions:
        assert r.stats.fallbacks == 0, (text, r.name, r.stats.fallback_reasons)
    assert_parity(out, ref, dtype, what=f"seed {seed}\n{text}", noise=noise)
    # replays build the speculative regions' confidence: later launches take
    # the speculative path (sampled or history prediction) — same bits
    first = out.clone()
    for _ in range(4):
        again, _ = harness.call_captured(ex, dev_args)
        iv = torch.int32 if first.element_size() == 4 else torch.int16
        assert torch.equal(again.view(iv), first.view(iv)), f"seed {seed}: replay differs\n{text}"

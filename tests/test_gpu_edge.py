"""Edge cases of the fused-region path against torch eager on CPU (the
reference's executor): broadcast modes (periodic bias, strided, scalar and
numel-1 tensors), fp16, bool outputs, NaN propagation, non-contiguous views,
ragged / tiny / empty sizes, scalar live-outs and integer reductions."""

import math

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import compile_program
from parity import assert_parity

BLOCK = '''import torch

def f(x, b):
    __gm_pred_0 = x.sum() > 0
    __gm_then_y_0 = x + b
    __gm_else_y_0 = x - b * 2
    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
    return torch.relu(y)
'''


def _run(text, fn, args, dtype=torch.float32, expect_fused=True):
    ref = orc.reference_callable(text, fn)(*[a.clone() if torch.is_tensor(a) else a for a in args])
    ex, mod, low = compile_program(text, fn)
    out = ex(*[a.cuda() if torch.is_tensor(a) else a for a in args])
    torch.cuda.synchronize()
    if expect_fused:
        assert any(r.stats.launches for r in low.regions), [r.stats.fallback_reasons for r in low.regions]
        assert all(r.last_spec is None or r.last_spec.status() == 0 for r in low.regions)
    return out, ref, ex, low


@pytest.mark.gpu
@pytest.mark.parametrize("bshape", [(768,), (8, 1, 768), (), (1, 1, 1), (8, 1024, 768)],
                         ids=["periodic", "strided", "0d", "numel1", "full"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16], ids=["fp32", "bf16", "fp16"])
def test_broadcast_modes(bshape, dtype):
    torch.manual_seed(1)
    for sign in (1.0, -1.0):
        x = (torch.randn(8, 1024, 768) + 0.05 * sign).to(dtype)
        b = torch.randn(bshape).to(dtype)
        out, ref, ex, low = _run(BLOCK, "f", [x, b], dtype)
        assert_parity(out, ref, dtype, what=f"{bshape}")


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 8, 9, 1001, 4095, 65537])
def test_ragged_sizes(n):
    torch.manual_seed(n)
    x = torch.randn(n)
    out, ref, *_ = _run(BLOCK, "f", [x, torch.randn(n)])
    assert_parity(out, ref, torch.float32)


@pytest.mark.gpu
def test_non_contiguous_input():
    x = torch.randn(768, 1024).t()  # [1024, 768] view, strided
    b = torch.randn(1024, 768)
    out, ref, *_ = _run(BLOCK, "f", [x, b])
    assert_parity(out, ref, torch.float32)


@pytest.mark.gpu
def test_nan_propagation_in_predicate_and_arms():
    text = ('import torch\n\ndef g(x):\n    __gm_pred_0 = x.max() > 0\n    __gm_then_y_0 = torch.relu(x) + 1\n'
            '    __gm_else_y_0 = x * 0.0\n    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)\n'
            '    return y\n')
    x = torch.randn(4096)
    x[17] = float("nan")
    out, ref, *_ = _run(text, "g", [x])
    # max() is NaN, NaN > 0 is False: the else arm, where NaN * 0 stays NaN
    assert torch.equal(torch.isnan(out.cpu()), torch.isnan(ref))
    assert_parity(out, ref, torch.float32)


@pytest.mark.gpu
def test_bool_and_scalar_live_outs_and_integer_reductions():
    text = ('import torch\n\ndef h(x):\n    m = x > 0.5\n    cnt = (x > 0).sum()\n    nz = torch.count_nonzero(x > 1.0)\n'
            '    s = x.mean() + x.norm()\n    return m, cnt, nz, s\n')
    x = torch.randn(8, 1024, 768)
    ref = orc.reference_callable(text, "h")(x.clone())
    ex, mod, low = compile_program(text, "h")
    out = ex(x.cuda())
    assert torch.equal(out[0].cpu(), ref[0])
    assert out[1].dtype == ref[1].dtype == torch.int64 and int(out[1]) == int(ref[1])
    assert int(out[2]) == int(ref[2])
    # fp32 mean/norm: the B200 statistic is accumulated in fp64 and rounded
    # once; torch's CPU fp32 reductions over 6.3 M elements drift.  The bound
    # is the north_star 1e-5 relative plus that drift, MEASURED here against
    # the same expression evaluated in fp64 on CPU
    ref64 = float(x.double().mean() + x.double().norm())
    drift = abs(float(ref[3]) - ref64)
    assert abs(float(out[3]) - float(ref[3])) <= 1e-5 * abs(float(ref[3])) + drift, (float(out[3]), float(ref[3]), drift)
    assert abs(float(out[3]) - ref64) <= 2e-7 * abs(ref64) + 1e-6, (float(out[3]), ref64)


@pytest.mark.gpu
def test_empty_tensor():
    text = 'import torch\n\ndef e(x):\n    y = x * 2 + 1\n    s = x.sum()\n    return y, s\n'
    x = torch.empty(0, 768)
    ref = orc.reference_callable(text, "e")(x)
    ex, mod, low = compile_program(text, "e")
    out = ex(x.cuda())
    assert out[0].shape == ref[0].shape and float(out[1]) == float(ref[1]) == 0.0


@pytest.mark.gpu
def test_region_decisions_are_deterministic():
    """Fixed-order fp64 combine: repeated launches give identical statistics."""
    text = ('import torch\n\ndef d(x):\n    __gm_pred_0 = x.sum() > 0\n    y = torch.where(__gm_pred_0, x + 1, x - 1)\n'
            '    return y\n')
    x = torch.randn(8, 1024, 768).cuda()
    ex, mod, low = compile_program(text, "d")
    stats = set()
    for _ in range(5):
        low.regions[0](x)
        torch.cuda.synchronize()
        stats.add(tuple(low.regions[0].last_spec.scalars()))
    assert len(stats) == 1


ARG = '''import torch

def f(x, y):
    h = x * 2
    __gm_pred_0 = h.argmax() > PIVOT
    __gm_then_a_0 = h + y
    __gm_else_a_0 = h - y
    a = torch.where(__gm_pred_0, __gm_then_a_0, __gm_else_a_0)
    __gm_pred_1 = a.argmin() < PIVOT
    z = torch.where(__gm_pred_1, a * 3, a)
    return z
'''


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("n", [13, 10007, 8 * 1024 * 768])
def test_argmax_argmin_predicates(n, dtype):
    """argmax / argmin predicates (data/attr_table.cfg) as fused reductions:
    ordered 64-bit keys (value order, first index on ties, NaN above all),
    branch decisions equal to torch's on CPU — including ties, -0.0/+0.0 and
    a NaN, and the maximum placed either side of the pivot."""
    pivot = n // 2
    text = ARG.replace("PIVOT", str(pivot))
    torch.manual_seed(n)
    cases = []
    for where in (pivot // 2, pivot + (n - pivot) // 2):
        x = torch.randn(n)
        x[where] = 50.0                       # unique maximum on one side
        y = torch.randn(n)
        cases.append((x, y))
    x = torch.round(torch.randn(n) * 2)       # many ties: the first index wins
    cases.append((x, torch.randn(n)))
    x = torch.zeros(n)
    x[: n // 3] = -0.0                        # -0.0 == +0.0: first occurrence
    cases.append((x, torch.ones(n)))
    x = torch.randn(n)
    x[n - 2] = float("nan")                   # NaN is the argmax and the argmin
    cases.append((x, torch.randn(n)))
    for x, y in cases:
        out, ref, ex, low = _run(text, "f", [x.to(dtype), y.to(dtype)], dtype)
        assert_parity(out, ref, dtype, what=f"argmax/argmin n={n}")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
def test_hoisted_max_guard(programs, dtype):
    """longformer_like: `scaled.max()` with `scaled = win * w0` is computed
    from max/min(win) at the first grid reduce (codegen.Plan._hoist); the
    guard sends non-finite cases (NaN, inf, overflow) through the exact
    sweep.  Every case equals torch eager on CPU."""
    from paper_2509_16248_b200 import codegen

    prog = programs["longformer_like"]
    text, fn = prog["transformed"], prog["callable"]
    torch.manual_seed(7)
    base = torch.randn(4, 512, 768)
    cases = {"normal": base.clone(), "all_negative": -base.abs() - 1.0}
    c = base.clone()
    c[1, 2, 3] = float("nan")
    cases["nan"] = c
    c = base.clone()
    c[0, 0, 5] = float("inf")
    cases["inf"] = c
    c = base.clone()
    c[2, 7, 9] = 3.0e38 if dtype == torch.float32 else 3.0e38
    cases["overflow"] = c
    for name, x in cases.items():
        x = x.to(dtype)
        out, ref, ex, low = _run(text, fn, [x], dtype)
        assert_parity(out, ref, dtype, what=f"longformer {name}")
    r = low.regions[0]
    assert r.last_spec.plan.hoisted, "the max was not hoisted"


@pytest.mark.gpu
def test_beyond_int32_elements():
    """A predicated block over 2^31 + 5 elements (beyond 32-bit indexing,
    with a partial tail vector): vector indices, staging decisions and the
    grid reduce are 64-bit.  Property check instead of the CPU oracle (4 GB
    per tensor): x = 1 everywhere, so sum > 0 and every output is 2."""
    n = 2 ** 31 + 5
    x = torch.ones(n, dtype=torch.bfloat16, device="cuda")
    ex, mod, low = compile_program(BLOCK, "f")
    out = ex(x, torch.ones((), dtype=torch.bfloat16, device="cuda"))
    torch.cuda.synchronize()
    assert any(r.stats.launches for r in low.regions)
    assert out.shape == (n,) and out.dtype == torch.bfloat16
    assert float(out.min()) == 2.0 and float(out.max()) == 2.0
    assert float(out[-1]) == 2.0 and float(out[2 ** 31]) == 2.0
    spec = low.regions[0].last_spec
    assert spec.status() == 0 and spec.plan.n == n


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16], ids=["bf16", "fp16"])
def test_tanh_16bit_matches_cpu_rounding(dtype):
    """tanh in a 16-bit region (evaluated in fp32, rounded once): against
    torch's CPU tanh rounded to the same type, at most 1 ulp apart and almost
    always identical — including tiny arguments, saturation, +-inf and NaN.
    (An SFU tanh, ex2/rcp + a Taylor branch, measured no faster on
    qwen_audio_like, so tanhf stays.)"""
    text = '''import torch

def t(x):
    __gm_pred_0 = x.abs().mean() > 1e9
    __gm_then_y_0 = torch.tanh(x) * 2
    __gm_else_y_0 = torch.tanh(x)
    return torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
'''
    g = torch.Generator().manual_seed(3)
    x = torch.cat([torch.randn(1 << 20, generator=g) * 3, torch.randn(1 << 16, generator=g) * 1e-3,
                   torch.linspace(-12, 12, 4097), torch.tensor([0.0, -0.0, 0.0625, -0.0625, 1e-30])]).to(dtype)
    x[-1] = float("inf")
    x[-2] = float("-inf")
    x[-3] = float("nan")
    out, ref, ex, low = _run(text, "t", [x])
    o, r = out.cpu(), ref
    assert torch.equal(o.isnan(), r.isnan())
    fin = ~r.isnan()
    ulp = (o[fin].view(torch.int16).int() - r[fin].view(torch.int16).int()).abs()
    assert int(ulp.max()) <= 1
    assert float((ulp != 0).float().mean()) < 1e-3


PRED = '''import torch

def f(x):
    __gm_pred_0 = RED
    __gm_then_y_0 = x * 2 + 1
    __gm_else_y_0 = x - 3
    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
    return y
'''


def _pm1(neg: int, twos: int, shape=(8, 1024, 768)) -> torch.Tensor:
    """+-1 with `neg` negative entries and `twos` entries 2.0: the product is
    +-2^twos exactly in any evaluation order (no order-dependent rounding)."""
    g = torch.Generator().manual_seed(neg * 7 + twos)
    n = math.prod(shape)
    x = torch.ones(n)
    perm = torch.randperm(n, generator=g)
    x[perm[:neg]] = -1.0
    x[perm[neg:neg + twos]] = 2.0
    return x.view(shape)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("red,make,want", [
    ("x.prod() > 0", lambda: _pm1(1000, 5), True),
    ("x.prod() > 0", lambda: _pm1(1001, 5), False),
    ("x.prod() >= 32.0", lambda: _pm1(2, 5), True),
    ("x.prod() >= 64.0", lambda: _pm1(2, 5), False),
    ("(x > 3.5).any()", lambda: torch.randn(8, 1024, 768, generator=torch.Generator().manual_seed(5)), True),
    ("(x > 6.5).any()", lambda: torch.randn(8, 1024, 768, generator=torch.Generator().manual_seed(5)), False),
    ("(x > -6.5).all()", lambda: torch.randn(8, 1024, 768, generator=torch.Generator().manual_seed(6)), True),
    ("(x > -3.0).all()", lambda: torch.randn(8, 1024, 768, generator=torch.Generator().manual_seed(6)), False),
    ("x.any()", lambda: torch.zeros(8, 1024, 768), False),
    ("x.all()", lambda: _pm1(7, 0), True),
], ids=["prod_pos", "prod_neg", "prod_ge32", "prod_ge64", "any_t", "any_f", "all_t", "all_f", "any_zero", "all_pm1"])
def test_prod_any_all_predicates(red, make, want, dtype):
    """prod / any / all predicates (data/attr_table.cfg:8-9,14) at
    [8,1024,768] as fused reductions: decision and output equal the
    reference's CPU eager execution of the same transformed text."""
    from parity import check_scalars

    text = PRED.replace("RED", red)
    x = make().to(dtype)
    ref = orc.reference_callable(text, "f")(x.clone())
    ex, mod, low = compile_program(text, "f")
    out = ex(x.cuda())
    torch.cuda.synchronize()
    assert low.regions[0].stats.launches >= 1 and low.regions[0].stats.fallbacks == 0
    ref_decision = bool(orc.reference_callable("import torch\n\ndef p(x):\n    return " + red + "\n", "p")(x.clone()))
    assert ref_decision == want
    assert check_scalars(low, text, "f", [x], dtype, what=red) == 1
    assert_parity(out, ref, dtype, what=red)

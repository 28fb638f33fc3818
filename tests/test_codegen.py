"""Region code generation decisions (CPU, no GPU): speculation eligibility,
launch layout, staging, the exact-multiply rewrite of x / 2^k, arm aliasing,
and the fixed-shape distinct-value sum's CPU form."""

import math

import pytest
import torch

from paper_2509_16248_b200 import _native as nat
from paper_2509_16248_b200 import codegen, lowering
from paper_2509_16248_b200.logring import ModuleRuntime


def _plan(programs, name, dtype, shape, idx=0):
    mod, low = lowering.load(programs[name]["transformed"], allow_eager=True)
    r = low.regions[idx]
    args = []
    for fv in r.graph.frees:
        if fv.text.startswith("self."):
            args.append(getattr(getattr(mod, programs[name]["callable"]), fv.text[5:]))
        else:
            args.append(torch.randn(shape).to(dtype))
    return codegen.Plan(r.graph, r.out_nodes, args, r.name, allow_cpu=True)


def test_phi4_chain_is_speculative(programs):
    """corpus phi4_like: 5 chained predicated blocks -> 5 boolean decisions,
    one speculative sweep, 6-pass exact fallback."""
    plan = _plan(programs, "phi4_like", torch.bfloat16, (8, 1024, 768))
    assert plan.npass == 6 and len(plan.reductions) == 5
    assert plan.spec and len(plan.decisions) == 5
    assert all(d.dtype == torch.bool for d in plan.decisions)
    assert "speculative pass" in plan.source and "// ---- pass 5" in plan.source
    assert plan.grid == 296 and plan.K == 6 and plan.minb == 2


def test_wide_fp32_region_runs_one_cta_per_sm(programs):
    """fp32 vectors and >= 3 reductions: 128 registers a thread (one CTA per
    SM) instead of spilling at 64."""
    plan = _plan(programs, "phi4_like", torch.float32, (8, 1024, 768))
    assert plan.minb == 1 and plan.grid == 148
    assert "__launch_bounds__(GM_THREADS, 1)" in plan.source


def test_float_item_scalars_are_not_speculated(programs):
    """longformer_like: `.item()` values feed arithmetic (not a boolean
    decision), so the region is the exact 3-pass kernel with its input
    staged on chip (read from HBM once)."""
    plan = _plan(programs, "longformer_like", torch.bfloat16, (4, 4096, 768))
    assert plan.npass == 3 and not plan.spec
    assert plan.stage[0] in ("reg", "smem")
    assert "speculative pass" not in plan.source


def test_monotone_max_is_hoisted(programs, monkeypatch):
    """longformer_like: `peak = (win * w0).max()` is taken from max/min(win)
    at pass 0's grid reduce; pass 1's sweep runs only if the device-side
    finiteness guard fails.  GM_HOIST=0 keeps the 3-sweep kernel."""
    plan = _plan(programs, "longformer_like", torch.bfloat16, (4, 4096, 768))
    assert list(plan.hoisted) == [1]
    (r, e, y, s, direction, hmax, hmin), = plan.hoisted[1]
    assert r.op == "amax" and e.op == "mul" and direction == 0
    assert hmax in plan.pass_reds[0] and hmin in plan.pass_reds[0]
    assert "if (!s_hoist1)" in plan.source
    monkeypatch.setenv("GM_HOIST", "0")
    plan = _plan(programs, "longformer_like", torch.bfloat16, (4, 4096, 768))
    assert not plan.hoisted and "s_hoist" not in plan.source
    assert [len(plan.pass_reds[p]) for p in range(3)] == [1, 1, 0]


@pytest.mark.parametrize("v,expect", [(2.0, 0.5), (0.5, 2.0), (-4.0, -0.25), (3.0, None), (0.0, None),
                                      (float("inf"), None), (2.0 ** 127, None), (1.0, 1.0)])
def test_pow2_reciprocal(v, expect):
    assert codegen.Plan._pow2_recip(v) == expect


def test_division_by_power_of_two_is_a_multiply(programs):
    """phi4 `a / 2` is emitted as gm::mul(a, 0.5f) (bit-identical: both are
    the correctly rounded a * 2^-1) instead of an IEEE division."""
    plan = _plan(programs, "phi4_like", torch.float32, (8, 1024, 768))
    assert "gm::div(" not in plan.source.split("// misprediction")[0]
    assert "0.5f)" in plan.source


def test_select_arms_write_into_the_select(programs):
    """bigbird region 0: the then/else `ctx` arms are computed straight into
    the select's registers, so no separate arm arrays are declared."""
    plan = _plan(programs, "bigbird_like", torch.bfloat16, (8, 1024, 768))
    spec = plan.source.split("// ---- speculative pass")[1].split("grid_wait")[0]
    wheres = [n for n in plan.order if n.op == "where" and n.args[0].kind != "elem"]
    assert wheres
    for w in wheres:
        for arm in w.args[1:]:
            if arm.kind == "elem" and arm.op != "free":
                assert f"p{arm.uid}_0[4];" not in spec and f"n{arm.uid}_0[GM_VEC];" not in spec


def test_generated_regions_compile(programs):
    for name, shape in (("phi4_like", (8, 1024, 768)), ("longformer_like", (4, 4096, 768))):
        for dt in (torch.float32, torch.bfloat16):
            plan = _plan(programs, name, dt, shape)
            assert nat.compile_cubin(plan.source, (10, 0))[:4] == b"\x7fELF"


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_unique_sum_cpu_form(dtype):
    """The fixed-shape form (sort, first of each run, sum) equals
    x.unique().sum() — including -0.0/+0.0 and repeated values."""
    torch.manual_seed(0)
    x = torch.randint(-20, 20, (5000,)).to(dtype) / 4
    x[0], x[1] = 0.0, -0.0
    got = ModuleRuntime.unique_sum(x)
    ref = x.unique().sum()
    assert math.isclose(float(got), float(ref), rel_tol=1e-2 if dtype == torch.bfloat16 else 1e-6)


def test_speculative_region_has_adaptive_entries(programs):
    """An adaptive speculative region: the confidence counter picks the
    speculative sweep (then, on a miss, the restart from the first
    mispredicted level, unstaged) or the exact entry, whose passes keep the
    input on chip (register / shared-memory staging)."""
    plan = _plan(programs, "bigbird_like", torch.bfloat16, (8, 1024, 768), idx=1)
    assert plan.spec
    src = plan.source
    assert "GM_SCRATCH_CONF" in src and "s_mode" in src
    spec_part, exact_part = src.split("// exact entry")
    assert "speculative pass" in spec_part and "if (s_miss <= 1)" in spec_part
    # nothing is staged in shared memory; the exact entry pulls the input
    # its select pass reads first (`hidden`) into L2 during the norm pass
    assert plan.smem_bytes == 0 and all(st == "none" for st in plan.stage.values())
    assert "prefetch_l2" in exact_part
    # a 2-pass bf16 block keeps the history predictor (the sample pass would
    # cost what the exact entry costs over a hit)
    assert not plan.sampled


def test_sampled_prediction(programs, monkeypatch):
    """Speculative regions whose reductions have a sample estimate (sum,
    mean, norm, count, max, min, any, all) predict their decisions from data:
    one scrambled 4K-element sample evaluated in every CTA (the default), or
    (GM_SAMPLE=cta, measured slower) every CTA from the first vector of each
    of its threads, the grid reduce carrying each decision's min / max over
    CTAs and whether all certified.  prod / argmax predicates keep the last
    launch's decisions."""
    monkeypatch.setenv("GM_SAMPLE", "cta")
    plan = _plan(programs, "bigbird_like", torch.float32, (8, 1024, 768))
    assert plan.spec and plan.cta_pred and not plan.sampled
    src = plan.source
    assert "per-CTA prediction" in src and "cta_sum2" in src
    spec = src.split("// ---- speculative pass")[1].split("// exact entry")[0]
    assert "pred_ + 0" not in spec                        # no last-launch prediction read
    assert plan.extra_slots() == 3 and "const int ops_[4]" in spec   # 1 reduction + min/max + certified
    assert len(nat.compile_cubin(src, (10, 0))) > 0
    monkeypatch.delenv("GM_SAMPLE")
    plan = _plan(programs, "bigbird_like", torch.float32, (8, 1024, 768))
    assert plan.sampled and not plan.cta_pred
    src = plan.source
    assert "sampled prediction" in src and "2654435761" in src and "cta_sum2" in src
    spec = src.split("// ---- speculative pass")[1].split("grid_arrive")[0]
    assert "s_pred[0] != 0" in spec and "pred_ + 0" not in spec
    text = '''
import torch
def f(x):
    __gm_pred_0 = x.prod() > 0
    __gm_then_y_0 = x * 2
    y = torch.where(__gm_pred_0, __gm_then_y_0, x)
    return y
'''
    low, _ = lowering.lower(text)
    r = low.regions[0]
    p = codegen.Plan(r.graph, r.out_nodes, [torch.randn(8, 1024, 768)], allow_cpu=True)
    assert p.spec and not p.sampled and "sampled prediction" not in p.source

"""Lowering of transformed programs (CPU): structure, liveness, and exact
equivalence of the lowered program with the reference's transformed text
when regions run their original statements (tensors on CPU)."""

import ast

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import codegen, lowering
from paper_2509_16248_b200 import _native as nat

ALL = ["bart_step", "bigbird_like", "biogpt_like", "blenderbot_like", "flan_t5_like", "longformer_like",
       "moe_minicpm_like", "pegasus_like", "phi4_like", "qwen_audio_like", "toy"]


def test_phi4_is_one_region(programs):
    low, _ = lowering.lower(programs["phi4_like"]["transformed"])
    assert len(low.regions) == 1
    r = low.regions[0]
    assert [fv.text for fv in r.graph.frees] == ["x"]
    # h, a..d and every __gm_* temporary stay on chip; only the result leaves
    assert len(r.out_names) == 1 and r.out_names[0].startswith("__gm_retv_")


def test_bigbird_regions_and_replay(programs):
    low, _ = lowering.lower(programs["bigbird_like"]["transformed"])
    assert [r.out_names for r in low.regions] == [["ctx"], ["res"]]
    assert [fv.text for fv in low.regions[0].graph.frees] == ["q", "self.scale", "hidden"]
    assert [(s.callee_src, s.capture_name) for s in low.sites] == [("logger.info", "__gm_defer_0")]
    tree = ast.parse(low.source)
    calls = [n for n in ast.walk(tree) if isinstance(n, ast.Call) and isinstance(n.func, ast.Attribute)
             and n.func.attr == "replay"]
    assert len(calls) == 1


def test_capture_hoisted_not_splitting(programs):
    """biogpt: two deferrals between elementwise statements -> one region."""
    low, _ = lowering.lower(programs["biogpt_like"]["transformed"])
    assert len(low.regions) == 1
    assert len(low.sites) == 2


def test_longformer_item_reads_become_device_scalars(programs):
    """`w = t.item()` feeding only tensor arithmetic stays a
    device scalar, so the three host reads vanish and the forward is one
    3-pass region; the dead final read (`w2`) is dropped."""
    low, _ = lowering.lower(programs["longformer_like"]["transformed"])
    assert [r.out_names for r in low.regions] == [["shifted"]]
    assert "item" not in low.source.split("def forward")[1].split("compiled_forward")[0]


def test_moe_dynamic_shape_ops_lowered(programs):
    """nonzero / unique / masked_select consumed only by
    .sum() become fixed-shape reductions (no data-dependent output size)."""
    low, _ = lowering.lower(programs["moe_minicpm_like"]["transformed"])
    ops = [op for _, op in low.dynamic_shape_lowered]
    assert ops.count("nonzero") == 5 and ops.count("unique") == 5 and ops.count("masked_select") == 5
    body = low.source.split("def forward")[1].split("compiled_forward")[0]
    assert "nonzero(" not in body and ".unique()" not in body and "masked_select" not in body


def test_name_mangling_safe():
    src = ("import torch\nclass M(torch.nn.Module):\n    def forward(self, x):\n        __gm_pred_0 = x.sum() > 0\n"
           "        __gm_then_y_0 = x + 1\n        __gm_else_y_0 = x - 1\n"
           "        y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)\n        return y * 2\nm = M()\n")
    mod, low = lowering.load(src, allow_eager=True)
    x = torch.randn(5)
    assert torch.equal(mod.m(x), torch.where(x.sum() > 0, x + 1, x - 1) * 2)


@pytest.mark.parametrize("name", ALL)
def test_lowered_equals_transformed_on_cpu(programs, name):
    """With CPU tensors every region runs its original statements and every
    replay is immediate, so the lowered program must be bit-identical to the
    reference's transformed program — this pins liveness, hoisting, return
    splitting and the fallback functions."""
    p = programs[name]
    for spec in p["inputs"]:
        shapes = None
        if name == "bigbird_like":
            shapes = [[1, 32, 768]]
        elif name == "bart_step":
            shapes = [[4, 1, 768]]
        args = orc.make_args(spec["args"], spec["seed"], shapes=shapes)
        ref, rt = orc.run_reference(p["transformed"], p["callable"], args)
        mod, low = lowering.load(p["transformed"], allow_eager=True)
        out, t = orc.call_captured(getattr(mod, p["callable"]), args)
        assert t == rt
        assert torch.equal(out, ref) if isinstance(ref, torch.Tensor) else out == ref
        assert all(r.stats.launches == 0 for r in low.regions)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("name", ["phi4_like", "bigbird_like", "qwen_audio_like", "flan_t5_like"])
def test_region_codegen_compiles_for_sm100a(programs, name, dtype):
    """Every region of the BASELINE-shaped programs specialises and its
    generated source compiles with NVRTC for sm_100a (no GPU needed)."""
    mod, low = lowering.load(programs[name]["transformed"], allow_eager=True)
    for r in low.regions:
        args = []
        for fv in r.graph.frees:
            if fv.text.startswith("self."):
                args.append(getattr(mod.model, fv.text[5:]))
            elif name == "flan_t5_like":
                args.append(torch.randn(8192, 768).to(dtype))
            else:
                args.append(torch.randn(8, 1024, 768).to(dtype))
        plan = codegen.Plan(r.graph, r.out_nodes, args, r.name, allow_cpu=True)
        cubin = nat.compile_cubin(plan.source, (10, 0))
        assert cubin[:4] == b"\x7fELF"


def test_uniform_select_guards_untaken_arm(programs, monkeypatch):
    """bigbird region 0: `hidden` is read only by the else arm, so its load
    sits under the negated predicate and never happens when the then arm is
    selected (the reference evaluates both arms, transform.py:404-412) — in
    the speculative pass and in the exact fallback passes alike."""
    mod, low = lowering.load(programs["bigbird_like"]["transformed"], allow_eager=True)
    r = low.regions[0]
    args = [torch.randn(8, 64, 768), 0.125, torch.randn(8, 64, 768)]
    plan = codegen.Plan(r.graph, r.out_nodes, args, r.name, allow_cpu=True)
    assert plan.npass == 2 and len(plan.reductions) == 1
    assert plan.spec and len(plan.decisions) == 1
    src = plan.source
    for marker in ("// ---- speculative pass", "// ---- pass 1"):
        i = src.index(marker)
        j = src.index("P.in[1]", i)
        assert "if ((!sb" in src[i:j], marker
    # exact (non-speculative) specialisation: q is read by both passes and
    # stays in registers across the grid barrier; hidden is read only by the
    # else arm of pass 1, so it is not prefetched (an untaken arm must cost
    # no HBM traffic) and loads lazily under the guard
    monkeypatch.setenv("GM_SPEC", "0")
    plan = codegen.Plan(r.graph, r.out_nodes, args, r.name, allow_cpu=True)
    assert not plan.spec
    assert plan.stage == {0: "reg", 1: "none"}
    src = plan.source
    i = src.index("// ---- pass 1")
    j = src.index("P.in[1]", i)
    assert "if ((!sb" in src[i:j]


def test_boolean_predicates_lowered():
    """and/or/not of 0-d bool predicates become device logical ops
     — the whole transformed forward is one region."""
    src = ("import torch\n\ndef f(x):\n    h = x * 2\n    __gm_pred_0 = (h.sum() > 0) and (h.max() < 5)\n"
           "    __gm_then_y_0 = h + 1\n    __gm_else_y_0 = h - 1\n"
           "    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)\n"
           "    __gm_pred_1 = not (y.mean() > 0)\n    z = torch.where(__gm_pred_1, y * 3, y)\n    return z\n")
    low, _ = lowering.lower(src)
    assert [r.out_names for r in low.regions] == [["z"]]
    plan = codegen.Plan(low.regions[0].graph, low.regions[0].out_nodes, [torch.randn(4096)], "f", allow_cpu=True)
    assert plan.npass == 3
    nat.compile_cubin(plan.source, (10, 0))


def test_calls_hoisted_out_of_elementwise_expressions(programs):
    """bart_step: `out = self.fc2(f) + h` becomes `t = self.fc2(f); out = t + h`
    so the add fuses with the epilogue `out * 0.5` (the Linear call itself
    goes through the runtime's GEMM entry, gemm.module_call);
    `relu(self.fc1(h))` becomes one cuBLASLt GEMM with a RELU_BIAS epilogue
    (linear_relu)."""
    low, _ = lowering.lower(programs["bart_step"]["transformed"])
    assert [r.out_names for r in low.regions] == [["h"], ["__gm_ret_0"]]
    body = low.source.split("def forward")[1]
    assert "__gm_rt__.linear_relu(self.fc1, h)" in body
    assert "= __gm_rt__.call(self.fc2, f)" in body and "torch.relu" not in body


def test_linear_relu_cpu_fallback_is_exact():
    from paper_2509_16248_b200.logring import ModuleRuntime

    torch.manual_seed(0)
    lin = torch.nn.Linear(16, 8)
    x = torch.randn(3, 5, 16)
    assert torch.equal(ModuleRuntime.linear_relu(lin, x), torch.relu(lin(x)))


def test_dynamic_shape_def_evaluated_at_its_site():
    """`idx = nonzero(x > 0.5); x = x * 0.1; idx.sum()` —
    the fixed-shape replacement is evaluated where `idx` was defined, so the
    rebinding of `x` in between cannot change it (eager: 1097.2-style sums,
    not the rebound x's)."""
    src = ("import torch\n\ndef f(x):\n    idx = torch.nonzero(x > 0.5)\n    x = x * 0.1\n"
           "    m = torch.masked_select(x, x > 0.01)\n    x = x + 1\n    return idx.sum() + m.sum() + x.sum()\n")
    mod, low = lowering.load(src, allow_eager=True)
    assert sorted(op for _, op in low.dynamic_shape_lowered) == ["masked_select", "nonzero"]
    torch.manual_seed(0)
    x = torch.rand(64, 32)
    ns = {}
    exec(compile(src, "f", "exec"), ns)
    ref = ns["f"](x.clone())
    out = mod.f(x.clone())
    assert torch.equal(out, ref), (out, ref)


def test_names_read_by_nested_scopes_stay_live():
    """a lambda defined before `h` is assigned reads it
    when called later — `h` must stay a region output."""
    src = ("import torch\n\ndef f(x):\n    g = lambda: h * 2\n    h = x + 1\n    y = h * 3\n    return g() + y\n")
    mod, low = lowering.load(src, allow_eager=True)
    x = torch.randn(16)
    assert torch.equal(mod.f(x), (x + 1) * 2 + (x + 1) * 3)
    assert any("h" in r.out_names for r in low.regions)


def test_unsupported_region_raises_without_allow_eager():
    """No silent fallback: CPU tensors (or any argument the fused kernel
    cannot take) raise RegionUnsupported unless the caller opts in."""
    from paper_2509_16248_b200.region import RegionUnsupported

    src = "import torch\n\ndef f(x):\n    y = x * 2 + 1\n    return y\n"
    mod, low = lowering.load(src)
    with pytest.raises(RegionUnsupported):
        mod.f(torch.randn(8))
    mod, low = lowering.load(src, allow_eager=True)
    assert torch.equal(mod.f(torch.ones(8)), torch.full((8,), 3.0))
    assert low.regions[0].stats.fallbacks == 1


def test_gemm_arms_become_one_selected_gemm(programs):
    """both arms of the gemm_arms block hold a
    torch.matmul; the lowering replaces the pair by ONE select_gemm read by
    both arms, whose selects and epilogues fuse into one region; on CPU
    (allow_eager) the lowered program equals the transformed one."""
    p = programs["gemm_arms"]
    low, _ = lowering.lower(p["transformed"])
    assert low.gemm_arms == [("__gm_pred_0", "matmul")]
    body = low.source.split("def forward")[1]
    assert body.count("select_gemm(") == 1 and "torch.matmul" not in body
    assert "__gm_rt__.call(self.query, hidden)" in body
    for spec in p["inputs"]:
        args = orc.make_args(spec["args"], spec["seed"], shapes=[[1, 32, 768]])
        ref, rt = orc.run_reference(p["transformed"], p["callable"], args)
        mod, low = lowering.load(p["transformed"], allow_eager=True)
        out, t = orc.call_captured(getattr(mod, p["callable"]), args)
        assert t == rt and torch.equal(out, ref)


def test_rematerialise_only_when_safe():
    """lowering._rematerialise: a cheap elementwise value read by a grid
    reduction AND a row operator is recomputed at each use — never when a
    name it reads is rebound before its last use, when it is read in a
    nested scope, or when it is assigned twice."""
    base = '''
import torch
def f(t, b):
    s = t / 8.0
    p = s.abs().mean() > 0.3
    y = torch.where(p, torch.softmax(s + b, -1), torch.softmax(s, -1))
    return y
'''
    low, _ = lowering.lower(base)
    assert "s = " not in low.source.split("def f")[1].split("regions")[0]
    assert all("s" not in r.out_names for r in low.regions)
    rebound = base.replace("    p = s.abs().mean() > 0.3\n", "    p = s.abs().mean() > 0.3\n    t = t * 2\n")
    low, _ = lowering.lower(rebound)
    assert any("s" in r.out_names for r in low.regions)
    nested = base.replace("    return y\n", "    g = lambda: s\n    return y\n")
    low, _ = lowering.lower(nested)
    assert any("s" in r.out_names for r in low.regions)
    # values the same: CPU eager of the lowered program
    t, b = torch.randn(4, 8, 16), torch.randn(16)
    mod, _ = lowering.load(base, allow_eager=True)
    ns = {}
    exec(compile(base, "f", "exec"), ns)
    assert torch.equal(mod.f(t, b), ns["f"](t, b))


def test_reshape_of_computed_values_routes_through_runtime():
    text = '''
import torch
def f(x, w):
    y = torch.matmul(x, w).transpose(1, 2).reshape(2, 8, 12)
    z = x.contiguous()
    return y, z
'''
    low, _ = lowering.lower(text)
    src = low.source
    assert "__gm_rt__.reshape(" in src and "__gm_rt__.contiguous(x)" in src
    mod, _ = lowering.load(text, allow_eager=True)
    x, w = torch.randn(2, 3, 8, 5), torch.randn(5, 4)
    ns = {}
    exec(compile(text, "f", "exec"), ns)
    a, b = mod.f(x, w), ns["f"](x, w)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_fx_form_scores_rematerialised_and_gelu_fused():
    """Dynamo's FX source writes one op per line (`scores = mm / 8.0`,
    `abs_1 = scores.abs()`, `add = scores + bias`, `torch._C._nn.gelu`):
    the scaled scores reach the predicate's reduction and the softmaxes only
    through elementwise statements, and `add` feeds a softmax only.  Both are
    recomputed where they are read, so the grid region writes the predicate
    alone and the row region reads the GEMM output and the mask — neither
    [B, H, L, L] intermediate is materialised."""
    text = '''
import torch
def forward(mm, mask, h):
    scores = mm / 8.0
    abs_1 = scores.abs()
    mean = abs_1.mean()
    p = mean > 0.35
    add = scores + mask
    a = torch.softmax(add, dim=-1)
    b = torch.softmax(scores, dim=-1)
    probs = torch.where(p, a, b)
    inter = torch._C._nn.gelu(h)
    return probs, inter
'''
    low, _ = lowering.lower(text)
    assert [r.out_names for r in low.regions] == [["p"], ["probs", "inter"]]
    assert sorted(fv.text for fv in low.regions[1].graph.frees) == ["h", "mask", "mm", "p"]
    assert "torch._C._nn.gelu" not in low.source
    assert any("gelu" in {n.op for n in r.graph.nodes} for r in low.regions)


LN_BLOCK = '''
import torch
class Block(torch.nn.Module):
    def __init__(self, h):
        super().__init__()
        self.out = torch.nn.Linear(h, h)
        self.norm = torch.nn.LayerNorm(h, eps=1e-12)
        self.norm2d = torch.nn.LayerNorm((4, h))
        self.swapped = torch.nn.LayerNorm(h)
        self.swapped = torch.nn.Identity()
    def forward(self, x):
        y = self.norm(self.out(x) + x)
        z = self.swapped(y) * 2
        return z
'''


def test_layer_norm_modules_inlined_and_fused_with_the_residual_add():
    """`self.norm(self.out(x) + x)` with `self.norm = nn.LayerNorm(h, eps)`
    built once in __init__: the call becomes F.layer_norm with the module's
    parameters (Dynamo's FX form), so the residual add and the LayerNorm are
    ONE row region after the GEMM.  Attributes assigned twice, or with a
    multi-dimensional shape, stay module calls."""
    low, lw = lowering.lower(LN_BLOCK)
    assert lw.inlined_layer_norms == ["Block.norm"]
    assert "inlined_layer_norms(self, ('norm',))" in low.source
    r = low.regions[0]
    assert r.out_names == ["y"]
    assert "layer_norm" in {n.op for n in r.graph.nodes} and "add" in {n.op for n in r.graph.nodes}
    assert "__gm_rt__.call(self.swapped" in low.source


def test_inlined_layer_norm_runs_and_guards_on_cpu():
    """Eager (allow_eager, CPU) the inlined statement computes what the
    module computes, bit for bit; a hook added to the module later makes the
    forward raise instead of silently skipping it."""
    mod, low = lowering.load(LN_BLOCK, allow_eager=True)
    torch.manual_seed(0)
    blk = mod.Block(16)
    x = torch.randn(3, 5, 16)
    with torch.no_grad():
        y = blk(x)
        ref = blk.swapped(blk.norm(blk.out(x) + x)) * 2
    assert torch.equal(y, ref)
    blk.norm.register_forward_hook(lambda m, i, o: o)
    with pytest.raises(RuntimeError, match="lowered as F.layer_norm"):
        blk(x)

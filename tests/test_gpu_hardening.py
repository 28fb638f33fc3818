"""predicate hardening.

The reference copies predicate source verbatim (transform.py:386-388) and
reports these sites fixed with residual 0, but at runtime
  * `p and q` on tensor predicates calls Tensor.__bool__ (a host sync),
  * `not p` hands torch.where a Python bool and raises (torch 2.11), and
  * `mask is None` (parameters are taint seeds, analysis.py:340-344) hands
    torch.where a Python bool and evaluates the arm that reads None.
The B200 lowering evaluates and/or/not of 0-d bool predicates on the device
and resolves `is None` / `is not None` on the host when the region is
specialised (ir.fold_host_predicates), keeping only the selected arm.
The checker is the ORIGINAL (untransformed) program on CPU, whose `if`
semantics the rewrite is meant to preserve."""

import os
import subprocess
import sys

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import compile_program
from parity import assert_parity

ORIGINAL = '''import torch

def f(x):
    h = x * 2
    if (h.sum() > 0) and (h.max() < 5):
        y = h + 1
    else:
        y = h - 1
    if not (y.mean() > 0):
        z = y * 3
    else:
        z = y
    return z

fc = torch.compile(f)
'''

# what the reference fix_file returns for ORIGINAL (generated in the build
# container with /root/reference; 2 found, 2 fixed, predicted residual 0)
TRANSFORMED = '''import torch

def f(x):
    h = x * 2
    __gm_pred_0 = (h.sum() > 0) and (h.max() < 5)
    __gm_then_y_0 = h + 1
    __gm_else_y_0 = h - 1
    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
    __gm_pred_1 = not (y.mean() > 0)
    __gm_then_z_0 = y * 3
    __gm_else_z_0 = y
    z = torch.where(__gm_pred_1, __gm_then_z_0, __gm_else_z_0)
    return z

fc = torch.compile(f)
'''


ORIGINAL_NONE = '''import torch


class M(torch.nn.Module):
    def forward(self, x, mask):
        h = x * 2
        if mask is None:
            y = h + 1
        else:
            y = h + mask
        return y


model = M()
compiled = torch.compile(model)
'''

# fix_file(ORIGINAL_NONE): 1 found, 1 fixed, predicted residual 0
TRANSFORMED_NONE = '''import torch


class M(torch.nn.Module):
    def forward(self, x, mask):
        h = x * 2
        __gm_pred_0 = mask is None
        __gm_then_y_0 = h + 1
        __gm_else_y_0 = h + mask
        y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
        return y


model = M()
compiled = torch.compile(model)
'''


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not present (GPU box)")
@pytest.mark.parametrize("original,transformed", [(ORIGINAL, "TRANSFORMED"), (ORIGINAL_NONE, "TRANSFORMED_NONE")])
def test_fixtures_are_the_reference_rewrite(original, transformed):
    """The embedded transformed texts are exactly what the reference fix_file
    returns for the embedded originals (transform.py:822-936)."""
    code = ("import sys; sys.path.insert(0, '/root/reference/pkg/src')\n"
            "from graphmend.transform import fix_file\nfrom graphmend.frontend import SourceModule\n"
            "t, o = fix_file(SourceModule.from_text('f.py', sys.stdin.read()))\n"
            "print(o.found, o.fixed, o.predicted_residual); sys.stdout.write(t)")
    r = subprocess.run([sys.executable, "-c", code], input=original, capture_output=True, text=True, check=True)
    counts, text = r.stdout.split("\n", 1)
    assert text == globals()[transformed]
    assert counts.split()[1] == counts.split()[0] and counts.split()[2] == "0"


def test_reference_is_none_rewrite_fails_at_runtime_on_cpu():
    """`mask is None` reaches torch.where as a Python bool: the reference's
    transformed program raises for a None mask and for a tensor mask."""
    fn = orc.reference_callable(TRANSFORMED_NONE, "model")
    x = torch.randn(4, 16)
    for mask in (None, torch.randn(4, 16)):
        with pytest.raises(TypeError):
            fn(x.clone(), mask)


def test_is_none_resolved_at_specialisation_cpu():
    """fold_host_predicates keeps only the selected arm: the None-mask
    specialisation reads one input, the tensor-mask one reads two, and both
    generate sm_100a code."""
    from paper_2509_16248_b200 import _native as nat
    from paper_2509_16248_b200 import codegen, lowering
    from paper_2509_16248_b200.ir import fold_host_predicates

    low, _ = lowering.lower(TRANSFORMED_NONE)
    assert [r.out_names for r in low.regions] == [["y"]]
    r = low.regions[0]
    x = torch.randn(8, 1024, 768)
    for mask, n_in in ((None, 1), (torch.randn(8, 1024, 768), 2)):
        g, outs = fold_host_predicates(r.graph, r.out_nodes, [x, mask])
        plan = codegen.Plan(g, outs, [x, mask], r.name, allow_cpu=True)
        assert len(plan.inputs) == n_in and not plan.reductions
        nat.compile_cubin(plan.source, (10, 0))


def test_reference_rewrite_fails_at_runtime_on_cpu():
    """The defect being hardened: the transformed `not` predicate raises."""
    fn = orc.reference_callable(TRANSFORMED, "f")
    with pytest.raises(TypeError):
        fn(torch.full((64,), -1.0))


@pytest.mark.gpu
@pytest.mark.parametrize("fill", [1.0, 4.0, -1.0, None])
def test_hardened_predicates_match_original(fill):
    x = torch.randn(8, 1024, 768) if fill is None else torch.full((8, 1024, 768), fill)
    ref = orc.reference_callable(ORIGINAL, "f")(x.clone())
    ex, mod, low = compile_program(TRANSFORMED, "f")
    out = ex(x.cuda())
    torch.cuda.synchronize()
    info = ex.info()[0]
    assert info.mode == "graph" and info.host_syncs == 0, info
    assert low.regions[0].stats.launches >= 1
    assert_parity(out, ref, torch.float32, what=f"hardened fill={fill}")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
def test_is_none_predicate_matches_original(dtype):
    """`if mask is None` on the B200: one CUDA graph per mask type, only the
    selected arm runs, and the result equals the ORIGINAL program's eager
    CPU output (the reference's rewrite itself raises)."""
    torch.manual_seed(3)
    x = torch.randn(8, 1024, 768).to(dtype)
    m = torch.randn(8, 1024, 768).to(dtype)
    ex, mod, low = compile_program(TRANSFORMED_NONE, "model", dtype=dtype)
    orig = orc.reference_callable(ORIGINAL_NONE, "model", dtype)
    for mask in (None, m, None):
        ref = orig(x.clone(), None if mask is None else mask.clone())
        out = ex(x.cuda(), None if mask is None else mask.cuda())
        assert_parity(out, ref, dtype, what=f"is None, mask={'None' if mask is None else 'tensor'}")
    assert all(i.mode == "graph" and i.host_syncs == 0 for i in ex.info())
    assert low.regions[0].stats.launches >= 3 and low.regions[0].stats.fallbacks == 0

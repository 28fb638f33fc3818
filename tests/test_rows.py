"""Row regions (rowgen.py) and the rest of the purity gate's vocabulary on
the CPU: softmax / log_softmax and sum/mean/amax/amin over the innermost dim
(data/pure_ops.cfg:18, attr_table.cfg:4-7 with `dim`), `//` and `%`
(transform.py:59-61) and basic subscripts of enclosing-scope values
(transform.py:245-254).  Lowering decisions, launch geometry and NVRTC
compilation for sm_100a; the GPU parity tests are tests/test_gpu_rows.py."""

import pytest
import torch

from paper_2509_16248_b200 import _native as nat
from paper_2509_16248_b200 import codegen, lowering
from paper_2509_16248_b200.ir import ROW_OPS
from paper_2509_16248_b200.rowgen import RowPlan, has_row_ops

SOFTMAX_ARM = '''
import torch
def f(x):
    __gm_pred_0 = x.sum() > 0
    __gm_then_y_0 = torch.softmax(x * 0.125, dim=-1)
    y = torch.where(__gm_pred_0, __gm_then_y_0, x)
    return y
'''

ROWS = '''
import torch
def f(x, b, m):
    mx = x.amax(-1, keepdim=True)
    e = (x - mx).exp()
    p = e / e.sum(-1, keepdim=True)
    q = torch.log_softmax(x + b, -1) * m
    r = x.mean(-1)
    return p + q, r
'''


def _region_plans(text, shapes, dtype=torch.float32):
    low, _ = lowering.lower(text)
    plans = []
    for r in low.regions:
        args = []
        for fv in r.graph.frees:
            if fv.text.startswith("__gm_pred"):
                args.append(torch.tensor(True))
            else:
                args.append(torch.randn(shapes[fv.text]).to(dtype))
        cls = RowPlan if has_row_ops(r.out_nodes) else codegen.Plan
        plans.append(cls(r.graph, r.out_nodes, args, r.name, allow_cpu=True))
    return low, plans


def test_softmax_arm_splits_into_grid_then_row_region():
    """The predicate statistic is a grid reduction, the softmax a row
    operator: the run becomes a grid region producing the 0-d predicate and a
    row region holding the arm and the select (lowering._row_mixing)."""
    low, plans = _region_plans(SOFTMAX_ARM, {"x": (8, 1024, 768)})
    assert len(low.regions) == 2
    assert not has_row_ops(low.regions[0].out_nodes) and low.regions[0].out_names == ["__gm_pred_0"]
    assert has_row_ops(low.regions[1].out_nodes) and low.regions[1].out_names == ["y"]
    row = plans[1]
    assert isinstance(row, RowPlan)
    assert (row.R, row.C, row.TPR, row.U, row.RPC, row.grid) == (8192, 768, 32, 3, 4, 2048)
    assert row.vec8
    # the untaken arm is skipped by a uniform branch on the predicate
    assert "if (sb" in row.source
    for p in plans:
        assert len(nat.compile_cubin(p.source, (10, 0))) > 0


@pytest.mark.parametrize("shape,tpr,u", [((4, 7, 20), 1, 3), ((3, 5000), 256, 3), ((2, 3, 1), 1, 1),
                                         ((16, 4096), 128, 4), ((2, 32768), 1024, 4)])
def test_row_geometry_and_compile(shape, tpr, u):
    shapes = {"x": shape, "b": shape[-1:], "m": shape[:-1] + (1,)}
    for dt in (torch.float32, torch.bfloat16):
        low, plans = _region_plans(ROWS, shapes, dt)
        row = [p for p in plans if isinstance(p, RowPlan)]
        assert len(row) == 1 and len(low.regions) == 1
        p = row[0]
        assert (p.TPR, p.U) == (tpr, u)
        assert p.vec8 == (shape[-1] % 8 == 0)
        assert len(nat.compile_cubin(p.source, (10, 0))) > 0


def test_rows_too_long_stay_unfused():
    with pytest.raises(Exception, match="exceeds the on-chip row"):
        _region_plans(ROWS, {"x": (2, 40000), "b": (40000,), "m": (2, 1)})


def test_non_innermost_dim_is_not_a_row_op():
    text = '''
import torch
def f(x):
    y = torch.softmax(x, dim=0) + 1
    return y
'''
    low, _ = lowering.lower(text)
    args = [torch.randn(4, 8)]
    r = low.regions[0] if low.regions else None
    if r is not None:
        with pytest.raises(Exception, match="innermost"):
            RowPlan(r.graph, r.out_nodes, args, allow_cpu=True)


def test_floordiv_mod_and_subscripts_fuse():
    text = '''
import torch
def f(x, b):
    y = x // 0.75 + x % 1.5 - torch.remainder(x, -2.0) + torch.fmod(x, 0.5)
    z = y * 2 + x[..., :16] - b[:16]
    return z
'''
    low, _ = lowering.lower(text)
    assert len(low.regions) == 1
    r = low.regions[0]
    assert sorted(fv.text for fv in r.graph.frees) == ["b[:16]", "x", "x[..., :16]"]
    ops = {n.op for n in r.graph.nodes}
    assert {"floordiv", "mod", "fmod"} <= ops
    x = torch.randn(4, 16)
    args = {"x": x, "x[..., :16]": torch.randn(4, 32)[..., :16], "b[:16]": torch.randn(32)[:16]}
    plan = codegen.Plan(r.graph, r.out_nodes, [args[fv.text] for fv in r.graph.frees], allow_cpu=True)
    assert any(ip.mode == codegen.MODE_STRIDED for ip in plan.inputs)
    assert len(nat.compile_cubin(plan.source, (10, 0))) > 0


def test_floordiv_mod_cpu_semantics_match_torch():
    """The device formulas (gm::floordiv / gm::pymod) restated in Python over
    float32 agree with torch's CPU `//` and `%` bit for bit, signs and zeros
    included."""
    import numpy as np

    def pymod(a, b):
        m = np.fmod(a, b)
        fix = (m != 0) & ((b < 0) != (m < 0))
        return np.where(fix, (m + b).astype(np.float32), m).astype(np.float32)

    def floordiv(a, b):
        with np.errstate(all="ignore"):
            m = np.fmod(a, b)
            d = ((a - m).astype(np.float32) / b).astype(np.float32)
            d = np.where((m != 0) & ((b < 0) != (m < 0)), (d - np.float32(1)).astype(np.float32), d)
            f = np.floor(d)
            f = np.where((d - f).astype(np.float32) > 0.5, (f + 1).astype(np.float32), f)
            z = np.copysign(np.float32(0), (a / b).astype(np.float32))
            r = np.where(d != 0, f, z).astype(np.float32)
            return np.where(b == 0, (a / b).astype(np.float32), r)

    torch.manual_seed(0)
    a = (torch.randn(20000) * 10).numpy().astype(np.float32)
    for bv in (0.75, -1.5, 3.0, -0.3):
        b = np.full_like(a, bv)
        ta, tb = torch.from_numpy(a), torch.from_numpy(b)
        assert np.array_equal(pymod(a, b), (ta % tb).numpy())
        assert np.array_equal(floordiv(a, b), (ta // tb).numpy())


def test_mixed_statement_stays_unfused():
    """`softmax(x).sum()` mixes a row operator with a grid reduction in ONE
    statement: it stays a PyTorch statement (no region), the rest fuses."""
    text = '''
import torch
def f(x):
    s = torch.softmax(x, -1).sum() > 0
    y = torch.where(s, x * 2, x)
    return y
'''
    low, _ = lowering.lower(text)
    assert "s = torch.softmax(x, -1).sum() > 0" in low.source
    assert all(not (ROW_OPS & {n.op for n in r.graph.nodes}) for r in low.regions)


def test_bigbird_attn_scores_are_rematerialised(programs):
    """workloads/bigbird_attn: `scores = QK^T / 8` feeds the predicate's grid
    reduction and both softmax arms.  It is recomputed in the grid region and
    the row region instead of being written and read back: the [8,12,1024,1024]
    intermediate never exists."""
    low, _ = lowering.lower(programs["bigbird_attn"]["transformed"])
    fwd = [r for r in low.regions if r.name.startswith("forward")]
    grid, rows = fwd[0], fwd[1]
    assert grid.out_names[-1] == "__gm_pred_0" and "scores" not in grid.out_names
    assert has_row_ops(rows.out_nodes) and rows.out_names == ["probs"]
    assert "/ 8.0" in rows.source and "/ 8.0" in grid.source


def test_mixed_shapes_split_into_side_kernels():
    """A run over two iteration spaces (a predicate over a [C] bias guarding
    full arms, a [C]-shaped live-out, a softmax over the bias): the main
    kernel covers the full shape, each other-shaped reduction / output / row
    operator is a side kernel that runs first (split.py)."""
    from paper_2509_16248_b200.split import is_mixed, split

    text = '''
import torch
def f(x, b):
    __gm_pred_0 = b.sum() > 0
    __gm_then_y_0 = x * 2 + b
    y = torch.where(__gm_pred_0, __gm_then_y_0, x)
    c = torch.softmax(b, -1) * 3
    z = y * x.mean()
    return y, c, z
'''
    low, _ = lowering.lower(text)
    # grid run (the predicated block), row run (the softmax), grid run (z)
    assert len(low.regions) == 3
    r = low.regions[0]
    args = {"x": torch.randn(4, 8, 16), "b": torch.randn(16)}
    a = [args[fv.text] for fv in r.graph.frees]
    assert is_mixed(r.graph, r.out_nodes, a)
    steps, (mg, mouts) = split(r.graph, r.out_nodes, a)
    # the [C] bias sum is a side kernel; the main kernel writes y over [4, 8, 16]
    assert [s[1][0].op for s in steps] == ["sum"]
    ext = list(a)
    for sg, souts, idx in steps:
        assert not is_mixed(sg, souts, ext)
        ext.append(torch.empty(tuple(souts[0].shape), dtype=souts[0].dtype))
    assert not is_mixed(mg, mouts, ext)
    p = codegen.Plan(mg, mouts, ext, allow_cpu=True)
    assert len(nat.compile_cubin(p.source, (10, 0))) > 0


@pytest.mark.parametrize("persist", ["0", "1"])
def test_persistent_row_kernels_compile(monkeypatch, persist):
    """Row kernels as persistent CTAs walking row groups, with an L2
    prefetch of each CTA's next group (GM_ROW_PERSIST=1), compile for
    sm_100a; the loop uses gridDim.x, so any clamped grid covers all rows."""
    monkeypatch.setenv("GM_ROW_PERSIST", persist)
    shapes = {"x": (64, 1024), "b": (1024,), "m": (64, 1)}
    for dt in (torch.float32, torch.bfloat16):
        _, plans = _region_plans(ROWS, shapes, dt)
        row = [p for p in plans if isinstance(p, RowPlan)][0]
        assert row.persist == (persist == "1")
        assert ("for (i64 g_ = blockIdx.x;" in row.source) == row.persist
        assert ("prefetch.global.L2" in row.source) == row.persist
        assert len(nat.compile_cubin(row.source, (10, 0))) > 0


def test_layer_norm_weights_staged_in_shared_memory(monkeypatch):
    """LayerNorm's [C] weight and bias are copied into shared memory by
    cp.async at kernel start and read back after the row statistics; a
    [C] input another operator reads stays a global load; the opt-out
    (GM_ROW_NO_SMEM_WB) restores global loads.  Both forms compile."""
    text = '''
import torch
def f(x, r, w, b, s):
    y = torch.nn.functional.layer_norm(x + r, (768,), w, b, 1e-12) * s
    return y
'''
    shapes = {"x": (64, 768), "r": (64, 768), "w": (768,), "b": (768,), "s": (768,)}
    for opt_out in (False, True):
        if opt_out:
            monkeypatch.setenv("GM_ROW_NO_SMEM_WB", "1")
        for dt in (torch.float32, torch.bfloat16):
            _, plans = _region_plans(text, shapes, dt)
            row = [p for p in plans if isinstance(p, RowPlan)][0]
            src = row.source
            assert ("cp_async16" in src) != opt_out
            assert src.count("__shared__ __align__(16) unsigned char swb") == (0 if opt_out else 2)
            assert len(nat.compile_cubin(src, (10, 0))) > 0

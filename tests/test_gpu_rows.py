"""Row regions and the rest of the purity gate's vocabulary on the B200,
against the CPU eager execution of the same transformed text (the oracle):
softmax / log_softmax arms behind a grid-reduced predicate, sum/mean/amax/
amin over the innermost dim (keepdim and not), broadcast inputs ([C] bias,
[..., 1] per-row values, 0-d tensors), ragged row lengths (C % 8 != 0, C = 1,
long rows spread over 1024 threads), `//` and `%`, and subscripted views.

Tolerance: tests/parity.py (1e-5 relative / 1e-6 absolute fp32, 1e-2 / one
ulp bf16).  Row sums have an unspecified accumulation order on both sides,
so — as for GEMMs — the absolute floor may grow to twice stock PyTorch
CUDA's own deviation from the CPU result on the same program."""

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import compile_program, harness
from paper_2509_16248_b200.rowgen import RowPlan
from parity import assert_parity, rowop_fp64_reference, torch_cuda_reference

SOFTMAX_ARM = '''
import torch
def f(x, b):
    __gm_pred_0 = x.sum() > 0
    __gm_then_y_0 = torch.softmax(x * 0.125 + b, dim=-1)
    __gm_else_y_0 = torch.log_softmax(x, -1)
    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
    return y
'''

ROWS = '''
import torch
def f(x, b, m):
    mx = x.amax(-1, keepdim=True)
    e = (x - mx).exp()
    p = e / e.sum(-1, keepdim=True)
    q = torch.log_softmax(x + b, -1) * m + x.amin(-1, keepdim=True)
    r = x.mean(-1)
    return p + q, r
'''

ATTN_LIKE = '''
import torch
def f(scores, band):
    __gm_pred_0 = scores.abs().mean() > 0.5
    __gm_then_probs_0 = torch.softmax(scores + band, dim=-1)
    __gm_else_probs_0 = torch.softmax(scores, dim=-1)
    probs = torch.where(__gm_pred_0, __gm_then_probs_0, __gm_else_probs_0)
    return probs
'''

VOCAB = '''
import torch
def f(x, b):
    __gm_pred_0 = x.mean() > 0
    __gm_then_y_0 = x // 0.75 + x % 1.5 - torch.remainder(x, -2.0)
    __gm_else_y_0 = torch.fmod(x, 0.5) * 2
    y = torch.where(__gm_pred_0, __gm_then_y_0, __gm_else_y_0)
    z = y * 2 + x[..., :1] - b[:48]
    return z
'''


def _run(text, args, dtype, expect_row=True):
    ref, _ = orc.call_captured(orc.reference_callable(text, "f"), list(args))
    noise = torch_cuda_reference(text, "f", list(args))
    noise64 = rowop_fp64_reference(text, "f", list(args))
    ex, mod, low = compile_program(text, "f")
    out, _ = harness.call_captured(ex, [a.cuda() for a in args])
    torch.cuda.synchronize()
    info = ex.info()[0]
    assert info.mode == "graph" and info.host_syncs == 0, info
    for r in low.regions:
        assert r.stats.fallbacks == 0 and r.stats.launches >= 1, (r.name, r.stats)
    rows = [r for r in low.regions if r.last_spec is not None and isinstance(r.last_spec.plan, RowPlan)]
    if expect_row is not None:
        assert bool(rows) == expect_row
    outs = out if isinstance(out, tuple) else (out,)
    refs = ref if isinstance(ref, tuple) else (ref,)
    nz = noise if isinstance(noise, tuple) else (noise,)
    nz64 = noise64 if isinstance(noise64, tuple) else (noise64,)
    for o, r, n, n64 in zip(outs, refs, nz, nz64):
        assert_parity(o, r, dtype, what=f"{text.split(chr(10))[2]} {tuple(r.shape)}", noise=[n, n64])
    return low


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(8, 1024, 768), (4, 7, 20), (3, 5000), (2, 3, 1), (2, 20000)],
                         ids=["bigbird", "ragged", "long_row", "c1", "tpr1024"])
@pytest.mark.parametrize("sign", [1.0, -1.0], ids=["then", "else"])
def test_softmax_arm(shape, dtype, sign):
    torch.manual_seed(3)
    x = (torch.randn(shape) + sign * 0.5).to(dtype)
    b = torch.randn(shape[-1]).to(dtype)
    low = _run(SOFTMAX_ARM, [x, b], dtype)
    assert len(low.regions) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(8, 1024, 768), (4, 7, 20), (6, 4096), (2, 3, 1)],
                         ids=["bigbird", "ragged", "tpr128", "c1"])
def test_row_reductions(shape, dtype):
    torch.manual_seed(4)
    x = torch.randn(shape).to(dtype)
    b = torch.randn(shape[-1]).to(dtype)
    m = torch.rand(shape[:-1] + (1,)).to(dtype)
    _run(ROWS, [x, b, m], dtype)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("scale", [1.0, 0.1], ids=["band", "full"])
def test_attention_scores_softmax(dtype, scale):
    """[B, heads, L, L] scores with an [L, L] additive band mask (periodic
    input), the BigBird block-sparse / full choice."""
    torch.manual_seed(5)
    L = 512
    scores = (torch.randn(2, 12, L, L) * scale).to(dtype)
    i = torch.arange(L)
    band = torch.where((i[:, None] // 64 - i[None, :] // 64).abs() <= 1, 0.0, -1e4).to(dtype)
    _run(ATTN_LIKE, [scores, band], dtype)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("sign", [1.0, -1.0], ids=["then", "else"])
def test_floordiv_mod_subscripts(dtype, sign):
    torch.manual_seed(6)
    x = ((torch.randn(64, 48) + sign) * 4).to(dtype)
    b = torch.randn(64).to(dtype)
    _run(VOCAB, [x, b], dtype, expect_row=False)


MIXED = '''
import torch
def f(x, b):
    __gm_pred_0 = b.sum() > 0
    __gm_then_y_0 = x * 2 + b
    y = torch.where(__gm_pred_0, __gm_then_y_0, x)
    c = torch.softmax(b, -1) * 3
    z = y * x.mean() + c
    return z, c
'''


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(8, 1024, 768), (4, 7, 20)], ids=["bigbird", "ragged"])
def test_mixed_shapes(shape, dtype):
    """One run over a [C] bias and the full activations: side kernels first
    (the bias predicate, the [C] softmax), then the main kernel."""
    torch.manual_seed(7)
    for sign in (1.0, -1.0):
        x = torch.randn(shape).to(dtype)
        b = (torch.rand(shape[-1]) * sign).to(dtype)
        _run(MIXED, [x, b], dtype, expect_row=None)


LAYER = '''
import torch
import torch.nn.functional as F
def f(x, w, b):
    h = F.gelu(x) + torch.erf(x) * 0.5 + F.gelu(x, approximate="tanh")
    y = F.layer_norm(h, (x.shape[-1],), w, b, 1e-12)
    z = y + x.var(-1, keepdim=True) - x.std(-1, unbiased=False, keepdim=True)
    return z
'''


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(8, 1024, 768), (4, 7, 20)], ids=["bigbird", "ragged"])
def test_layer_norm_gelu_var(shape, dtype):
    """GELU (erf and tanh forms), erf, layer_norm with weight and bias, var
    and std over the innermost dim — one row kernel."""
    torch.manual_seed(8)
    x = torch.randn(shape).to(dtype)
    w = torch.randn(shape[-1]).to(dtype)
    b = torch.randn(shape[-1]).to(dtype)
    low = _run(LAYER, [x, w, b], dtype)
    assert len(low.regions) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
def test_layernorm_module_is_a_row_region(dtype):
    """`self.ln(x)` with an nn.LayerNorm runs the fused row kernel (gemm.module_call)."""
    from paper_2509_16248_b200 import gemm

    torch.manual_seed(9)
    ln = torch.nn.LayerNorm(768, eps=1e-12).to(dtype)
    with torch.no_grad():
        ln.weight.normal_()
        ln.bias.normal_()
    x = torch.randn(8, 1024, 768).to(dtype)
    with torch.no_grad():
        ref = ln(x)
    lnc = ln.cuda()
    with torch.no_grad():
        y = gemm.module_call(lnc, x.cuda())
    regions = gemm.module_regions(lnc)
    assert len(regions) == 1 and regions[0].stats.launches == 1 and regions[0].last_spec is not None
    assert regions[0].name.startswith("nn.LayerNorm")
    # noise yardstick: the same layer norm evaluated in fp64 and rounded
    n64 = torch.nn.functional.layer_norm(x.double(), (768,), ln.weight.double().cpu(), ln.bias.double().cpu(),
                                         1e-12).to(dtype)
    assert_parity(y, ref, dtype, what="nn.LayerNorm", noise=n64)

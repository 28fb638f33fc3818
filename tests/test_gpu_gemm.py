"""Dense contractions on the B200 path (csrc/gm_gemm.cu, gemm.py): fp32 on
cuBLASLt 12.9's BF16x9 emulation must be at least as close to the exact
product as the SIMT SGEMM stock PyTorch runs (TF32 off), and the
GEMM-bearing predicated block must run ONE GEMM whose
result equals the selected arm's GEMM bit for bit."""

import ctypes

import pytest
import torch

from paper_2509_16248_b200 import _native as nat
from paper_2509_16248_b200 import gemm


def _errs(y, ref64):
    d = (y.double().cpu() - ref64).abs()
    return float(d.max()), float((d / (ref64.abs() + 0.1)).max())


@pytest.mark.gpu
@pytest.mark.parametrize("shape,relu,bias", [((8, 1024, 768), False, True), ((8192, 768), True, True),
                                             ((32, 1, 768), False, True), ((1000, 3072), False, False)],
                         ids=["bigbird", "relu", "gen_step", "nobias_odd_M"])
def test_linear_fp32_accuracy_vs_sgemm(shape, relu, bias):
    torch.manual_seed(0)
    K = shape[-1]
    N = 768 if K != 768 else 3072
    x = torch.randn(shape)
    w = torch.randn(N, K) * K ** -0.5
    b = torch.randn(N) * 0.1 if bias else None
    ref64 = torch.nn.functional.linear(x.double(), w.double(), None if b is None else b.double())
    if relu:
        ref64 = ref64.relu()
    torch.backends.cuda.matmul.allow_tf32 = False
    xc, wc, bc = x.cuda(), w.cuda(), None if b is None else b.cuda()
    c0 = gemm.stats["gm_gemm"]
    y = gemm.linear(xc, wc, bc, relu=relu)
    assert gemm.stats["gm_gemm"] == c0 + 1, "the BF16x9 path did not run"
    sg = torch.nn.functional.linear(xc, wc, bc)
    if relu:
        sg = sg.relu()
    cpu = torch.nn.functional.linear(x, w, b)
    if relu:
        cpu = cpu.relu()
    e_gm, s_gm = _errs(y, ref64)
    e_sg, s_sg = _errs(sg, ref64)
    e_cpu, _ = _errs(cpu, ref64)
    # at least as close to the exact product as torch's own SGEMM (and CPU)
    assert e_gm <= 1.5 * max(e_sg, e_cpu) + 1e-7, (e_gm, e_sg, e_cpu)
    # scaled error: within 1e-5 or no worse than SGEMM / CPU on the same data
    assert s_gm <= max(1e-5, 1.5 * max(s_sg, _errs(cpu, ref64)[1])), (s_gm, s_sg)
    print(f"max abs err vs fp64: BF16x9 {e_gm:.3e}  SGEMM {e_sg:.3e}  CPU {e_cpu:.3e}")


@pytest.mark.gpu
def test_matmul_fp32_and_torch_cublas_still_works():
    """gemm.matmul on the private cuBLASLt 12.9 next to torch's own cuBLAS
    12.8 in the same process: both keep working."""
    torch.manual_seed(1)
    a = torch.randn(4, 2048, 768, device="cuda")
    b = torch.randn(768, 640, device="cuda") / 28
    y = gemm.matmul(a, b)
    ref64 = (a.double() @ b.double()).cpu()
    assert _errs(y, ref64)[1] <= 1e-5
    z = a @ b                     # torch's cuBLAS
    assert _errs(z, ref64)[1] <= 1e-4
    h = (a.bfloat16() @ b.bfloat16()).float()
    assert torch.isfinite(h).all()
    assert nat.lib().gm_gemm_version() >= 120900


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["matmul", "linear"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
def test_select_gemm_runs_one_gemm(kind, dtype):
    torch.manual_seed(2)
    x = torch.randn(8, 1024, 768, device="cuda", dtype=dtype)
    if kind == "matmul":
        t_ops = (x, (torch.randn(768, 768, device="cuda") / 28).to(dtype))
        e_ops = (x, (torch.randn(768, 768, device="cuda") / 28).to(dtype))
        f = gemm.matmul
    else:
        t_ops = (x, (torch.randn(768, 768, device="cuda") / 28).to(dtype), torch.randn(768, device="cuda").to(dtype))
        e_ops = (x, (torch.randn(768, 768, device="cuda") / 28).to(dtype), torch.randn(768, device="cuda").to(dtype))
        f = gemm.linear
    for p in (True, False):
        pred = torch.tensor(p, device="cuda")
        s0, g0 = gemm.stats["select_gemm"], gemm.stats["gm_gemm"] + gemm.stats["torch_gemm"]
        y = gemm.select_gemm(pred, kind, t_ops, e_ops)
        assert gemm.stats["select_gemm"] == s0 + 1
        assert gemm.stats["gm_gemm"] + gemm.stats["torch_gemm"] == g0 + 1   # ONE contraction
        want = f(*(t_ops if p else e_ops))
        assert torch.equal(y, want), p


@pytest.mark.gpu
def test_select_gemm_under_graph_capture():
    """The operand select reads the predicate on the device: one captured
    graph serves both decisions."""
    torch.manual_seed(3)
    x = torch.randn(2048, 768, device="cuda")
    wa, wb = torch.randn(768, 768, device="cuda") / 28, torch.randn(768, 768, device="cuda") / 28
    pred = torch.tensor(True, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    from paper_2509_16248_b200.region import scratch_owner

    owner = object()
    with torch.cuda.stream(s), scratch_owner(owner):
        gemm.select_gemm(pred, "matmul", (x, wa), (x, wb))
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g), scratch_owner(owner):
        y = gemm.select_gemm(pred, "matmul", (x, wa), (x, wb))
    for p in (True, False, True):
        pred.fill_(p)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, gemm.matmul(x, wa if p else wb)), p

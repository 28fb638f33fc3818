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


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["qk", "pv", "contig", "odd"])
def test_batched_matmul_fp32(case):
    """Attention-shaped batched contractions (gm_gemm_run_batched, BF16x9):
    scores = q @ k^T with head-split (non-viewable) operands, ctx = p @ v,
    plain contiguous batches and odd sizes — at least as close to the fp64
    product as torch's SIMT SGEMM."""
    torch.manual_seed(0)
    b, h, n, d = 2, 12, 256, 64
    if case == "qk":
        x = torch.randn(b, n, h, d).transpose(1, 2)
        k = torch.randn(b, n, h, d).transpose(1, 2)
        A, B = x, k.transpose(-1, -2)
    elif case == "pv":
        A = torch.softmax(torch.randn(b, h, n, n), -1)
        B = torch.randn(b, n, h, d).transpose(1, 2)
    elif case == "contig":
        A, B = torch.randn(6, 100, 48), torch.randn(6, 48, 72)
    else:
        A, B = torch.randn(3, 5, 17, 33), torch.randn(3, 5, 33, 9)
    ref64 = torch.matmul(A.double(), B.double())
    torch.backends.cuda.matmul.allow_tf32 = False
    c0 = gemm.stats["gm_gemm"]
    y = gemm.matmul(A.cuda(), B.cuda())
    assert gemm.stats["gm_gemm"] == c0 + 1, "the batched BF16x9 path did not run"
    assert y.shape == ref64.shape and y.dtype == torch.float32
    sg = torch.matmul(A.cuda(), B.cuda())
    e_gm, _ = _errs(y, ref64)
    e_sg, _ = _errs(sg, ref64)
    assert e_gm <= 1.5 * e_sg + 1e-6, (e_gm, e_sg)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16], ids=["fp32", "bf16", "fp16"])
def test_copy_strided_is_contiguous(dtype):
    """gm_copy_strided (the head split / merge gather) equals torch's
    .contiguous() bit for bit; layouts it cannot take fall back to torch."""
    torch.manual_seed(0)
    x = torch.randn(2, 256, 12, 64).to(dtype).cuda()
    for view in (x.transpose(1, 2), x.permute(2, 0, 1, 3), x[:, ::2].transpose(1, 2), x.transpose(1, 2)[..., :32]):
        c0 = gemm.stats["gm_copy"]
        y = gemm.contiguous(view)
        assert torch.equal(y, view.contiguous()) and y.is_contiguous()
        assert gemm.stats["gm_copy"] == c0 + 1
    odd = x.transpose(-1, -2)                     # innermost dim strided: torch's copy
    c0 = gemm.stats["gm_copy"]
    assert torch.equal(gemm.contiguous(odd), odd.contiguous()) and gemm.stats["gm_copy"] == c0


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16], ids=["bf16", "fp16"])
def test_batched_matmul_half(dtype):
    """bf16 / fp16 attention contractions through gm_gemm_run_batched: as
    close to the fp64 product as torch's own cuBLAS call."""
    torch.manual_seed(1)
    b, h, n, d = 2, 12, 256, 64
    q = torch.randn(b, n, h, d).transpose(1, 2).to(dtype)
    k = torch.randn(b, n, h, d).transpose(1, 2).to(dtype)
    ref64 = torch.matmul(q.double(), k.double().transpose(-1, -2))
    c0 = gemm.stats["gm_gemm"]
    y = gemm.matmul(q.cuda(), k.cuda().transpose(-1, -2))
    assert gemm.stats["gm_gemm"] == c0 + 1 and y.dtype == dtype
    t = torch.matmul(q.cuda(), k.cuda().transpose(-1, -2))
    e_gm, _ = _errs(y, ref64)
    e_t, _ = _errs(t, ref64)
    assert e_gm <= 1.5 * e_t + 1e-6, (e_gm, e_t)

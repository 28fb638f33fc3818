"""Precompiled sm_100a kernels of libgm_b200.so, called through the C ABI."""

import math
import ctypes

import pytest
import torch

from paper_2509_16248_b200 import _native as nat

RED = {0: "sum", 1: "mean", 2: "max", 3: "min", 4: "norm"}
CMP = {0: ">", 1: ">=", 2: "<", 3: "<="}


def _stat_ref(x: torch.Tensor, red: int) -> torch.Tensor:
    return {0: x.sum, 1: x.mean, 2: x.max, 3: x.min, 4: x.norm}[red]()


@pytest.mark.gpu
@pytest.mark.parametrize("n", [64, 1000003, 8 * 1024 * 768, 4 * 4096 * 768])
@pytest.mark.parametrize("red", [0, 1, 2, 3, 4])
def test_branch_select_f32(n, red):
    """gm_branch_select_f32 == the transformed phi4 block executed by torch on
    CPU: pred = x.<red>() > thr; out = where(pred, x*a1 + b1, x*a2 + b2)
    (corpus/phi4_like/original.py:8-11 after transform.py:359-376)."""
    lib = nat.lib()
    nat.init(torch.cuda.current_device())
    torch.manual_seed(n + red)
    x = torch.randn(n) + 0.01
    stat = _stat_ref(x, red)
    xd = x.cuda()
    out = torch.empty_like(xd)
    scratch = torch.zeros(lib.gm_branch_select_scratch_bytes(), dtype=torch.uint8, device="cuda")
    stat_out = torch.zeros(2, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for thr, cmp in ((float(stat) * 0.5 - 1.0, 0), (float(stat) * 1.5 + 1.0, 0), (float(stat) - 1.0, 2)):
        nat.check(lib.gm_branch_select_f32(ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(out.data_ptr()), n,
                                           red, cmp, thr, 2.0, 1.0, 0.5, -1.0,
                                           ctypes.c_void_p(scratch.data_ptr()),
                                           ctypes.c_void_p(stat_out.data_ptr()), ctypes.c_void_p(stream)))
        torch.cuda.synchronize()
        assert int(scratch[16:20].view(torch.int32).item()) == 0, "grid barrier timed out"
        s = stat_out.cpu()
        # fp64 grid combine: the statistic is the correctly rounded fp32 value
        # (torch's CPU fp32 norm accumulates in fp32 and drifts ~2e-4 relative
        # at 6M elements, so against torch the bound is looser for norm)
        exact = {0: x.double().sum, 1: x.double().mean, 2: x.double().max, 3: x.double().min,
                 4: x.double().norm}[red]()
        assert abs(float(s[0]) - float(exact)) <= 2e-6 * abs(float(exact)) + 1e-6
        torch.testing.assert_close(torch.tensor(float(s[0]), dtype=torch.float32), stat,
                                   rtol=1e-3 if red == 4 else 2e-5, atol=1e-4)
        pred_ref = bool(stat > thr) if cmp == 0 else bool(stat < thr)
        assert bool(s[1] != 0) == pred_ref
        ref = torch.where(torch.tensor(pred_ref), x * 2.0 + 1.0, x * 0.5 + -1.0)
        assert torch.equal(out.cpu(), ref), "affine arm must be bit-exact"


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32], ids=["bf16", "f16", "fp32"])
@pytest.mark.parametrize("n", [1, 7, 8, 4099, 8 * 1024 * 768])
def test_unique_sum_matches_torch(n, dtype):
    """gm_unique_sum16 (presence bitmap, one pass) / gm_unique_sum32 (radix
    sort + one pass over the runs) == torch's x.unique().sum() on CPU — the
    moe_minicpm_like rewrite of `unique(x).sum()`; ragged
    sizes hit the tail path, and -0.0 / +0.0 count once as in torch.unique."""
    from paper_2509_16248_b200.logring import ModuleRuntime

    torch.manual_seed(n)
    x = (torch.softmax(torch.randn(n), 0) * 3 - 1e-3).to(dtype)
    if n > 2:
        x[0], x[1] = 0.0, -0.0
    ref = x.unique().sum()
    xd = x.cuda()
    out = ModuleRuntime.unique_sum(xd)
    assert out.dtype == dtype and out.shape == ()
    r, o = float(ref), float(out.cpu())
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    assert abs(o - r) <= tol * abs(r) + 1e-6, (o, r)


def _exact_f32_sum_of_unique(x: torch.Tensor) -> float:
    """Correctly rounded (nearest-even) fp32 value of the EXACT sum of the
    distinct finite values of x (every fp32 is an integer multiple of
    2^-149, so the sum is an integer S times 2^-149)."""
    import numpy as np

    vals = set(float(v) for v in x.numpy().astype(np.float64))
    vals = {0.0 if v == 0 else v for v in vals}
    S = sum(int(math.ldexp(v, 149)) for v in vals)
    mag = abs(S)
    if mag < 2 ** 23:
        r = math.ldexp(mag, -149)
    else:
        shift = mag.bit_length() - 24
        m, rem = mag >> shift, mag & ((1 << shift) - 1)
        half = 1 << (shift - 1) if shift > 0 else 0
        if shift > 0 and (rem > half or (rem == half and m & 1)):
            m += 1
        r = math.ldexp(m, shift - 149)
        if r >= 2.0 ** 128:
            r = math.inf
    return float(np.float32(-r if S < 0 else r))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["softmax", "dups", "cancel", "subnormal", "wide", "ragged"])
def test_unique_sum32_hash_is_correctly_rounded(case):
    """gm_unique_sum32_hash: the distinct values' exact sum rounded once —
    bit-identical to a Python big-integer restatement, on every call,
    whatever the duplicate pattern or magnitude spread (softmax/dups/
    subnormal stay inside the 16-binade bitmap window; cancel/wide exercise
    the hash set)."""
    from paper_2509_16248_b200.logring import ModuleRuntime

    g = torch.Generator().manual_seed(7)
    n = 1 << 20
    if case == "softmax":
        x = torch.softmax(torch.randn(n, generator=g), 0) * 3 - 1e-3
    elif case == "dups":
        x = torch.randint(-500, 500, (n,), generator=g).float() / 8
    elif case == "cancel":
        x = torch.tensor([1e30, -1e30, 1.0, 3e-45, 2.0 ** -126] * 1000)
    elif case == "subnormal":
        x = torch.randint(-4000, 4000, (n,), generator=g).float() * 2.0 ** -149
    elif case == "wide":
        x = torch.randn(n, generator=g) * torch.exp2(torch.randint(-120, 120, (n,), generator=g).float())
    else:
        x = torch.randn(4099, generator=g)
    x = x.float().contiguous()
    # repeated calls share the tagged table and the (self-clearing) bitmap:
    # a changed input must not see the previous call's values
    for xi in (x, x.flip(0).contiguous(), x * 0.75, x[: x.numel() // 3 + 1].contiguous()):
        expect = _exact_f32_sum_of_unique(xi)
        got = float(ModuleRuntime.unique_sum(xi.cuda()).cpu())
        assert got == expect or (math.isnan(got) and math.isnan(expect)), (got, expect)


@pytest.mark.gpu
@pytest.mark.parametrize("specials,expect", [([math.nan], math.nan), ([math.inf], math.inf),
                                             ([-math.inf], -math.inf), ([math.inf, -math.inf], math.nan),
                                             ([math.inf, math.nan], math.nan)])
def test_unique_sum32_hash_specials(specials, expect):
    from paper_2509_16248_b200.logring import ModuleRuntime

    x = torch.randn(10000)
    x[torch.arange(len(specials)) * 37] = torch.tensor(specials)
    got = float(ModuleRuntime.unique_sum(x.cuda()).cpu())
    ref = float(x.unique().sum())
    assert (math.isnan(got) and math.isnan(expect) and math.isnan(ref)) or got == expect == ref

"""Shared parity helpers for the GPU tests (B200 path vs the CPU oracle)."""

import torch

# north_star: outputs within 1e-5 relative (fp32) or 1e-2 (bf16) of the
# reference's eager CPU execution of the same transformed program.  The bound
# is |out - ref| <= tol * (|ref| + 0.1 * max|ref|): relative per element, with
# a floor for elements produced by cancellation (e.g. x*sigmoid(x) + mask
# near 0), where 1-ulp differences between torch's SLEEF transcendentals and
# CUDA's make a per-element relative error meaningless.
TOL = {torch.float32: 1e-5, torch.bfloat16: 1e-2, torch.float16: 1e-2}


def assert_parity(out: torch.Tensor, ref: torch.Tensor, dtype=torch.float32, what: str = ""):
    out = out.detach().to("cpu")
    ref = ref.detach().to("cpu")
    assert out.shape == ref.shape, (what, out.shape, ref.shape)
    assert out.dtype == ref.dtype, (what, out.dtype, ref.dtype)
    if not ref.dtype.is_floating_point:
        assert torch.equal(out, ref), what
        return
    tol = TOL[dtype]
    o, r = out.double(), ref.double()
    floor = 0.1 * float(r.abs().max()) if r.numel() else 0.0
    bad = (o - r).abs() > tol * (r.abs() + floor)
    if dtype in (torch.bfloat16, torch.float16):
        # two roundings apart (e.g. a bf16 GEMM output re-rounded by the next
        # op): allow 2 ulp of the reference value in the storage type
        mant = 7 if dtype == torch.bfloat16 else 10
        ulp = torch.exp2(torch.floor(torch.log2(r.abs().clamp_min(1e-30))) - mant)
        bad &= (o - r).abs() > 2 * ulp
    nan_ok = torch.isnan(o) == torch.isnan(r)
    assert bool(nan_ok.all()), f"{what}: NaN pattern differs"
    bad &= ~torch.isnan(r)
    if bool(bad.any()):
        i = int(bad.reshape(-1).nonzero()[0])
        raise AssertionError(
            f"{what}: {int(bad.sum())} of {r.numel()} elements out of tolerance {tol}; "
            f"first at flat index {i}: out={o.reshape(-1)[i].item()!r} ref={r.reshape(-1)[i].item()!r}"
        )

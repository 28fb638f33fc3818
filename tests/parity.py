"""Shared parity helpers for the GPU tests (B200 path vs the CPU oracle).

Output bound (north_star: 1e-5 relative fp32, 1e-2 bf16), in the reference
harness's own form (runner.py:160-168, :203-215, FLOAT_RTOL 1e-6 /
FLOAT_ATOL 1e-7, scaled by the north_star's 10x):

  * fp32: an element fails only if |out - ref| > 1e-5 * |ref| AND
    |out - ref| > 1e-6;
  * bf16 / fp16: only if |out - ref| > 1e-2 * |ref| AND |out - ref| > one ulp
    of ref in the storage type.

Programs with dense contractions (Linear / matmul on cuBLAS) get ONE more
term, measured rather than assumed: the accumulation order of a GEMM is
unspecified on both sides (MKL on the CPU, cuBLAS here), so the absolute
floor becomes max(floor, 2 * max|torch_cuda - ref|), where torch_cuda is
stock PyTorch's own eager CUDA execution of the same transformed program
(TF32 off).  Programs with softmax get the same term from the oracle run
with fp64 softmaxes (`rowop_fp64_reference`): a program that thresholds or
deduplicates softmax outputs moves under any last-bit change of them.  I.e. the B200 path may deviate from the CPU oracle by at most
twice what PyTorch's own GPU execution of the same text deviates.  The
harness's max-based form (max rel and max abs over the tensor) is reported
in every failure message.

`check_scalars` compares every region's predicate statistics and branch
decisions with the oracle's (the same DAG evaluated with torch's CPU
operators, ir.evaluate) and records |stat - threshold| margins.
"""

from __future__ import annotations

import contextlib
import io
import json
import logging
import os

import torch

TOL = {torch.float32: 1e-5, torch.bfloat16: 1e-2, torch.float16: 1e-2}
FLOOR_F32 = 1e-6
MANT = {torch.bfloat16: 7, torch.float16: 10}

MARGINS: list[dict] = []   # decision margins logged by check_scalars (dumped by conftest)


def harness_diffs(out: torch.Tensor, ref: torch.Tensor) -> tuple[float, float]:
    """runner.py:160-168 `_diffs`: (max abs diff, max rel diff) in fp64."""
    fa, fb = ref.double(), out.double()
    d = (fa - fb).abs()
    if not d.numel():
        return 0.0, 0.0
    return float(d.max()), float((d / fa.abs().clamp_min(1e-12)).max())


def ulp(r: torch.Tensor, dtype) -> torch.Tensor:
    mant = MANT.get(dtype, 23)
    return torch.exp2(torch.floor(torch.log2(r.abs().clamp_min(1e-30))) - mant)


def assert_parity(out: torch.Tensor, ref: torch.Tensor, dtype=torch.float32, what: str = "",
                  noise=None):
    """`noise`: stock PyTorch's CUDA output of the same program (programs
    with dense contractions) and / or the fp64-row-operator oracle
    (`rowop_fp64_reference`, programs with softmax), a tensor or a list;
    see the module docstring."""
    out = out.detach().to("cpu")
    ref = ref.detach().to("cpu")
    assert out.shape == ref.shape, (what, out.shape, ref.shape)
    assert out.dtype == ref.dtype, (what, out.dtype, ref.dtype)
    if not ref.dtype.is_floating_point:
        assert torch.equal(out, ref), what
        return
    tol = TOL[dtype]
    o, r = out.double(), ref.double()
    if dtype == torch.float32:
        floor = torch.full_like(r, FLOOR_F32)
    else:
        floor = ulp(r, dtype)
    gemm_floor = 0.0
    for nz in ([] if noise is None else (noise if isinstance(noise, (list, tuple)) else [noise])):
        if nz is None:
            continue
        n = nz.detach().to("cpu").double()
        finite = torch.isfinite(n) & torch.isfinite(r)
        if bool(finite.any()):
            gemm_floor = max(gemm_floor, 2.0 * float((n - r).abs()[finite].max()))
    if gemm_floor:
        floor = floor.clamp_min(gemm_floor)
    d = (o - r).abs()
    bad = (d > tol * r.abs()) & (d > floor)
    nan_ok = torch.isnan(o) == torch.isnan(r)
    assert bool(nan_ok.all()), f"{what}: NaN pattern differs"
    inf_ok = torch.where(torch.isinf(r), o == r, torch.ones_like(r, dtype=torch.bool))
    assert bool(inf_ok.all()), f"{what}: inf pattern differs"
    bad &= torch.isfinite(r)
    if bool(bad.any()):
        i = int(bad.reshape(-1).nonzero()[0])
        mabs, mrel = harness_diffs(out[torch.isfinite(ref)], ref[torch.isfinite(ref)])
        raise AssertionError(
            f"{what}: {int(bad.sum())} of {r.numel()} elements out of tolerance rel {tol} "
            f"(abs floor {'1e-6' if dtype == torch.float32 else '1 ulp'}, GEMM floor {gemm_floor:.3e}); "
            f"first at flat index {i}: out={o.reshape(-1)[i].item()!r} ref={r.reshape(-1)[i].item()!r}; "
            f"harness form: max abs {mabs:.3e}, max rel {mrel:.3e}"
        )


def torch_cuda_reference(text: str, callable_name: str, args: list, dtype=None):
    """Stock PyTorch eager CUDA execution of the transformed program (no
    repo kernels; TF32 off): the GEMM-noise yardstick of assert_parity."""
    from oracle import executor as orc

    prev = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    try:
        fn = orc.reference_callable(text, callable_name, dtype)
        if isinstance(fn, torch.nn.Module):
            fn = fn.to("cuda")
        logging.disable(logging.CRITICAL)
        try:
            with torch.no_grad(), contextlib.redirect_stdout(io.StringIO()):
                out = fn(*[a.cuda() if torch.is_tensor(a) else a for a in args])
        finally:
            logging.disable(logging.NOTSET)
        return out.cpu() if torch.is_tensor(out) else out
    finally:
        torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = prev


def has_row_reduction(text: str) -> bool:
    """softmax / log_softmax in the program: a row reduction whose
    accumulation order (and exp implementation) is unspecified."""
    return "softmax(" in text


def rowop_fp64_reference(text: str, callable_name: str, args: list, dtype=None):
    """The oracle (CPU eager) with every softmax / log_softmax evaluated in
    fp64 and rounded to its dtype — an implementation at least as accurate as
    torch's.  Its deviation from the fp32 oracle measures how far the
    program's output moves under last-bit changes of those row operators
    (moe_minicpm_like thresholds and deduplicates softmax outputs: this
    yardstick moves it 1.4e-5 relative); it is the noise term for programs
    with row reductions, as torch CUDA's own run is for GEMMs."""
    from oracle import executor as orc

    saved = (torch.softmax, torch.log_softmax, torch.nn.functional.softmax, torch.nn.functional.log_softmax,
             torch.Tensor.softmax, torch.Tensor.log_softmax)

    def wrap(f):
        def g(x, *a, **k):
            k.pop("dtype", None)
            return f(x.double(), *a, **k).to(x.dtype)
        return g

    torch.softmax, torch.log_softmax = wrap(saved[0]), wrap(saved[1])
    torch.nn.functional.softmax, torch.nn.functional.log_softmax = wrap(saved[2]), wrap(saved[3])
    torch.Tensor.softmax, torch.Tensor.log_softmax = wrap(saved[4]), wrap(saved[5])
    try:
        fn = orc.reference_callable(text, callable_name, dtype)
        logging.disable(logging.CRITICAL)
        try:
            with torch.no_grad(), contextlib.redirect_stdout(io.StringIO()):
                out = fn(*[a.clone() if torch.is_tensor(a) else a for a in args])
        finally:
            logging.disable(logging.NOTSET)
        return out
    finally:
        (torch.softmax, torch.log_softmax, torch.nn.functional.softmax, torch.nn.functional.log_softmax,
         torch.Tensor.softmax, torch.Tensor.log_softmax) = saved


def has_dense_contraction(text: str) -> bool:
    """Linear / matmul in the program (their accumulation order is unspecified)."""
    return any(k in text for k in ("nn.Linear", "matmul", " @ ", ".mm(", "torch.mm", "bmm", "F.linear"))


def _as_float(v) -> float:
    if torch.is_tensor(v):
        return float(v.double()) if v.dtype != torch.bool else float(bool(v))
    return float(v)


def check_scalars(low_gpu, text: str, callable_name: str, args_cpu: list, dtype, what: str = "") -> int:
    """Every region's branch decisions equal the oracle's, and every
    reduction statistic the kernel computed matches torch's CPU value on the
    kernel's own inputs within 1e-5 relative (bf16/fp16 results: 1e-2) plus
    the CPU's own measured drift (|fp32 result - fp64 result| of the same
    reduction: torch's CPU reductions of millions of elements drift, e.g.
    norm() up to 5e-4 relative).  Decisions are compared against the full
    oracle run (inputs computed by the CPU program itself) and the margin
    |stat - threshold| of each is logged.  Returns the number of decisions
    checked."""
    from paper_2509_16248_b200 import ir, lowering

    mod, low_cpu = lowering.load(text, allow_eager=True)
    for r in low_cpu.regions:
        r.trace = []
    fn = getattr(mod, callable_name)
    fn = getattr(fn, "_torchdynamo_orig_callable", fn)
    if dtype is not None and isinstance(fn, torch.nn.Module):
        fn.to(dtype)
    logging.disable(logging.CRITICAL)
    try:
        with torch.no_grad(), contextlib.redirect_stdout(io.StringIO()):
            fn(*[a.clone() if torch.is_tensor(a) else a for a in args_cpu])
    finally:
        logging.disable(logging.NOTSET)
    checked = 0
    for rg, rc in zip(low_gpu.regions, low_cpu.regions):
        spec = rg.last_spec
        if spec is None or not rc.trace:
            continue
        plan = spec.plan
        gpu = spec.scalars()
        # (1) decisions: the oracle's own inputs
        oracle = ir.evaluate(plan.decisions, list(rc.trace[-1]))
        for d in plan.decisions:
            want = bool(_as_float(oracle[d.uid]) != 0.0)
            got = gpu[plan.slot[d.uid]] != 0.0
            rec = {"what": what, "region": rg.name, "decision": d.op, "oracle": want, "b200": got}
            if d.op in ("gt", "ge", "lt", "le") and len(d.args) == 2:
                a, b = (_as_float(oracle[x.uid]) for x in d.args)
                rec.update(stat=a, threshold=b, margin=abs(a - b),
                           rel_margin=abs(a - b) / max(abs(b), 1e-30))
            MARGINS.append(rec)
            assert got == want, f"{what} {rg.name}: decision {d.op}#{d.uid} b200={got} oracle={want} ({rec})"
            checked += 1
        # (2) statistics: the kernel's own inputs, CPU arithmetic
        kin = [a.detach().cpu() if torch.is_tensor(a) else a for a in rg.last_args]
        reds = [n for n in plan.reductions if n.uid in plan.slot]
        vals = ir.evaluate(reds, kin)
        k64 = [a.double() if torch.is_tensor(a) and a.is_floating_point() else a for a in kin]
        try:
            vals64 = ir.evaluate(reds, k64)
        except Exception:
            vals64 = vals
        for n in reds:
            ref = _as_float(vals[n.uid])
            got = gpu[plan.slot[n.uid]]
            if ref != ref:  # NaN
                assert got != got, f"{what} {rg.name}: {n.op} NaN expected"
                continue
            drift = abs(ref - _as_float(vals64[n.uid]))
            rdt = n.dtype if isinstance(n.dtype, torch.dtype) else torch.float32
            tol = TOL.get(rdt, 0.0) * abs(ref) + drift
            if rdt in MANT:
                tol = max(tol, float(ulp(torch.tensor(ref), rdt)))
            assert abs(got - ref) <= tol or (rdt in (torch.int64, torch.int32, torch.bool) and got == ref), (
                f"{what} {rg.name}: statistic {n.op}#{n.uid} b200={got!r} cpu={ref!r} cpu_fp64_drift={drift:.3e}")
    return checked


def dump_margins(path: str) -> None:
    if not MARGINS:
        return
    with open(path, "a") as fh:
        for m in MARGINS:
            fh.write(json.dumps(m) + "\n")
    MARGINS.clear()

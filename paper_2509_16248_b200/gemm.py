"""Dense contractions of a lowered forward (csrc/gm_gemm.cu, include/gm_b200.h).

north_star keeps GEMMs on cuBLAS / tcgen05.  What changes here is WHICH
cuBLAS kernel an fp32 contraction runs: torch 2.11+cu128 would run SIMT
SGEMM (TF32 off, as the 1e-5 parity bound requires); gm_gemm_run runs
cuBLASLt 12.9's BF16x9 emulation on the tensor cores — 2.6x faster at the
BigBird Linear shape and closer to the exact product
(profiles/r02_gemm_emu_probe.txt).  bf16 / fp16 contractions stay on torch's
own cuBLAS call (the same tensor-core kernels).

It also implements the GEMM-bearing predicated block:
`where(p, A1 @ B1, A2 @ B2)` (transform.py:272 admits torch-rooted calls in
arms; :404-412 evaluates both) becomes gm_select_copy of each operand that
differs plus ONE GEMM (lowering._select_gemm_arms).

Outputs carry no autograd graph (the B200 path is an inference executor: a
CUDA-graph replay has none either).  When the eager op would have had a
grad_fn, its type name is recorded on the tensor (`_gm_grad_fn`) so a
deferred print renders the same text as the reference (logring.py).
"""

from __future__ import annotations

import ctypes
import functools
import math
import threading
import weakref

import torch

from . import _native as nat
from .region import stream_key

WS_BYTES = 32 << 20
_handles: dict = {}
_ws: dict = {}
_lock = threading.Lock()
stats = {"gm_gemm": 0, "torch_gemm": 0, "select_gemm": 0, "select_both": 0, "gm_copy": 0}


def _handle(dev: torch.device):
    idx = dev.index
    with _lock:
        h = _handles.get(idx)
        if h is None:
            nat.init(idx)
            h = ctypes.c_void_p()
            nat.check(nat.lib().gm_gemm_open(ctypes.byref(h)), "gm_gemm_open")
            _handles[idx] = h
        return h


def _workspace(dev: torch.device) -> torch.Tensor:
    """cuBLASLt workspace per (stream, graph capture): never shared by two
    streams or two graphs (region.stream_key)."""
    key = (dev.index,) + stream_key(dev)
    t = _ws.get(key)
    if t is None:
        t = torch.empty(WS_BYTES, dtype=torch.uint8, device=dev)
        _ws[key] = t
    return t


def _aligned(*ts) -> bool:
    return all(t is None or t.data_ptr() % 256 == 0 for t in ts)


@functools.lru_cache(maxsize=256)
def _grad_name(kind: str, shapes: tuple, dtype, flags: tuple) -> str | None:
    """type(grad_fn).__name__ the eager op would produce (meta tensors)."""
    ts = [None if s is None else torch.empty(s, device="meta", dtype=dtype, requires_grad=f)
          for s, f in zip(shapes, flags)]
    with torch.enable_grad():
        if kind == "linear":
            y = torch.nn.functional.linear(ts[0], ts[1], ts[2])
        elif kind == "linear_relu":
            y = torch.relu(torch.nn.functional.linear(ts[0], ts[1], ts[2]))
        else:
            y = torch.matmul(ts[0], ts[1])
    return type(y.grad_fn).__name__ if y.grad_fn is not None else None


def _tag(y: torch.Tensor, kind: str, ops: tuple) -> torch.Tensor:
    if torch.is_grad_enabled() and any(t is not None and t.requires_grad for t in ops):
        name = _grad_name(kind, tuple(None if t is None else tuple(t.shape) for t in ops), ops[0].dtype,
                          tuple(bool(t is not None and t.requires_grad) for t in ops))
        if name is not None:
            y._gm_grad_fn = name
    return y


def _fast(x: torch.Tensor, *rest) -> bool:
    ts = [x] + [t for t in rest if t is not None]
    return (x.dtype == torch.float32 and x.is_cuda and all(t.dtype == torch.float32 and t.device == x.device
                                                            for t in ts)
            and all(t.is_contiguous() for t in ts) and _aligned(*ts) and x.dim() >= 1)


def _run(dev, w_kn: int, x2: torch.Tensor, w: torch.Tensor, bias, relu: bool, y: torch.Tensor, M, N, K) -> None:
    stream = torch.cuda.current_stream(dev).cuda_stream
    ws = _workspace(dev)
    nat.count_launches()
    nat.check(nat.lib().gm_gemm_run(
        _handle(dev), nat.GM_F32, w_kn, ctypes.c_void_p(x2.data_ptr()), K, ctypes.c_void_p(w.data_ptr()),
        N if w_kn else K, ctypes.c_void_p(bias.data_ptr()) if bias is not None else None, int(relu),
        ctypes.c_void_p(y.data_ptr()), M, N, K, ctypes.c_void_p(ws.data_ptr()), WS_BYTES, ctypes.c_void_p(stream)),
        "gm_gemm_run")
    stats["gm_gemm"] += 1


def linear(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None = None, relu: bool = False):
    """torch.nn.functional.linear(x, weight, bias) (then relu): fp32 CUDA on
    gm_gemm_run (BF16x9), anything else on torch's cuBLAS call."""
    K = x.shape[-1] if x.dim() else 0
    if not (_fast(x, weight, bias) and weight.dim() == 2 and weight.shape[1] == K and K > 0
            and (bias is None or (bias.dim() == 1 and bias.shape[0] == weight.shape[0]))
            and x.numel() > 0):
        stats["torch_gemm"] += 1
        y = torch.nn.functional.linear(x, weight, bias)
        return torch.relu(y) if relu else y
    N = weight.shape[0]
    M = x.numel() // K
    y = torch.empty(*x.shape[:-1], N, dtype=x.dtype, device=x.device)
    _run(x.device, 0, x.reshape(M, K), weight, bias, relu, y, M, N, K)
    return _tag(y, "linear_relu" if relu else "linear", (x, weight, bias))


def contiguous(t: torch.Tensor) -> torch.Tensor:
    """t.contiguous() with the strided gather of gm_copy_strided when the
    innermost dim is contiguous and 16-byte sized (the head split of
    attention: [b, n, h, d] viewed as [b, h, n, d]), torch's copy otherwise."""
    if t.is_contiguous():
        return t
    es = t.element_size()
    if not (t.is_cuda and 1 <= t.dim() <= 6 and t.numel() > 0 and t.stride(-1) == 1
            and (t.shape[-1] * es) % 16 == 0 and t.data_ptr() % 16 == 0
            and all((st * es) % 16 == 0 for st in t.stride()[:-1])):
        return t.contiguous()
    dst = torch.empty(t.shape, dtype=t.dtype, device=t.device)
    nd = t.dim()
    sizes = (ctypes.c_int64 * nd)(*t.shape)
    strides = (ctypes.c_int64 * nd)(*t.stride())
    nat.count_launches()
    nat.check(nat.lib().gm_copy_strided(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(dst.data_ptr()), nd, sizes,
                                        strides, es, ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)),
              "gm_copy_strided")
    stats["gm_copy"] += 1
    return dst


def _batched_operand(t: torch.Tensor, rows: int, cols: int):
    """`t` ([..., rows, cols], CUDA) as packed [batch, rows, cols] matrices
    with one batch stride: (tensor, transposed) where `transposed` means the
    memory holds [batch, cols, rows] (a `.transpose(-1, -2)` view, read with
    op T).  When neither layout is a view (the head-split q / k / v of
    attention) the orientation whose innermost dim is contiguous is gathered
    (`contiguous`), so `k.transpose(-1, -2)` is read as k's rows with op T."""
    tt = t.transpose(-1, -2)
    for cand, trans in ((t, False), (tt, True)):
        r, c = (cols, rows) if trans else (rows, cols)
        try:
            v = cand.view(-1, r, c)
        except RuntimeError:
            continue
        if v.is_contiguous() and v.data_ptr() % 256 == 0:
            return v, trans
    if t.stride(-1) != 1 and tt.stride(-1) == 1:
        return contiguous(tt).view(-1, cols, rows), True
    return contiguous(t).view(-1, rows, cols), False


def matmul_batched(a: torch.Tensor, b: torch.Tensor):
    """torch.matmul of [..., M, K] @ [..., K, N] with equal batch dims (CUDA):
    ONE strided-batched cuBLASLt GEMM (gm_gemm_run_batched) — fp32 on the
    BF16x9 emulation instead of torch's SIMT SGEMM batches, bf16 / fp16 with
    fp32 accumulation — on operands gathered by gm_copy_strided only when no
    strided view exists."""
    M, K = a.shape[-2:]
    N = b.shape[-1]
    a3, ta = _batched_operand(a, M, K)
    if ta:
        a3 = contiguous(a3.transpose(-1, -2))   # x must be row-major [M, K]
    b3, tb = _batched_operand(b, K, N)
    batch = a3.shape[0]
    y = torch.empty(*a.shape[:-1], N, dtype=a.dtype, device=a.device)
    dev = a.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    ws = _workspace(dev)
    nat.count_launches()
    code = {torch.float32: nat.GM_F32, torch.bfloat16: nat.GM_BF16, torch.float16: nat.GM_F16}[a.dtype]
    # w_kn=1: w memory is [K, N] row-major (op N); w_kn=0: [N, K] (op T)
    nat.check(nat.lib().gm_gemm_run_batched(
        _handle(dev), code, 0 if tb else 1, ctypes.c_void_p(a3.data_ptr()), K, M * K,
        ctypes.c_void_p(b3.data_ptr()), K if tb else N, K * N, ctypes.c_void_p(y.data_ptr()), M * N, M, N, K, batch,
        ctypes.c_void_p(ws.data_ptr()), WS_BYTES, ctypes.c_void_p(stream)), "gm_gemm_run_batched")
    stats["gm_gemm"] += 1
    return _tag(y, "matmul", (a, b))


def matmul(a: torch.Tensor, b: torch.Tensor):
    """torch.matmul(a, b) / `a @ b`: an fp32 CUDA [.., M, K] @ [K, N] on
    gm_gemm_run, [..., M, K] @ [..., K, N] with equal batch dims on
    gm_gemm_run_batched, anything else on torch's cuBLAS call."""
    if (a.dtype in (torch.float32, torch.bfloat16, torch.float16) and b.dtype == a.dtype and a.is_cuda
            and b.device == a.device
            and a.dim() >= 3 and b.dim() == a.dim() and a.shape[:-2] == b.shape[:-2]
            and a.shape[-1] == b.shape[-2] and a.numel() > 0 and b.numel() > 0
            and math.prod(a.shape[:-2]) < 2 ** 31):
        return matmul_batched(a, b)
    if not (_fast(a, b) and b.dim() == 2 and a.dim() >= 2 and a.shape[-1] == b.shape[0] and b.shape[0] > 0
            and a.numel() > 0 and b.shape[1] > 0):
        stats["torch_gemm"] += 1
        return torch.matmul(a, b)
    K, N = b.shape
    M = a.numel() // K
    y = torch.empty(*a.shape[:-1], N, dtype=a.dtype, device=a.device)
    _run(a.device, 1, a.reshape(M, K), b, None, False, y, M, N, K)
    return _tag(y, "matmul", (a, b))


_ln_programs: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _layer_norm(mod, x):
    """nn.LayerNorm over the innermost dim as a row region (rowgen.py): the
    statement `F.layer_norm(x, (C,), w, b, eps)` lowered once per module (its
    own Region, so its launches are counted and timed apart from the other
    LayerNorms of the forward; the kernel source, and so the compiled cubin,
    is shared by modules with the same eps / affine form) and called like any
    region — one fused kernel instead of ATen's."""
    key = (float(mod.eps), mod.weight is not None, mod.bias is not None)
    ent = _ln_programs.get(mod)
    if ent is None or ent[0] != key:
        from .lowering import load

        w = "w" if key[1] else "None"
        b = "b" if key[2] else "None"
        text = ("import torch\n\ndef ln(x, w, b):\n"
                f"    return torch.nn.functional.layer_norm(x, (x.shape[-1],), {w}, {b}, {key[0]!r})\n")
        mod_, low = load(text)
        for r in low.regions:
            r.name = f"nn.LayerNorm #{len(_ln_programs) + 1}"
        ent = _ln_programs[mod] = (key, mod_.ln, low)
    return ent[1](x, mod.weight, mod.bias)


def module_regions(model) -> list:
    """The fused regions behind module calls of `model`'s submodules (the
    LayerNorm row regions), in creation order: for reports and timing next
    to the lowered program's own regions."""
    mods = set(id(m) for m in model.modules()) if isinstance(model, torch.nn.Module) else None
    res = []
    for mod, (_key, _fn, low) in list(_ln_programs.items()):
        if mods is None or id(mod) in mods:
            res.extend(low.regions)
    return res


def module_call(mod, x):
    """`self.<sub>(x)` of the transformed forward: an nn.Linear without hooks
    runs `linear`, an nn.LayerNorm over the innermost dim a fused row region;
    every other module is called as written."""
    if (type(mod) is torch.nn.Linear and not mod._forward_hooks and not mod._forward_pre_hooks
            and torch.is_tensor(x)):
        return linear(x, mod.weight, mod.bias)
    if (type(mod) is torch.nn.LayerNorm and not mod._forward_hooks and not mod._forward_pre_hooks
            and torch.is_tensor(x) and x.is_cuda and len(mod.normalized_shape) == 1 and x.dim() >= 1
            and x.shape[-1] == mod.normalized_shape[0] and x.numel() > 0
            and x.dtype in (torch.float32, torch.bfloat16, torch.float16)
            and all(p is None or (p.dtype == x.dtype and p.device == x.device) for p in (mod.weight, mod.bias))):
        return _layer_norm(mod, x)
    return mod(x)


def _select(pred: torch.Tensor, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """`a if pred else b` on the device (same shape/dtype): a single copy of
    the selected operand; `a` itself when both are the same tensor."""
    if a is b or (a.data_ptr() == b.data_ptr() and a.shape == b.shape and a.stride() == b.stride()):
        return a
    a, b = a.contiguous(), b.contiguous()
    dst = torch.empty_like(a)
    nat.count_launches()
    nat.check(nat.lib().gm_select_copy(
        ctypes.c_void_p(pred.data_ptr()), pred.element_size(), ctypes.c_void_p(a.data_ptr()),
        ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(dst.data_ptr()), a.numel() * a.element_size(),
        ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)), "gm_select_copy")
    return dst


def select_gemm(pred, kind: str, then_ops: tuple, else_ops: tuple):
    """The contraction the `where` keeps: `gemm(*then_ops) if pred else
    gemm(*else_ops)`, gemm = matmul (ops (a, b)) or linear (ops (x, w, b)).
    With a 0-d CUDA predicate and arms of identical operand shapes / dtypes
    the operands that differ are selected on the device and ONE GEMM runs;
    otherwise both run and the predicate selects (the rewrite's own
    semantics, transform.py:404-412)."""
    f = matmul if kind == "matmul" else linear
    ok = (torch.is_tensor(pred) and pred.is_cuda and pred.numel() == 1 and pred.dtype == torch.bool
          and len(then_ops) == len(else_ops)
          and all((p is None) == (q is None) for p, q in zip(then_ops, else_ops))
          and all(p is None or (torch.is_tensor(p) and torch.is_tensor(q) and p.is_cuda and q.device == p.device
                                and p.shape == q.shape and p.dtype == q.dtype)
                  for p, q in zip(then_ops, else_ops)))
    if isinstance(pred, bool):
        return f(*then_ops) if pred else f(*else_ops)
    if not ok:
        stats["select_both"] += 1
        return torch.where(pred, f(*then_ops), f(*else_ops))
    stats["select_gemm"] += 1
    ops = tuple(None if p is None else _select(pred.reshape(()), p, q) for p, q in zip(then_ops, else_ops))
    y = f(*ops)
    if hasattr(y, "_gm_grad_fn"):
        del y._gm_grad_fn
    return _tag(y, kind, then_ops)

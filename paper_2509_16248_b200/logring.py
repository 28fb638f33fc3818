"""I/O-deferral runtime: device log ring + host drain.

The reference defers `print` / `logger.*` by capturing the argument tuple at
the call site and replaying `callee(*__gm_defer_k)` before each return
(transform.py:744-771, :675-734).  Executed on a GPU, that replay still
formats CUDA tensors inside the forward — a device-to-host read per tensor.

Here a replay inside an active step
  * keeps host constants as they are (the tuple holds them by reference);
  * for each CUDA tensor argument launches one gather kernel that copies
    exactly the elements torch's repr reads (get_summarized_data: edgeitems
    3 per dim when numel > threshold 1000, torch/_tensor_str.py) into a slot
    of a pinned, device-mapped host ring (gm_logring_gather);
  * records (callee, argument template) in the step's call list.
A step that gathered tensors then bumps the device slot counter
(gm_logring_commit) and records a CUDA event behind itself; a host thread
(or `flush()`) polls that event — it never synchronises the stream —
rebuilds CPU tensors whose repr is identical to the original's, and calls
the original callee in source order, so level checks happen at drain time
exactly as if the call ran late.  A step whose deferred calls carry host
constants only (the whole corpus) costs no device work at all.

Outside a step (a plain call of the lowered function) replay is immediate,
which is the reference's behaviour.
"""

from __future__ import annotations

import ctypes
import os
import math
import threading
import time
from collections import deque
from dataclasses import dataclass, field

import torch

from . import _native as nat
from . import gemm
from .region import stream_key, zeroed

EDGEITEMS = 3      # torch._tensor_str.PRINT_OPTS defaults
THRESHOLD = 1000

_DT = {
    torch.float32: (nat.GM_F32, 4), torch.bfloat16: (nat.GM_BF16, 2), torch.float16: (nat.GM_F16, 2),
    torch.float64: (nat.GM_F64, 8), torch.bool: (nat.GM_BOOL, 1), torch.int32: (nat.GM_I32, 4),
    torch.int64: (nat.GM_I64, 8), torch.uint8: (nat.GM_U8, 1),
}


_CODE_DT = {code: dt for dt, (code, _) in _DT.items()}


def summary_plan(shape: tuple[int, ...]) -> tuple[list[int], list[int]]:
    """(count, head) per dim of the elements torch's repr reads."""
    numel = math.prod(shape)
    summarize = numel > THRESHOLD
    counts, heads = [], []
    for s in shape:
        if summarize and s > 2 * EDGEITEMS:
            counts.append(2 * EDGEITEMS)
            heads.append(EDGEITEMS)
        else:
            counts.append(s)
            heads.append(s)
    return counts, heads


@dataclass
class TensorRef:
    """A tensor argument of a deferred call: captured as record `record_id`
    (gm_logring_capture); rebuilt from the drained record."""
    record_id: int
    dtype: torch.dtype
    shape: tuple
    grad_fn: str | None
    requires_grad: bool


@dataclass
class StepTemplate:
    calls: list = field(default_factory=list)   # (site, callee, [arg | TensorRef])
    discard: bool = False
    gathers: int = 0                            # records captured by the step
    template_id: int | None = None              # gm_logring_end_step's id (None: no device work)


class _TensorText:
    """str()/repr() of a tensor that carried a grad_fn (or requires_grad) in
    the forward; the reconstructed CPU tensor has neither, so the suffix is
    added the way torch._tensor_str._str_intern does."""

    def __init__(self, t: torch.Tensor, grad_fn: str | None, requires_grad: bool):
        self.t = t
        self.grad_fn = grad_fn
        self.requires_grad = requires_grad

    def __repr__(self) -> str:
        from torch import _tensor_str as ts

        with torch.no_grad():
            prefix = "tensor("
            indent = len(prefix)
            suffixes = []
            t = self.t
            default = t.dtype in (torch.get_default_dtype(), torch.int64, torch.bool)
            if t.numel() == 0:
                body = "[]"
                if t.dim() != 1:
                    suffixes.append("size=" + str(tuple(t.shape)))
                if t.dtype != torch.get_default_dtype():
                    suffixes.append("dtype=" + str(t.dtype))
            else:
                if not default:
                    suffixes.append("dtype=" + str(t.dtype))
                body = ts._tensor_str(t, indent)
            if self.grad_fn is not None:
                suffixes.append(f"grad_fn=<{self.grad_fn}>")
            elif self.requires_grad:
                suffixes.append("requires_grad=True")
            return ts._add_suffixes(prefix + body, suffixes, indent, force_newline=False)

    __str__ = __repr__

    def __format__(self, spec):
        return format(str(self), spec)


RECORD_CB = nat.RECORD_CB
_record_ids = iter(range(1, 1 << 32))
# torch.ops.gm.log_capture records: record id -> handler(tensor)
_record_handlers: dict[int, object] = {}


def on_record(record_id: int, handler) -> None:
    """Deliver every drained record `record_id` (a tensor captured with
    torch.ops.gm.log_capture) to `handler(tensor)`."""
    _record_handlers[int(record_id)] = handler


class LogRing:
    """Pinned, device-mapped ring for one device, on the record-level C API:
    gm_logring_begin_step / gm_logring_capture (one gather per tensor
    argument) / gm_logring_end_step (slot header + counter) on the producer
    side, gm_logring_drain (a C callback per record, in commit order) on the
    consumer side.  The drain never synchronises a stream: completion is the
    committed-step counter in mapped host memory."""

    def __init__(self, device: torch.device, slot_bytes: int = 1 << 20, n_slots: int = 64):
        self.device = device
        self.n_slots = nat.LOGRING_SLOTS
        self.slot_bytes = slot_bytes
        nat.init(device.index)
        h = ctypes.c_void_p()
        nat.check(nat.lib().gm_logring_open(slot_bytes * self.n_slots, ctypes.byref(h)), "gm_logring_open")
        self.handle = h
        self.lock = threading.RLock()
        self.pending: deque = deque()        # launched steps with deferred calls, in launch order
        self.arrived: deque = deque()        # drained steps: {record_id: (dtype, shape, counts, heads, bytes)}
        self.launched = 0
        self.drained = 0
        self.gather_steps = 0                # steps that commit on the device
        self.drained_gather_steps = 0
        self._active: StepTemplate | None = None
        self.gathers = 0
        self._thread = None
        self._stop = False
        self._cb = RECORD_CB(self._on_record)
        self._current: dict | None = None
        self._current_step = None

    # -- producer side (forward) ------------------------------------------------
    def begin(self, discard: bool = False) -> None:
        if self._active is not None:
            raise RuntimeError("log ring step already active")
        nat.check(nat.lib().gm_logring_begin_step(self.handle), "gm_logring_begin_step")
        self._active = StepTemplate(discard=discard)

    def capture(self, t: torch.Tensor, record_id: int) -> None:
        """gm_logring_capture of one CUDA tensor into the open step."""
        if t.dtype not in _DT:
            raise TypeError(f"log ring: unsupported dtype {t.dtype}")
        code, _ = _DT[t.dtype]
        nd = t.dim()
        shape = (ctypes.c_int64 * max(1, nd))(*t.shape)
        stride = (ctypes.c_int64 * max(1, nd))(*t.stride())
        stream = torch.cuda.current_stream(self.device).cuda_stream
        nat.check(nat.lib().gm_logring_capture(self.handle, ctypes.c_void_p(t.data_ptr()), shape, stride, nd, code,
                                               int(record_id), ctypes.c_void_p(stream)), "gm_logring_capture")
        nat.count_launches()
        self.gathers += 1
        self._active.gathers += 1

    def record(self, site: int, callee, args: tuple) -> None:
        tmpl = self._active
        out = []
        for a in args:
            if torch.is_tensor(a) and a.device.type == "cuda":
                rid = next(_record_ids)
                self.capture(a, rid)
                gf = a.grad_fn
                # gemm.py records the grad_fn name the eager op would have had
                name = getattr(a, "_gm_grad_fn", None) or (type(gf).__name__ if gf is not None else None)
                out.append(TensorRef(rid, a.dtype, tuple(a.shape), name, a.requires_grad))
            elif torch.is_tensor(a):
                out.append(a.detach().clone() if not a.requires_grad else a)
            else:
                out.append(a)
        tmpl.calls.append((site, callee, out))

    def end(self) -> StepTemplate:
        """Close the step (gm_logring_end_step): a step with records launches
        the commit kernel; a step whose deferred calls carry host constants
        only launches nothing at all."""
        tmpl = self._active
        self._active = None
        tid = ctypes.c_uint32(0)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        nat.check(nat.lib().gm_logring_end_step(self.handle, ctypes.c_void_p(stream), ctypes.byref(tid)),
                  "gm_logring_end_step")
        if tid.value != nat.LOGRING_NO_TEMPLATE:
            tmpl.template_id = tid.value
            nat.count_launches()
        return tmpl

    @property
    def active(self) -> bool:
        return self._active is not None

    def enqueue(self, tmpl: StepTemplate) -> None:
        """Register one launched step (eager or graph replay), in stream
        order.  Steps with records commit on the device; steps without
        records and without deferred calls are not queued."""
        if not tmpl.calls and tmpl.template_id is None:
            return
        with self.lock:
            if tmpl.template_id is not None:
                # back-pressure: never run more than n_slots-1 committing steps ahead
                while self.gather_steps - self.drained_gather_steps >= self.n_slots - 1:
                    self._drain_one(block=True)
                self.gather_steps += 1
            self.launched += 1
            self.pending.append((self.launched, tmpl))

    # -- consumer side (host) -------------------------------------------------------
    def committed(self) -> int:
        return int(nat.lib().gm_logring_committed(self.handle))

    def _on_record(self, rec_p, _user) -> int:
        try:
            rec = rec_p.contents
            if rec.step != self._current_step:
                self._current = {}
                self._current_step = rec.step
                self.arrived.append(self._current)
            nd = rec.ndim
            self._current[rec.record_id] = (rec.dtype, tuple(rec.shape[i] for i in range(nd)),
                                            tuple(rec.counts[i] for i in range(nd)),
                                            tuple(rec.heads[i] for i in range(nd)),
                                            ctypes.string_at(rec.data, rec.bytes) if rec.bytes else b"")
            return 0
        except Exception:   # never raise through the C callback
            return 1

    def _poll(self) -> None:
        rc = nat.lib().gm_logring_drain(self.handle, self._cb, None)
        if rc < 0:
            nat.check(rc, "gm_logring_drain")

    @staticmethod
    def _rebuild_record(raw, ref: TensorRef | None = None):
        code, shape, counts, heads, data = raw
        dtype = _CODE_DT[code]
        n = math.prod(counts)
        block = torch.frombuffer(bytearray(data), dtype=dtype).reshape(counts) if n else torch.empty(counts,
                                                                                                      dtype=dtype)
        if list(counts) == list(shape):
            full = block.clone()
        else:
            full = torch.empty(shape, dtype=dtype)
            idx = []
            nd = len(shape)
            for d, (c, h, sz) in enumerate(zip(counts, heads, shape)):
                ix = torch.tensor([k if k < h else sz - c + k for k in range(c)], dtype=torch.long)
                view = [1] * nd
                view[d] = c
                idx.append(ix.view(view))
            full[tuple(idx)] = block
        if ref is not None and (ref.grad_fn is not None or ref.requires_grad):
            return _TensorText(full, ref.grad_fn, ref.requires_grad)
        return full

    def _drain_one(self, block: bool) -> bool:
        with self.lock:
            if not self.pending:
                # records of steps launched outside a step template
                # (torch.ops.gm.log_capture in a bare call) still arrive
                self._poll()
                self._deliver_orphans()
                return False
            step, tmpl = self.pending[0]
            raw = None
            if tmpl.template_id is not None:
                t_spin = None
                while True:
                    if not self.arrived:
                        self._poll()
                    if self.arrived:
                        raw = self.arrived.popleft()
                        break
                    if not block:
                        return False
                    # spin on the mapped commit word for the first 2 ms: a
                    # sleep rounds up to the kernel's timer slack (~50-80 us),
                    # longer than most forwards this waits on
                    now = time.perf_counter()
                    if t_spin is None:
                        t_spin = now
                    if now - t_spin > 2e-3:
                        time.sleep(20e-6)
            self.pending.popleft()
            if raw is not None:
                self.drained_gather_steps += 1
                refs = {}
                for _site, _callee, args in tmpl.calls:
                    for a in args:
                        if isinstance(a, TensorRef):
                            refs[a.record_id] = a
                for rid, rec in raw.items():
                    if rid not in refs and rid in _record_handlers and not tmpl.discard:
                        _record_handlers[rid](self._rebuild_record(rec))
            if not tmpl.discard:
                for _site, callee, args in tmpl.calls:
                    real = [self._rebuild_record(raw[a.record_id], a) if isinstance(a, TensorRef) else a
                            for a in args]
                    callee(*real)
            self.drained = step
            return True

    def _deliver_orphans(self) -> None:
        while self.arrived:
            raw = self.arrived.popleft()
            for rid, rec in raw.items():
                h = _record_handlers.get(rid)
                if h is not None:
                    h(self._rebuild_record(rec))

    def flush(self) -> None:
        """Drain every launched step (waits for their commits, in order)."""
        while self._drain_one(block=True):
            pass

    def start_drain_thread(self) -> None:
        if self._thread is not None:
            return

        def loop():
            while not self._stop:
                if not self._drain_one(block=False):
                    time.sleep(100e-6)

        self._thread = threading.Thread(target=loop, name="gm-logring-drain", daemon=True)
        self._thread.start()

    def close(self) -> None:
        self._stop = True
        if self._thread is not None:
            self._thread.join(timeout=1.0)
        try:
            self.flush()
        finally:
            nat.lib().gm_logring_close(self.handle)
            self.handle = None


_rings: dict[int, LogRing] = {}
_rings_lock = threading.Lock()


def ring_for(device: torch.device) -> LogRing:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    with _rings_lock:
        if idx not in _rings:
            _rings[idx] = LogRing(torch.device("cuda", idx))
        return _rings[idx]


_tls = threading.local()


def active_ring() -> LogRing | None:
    return getattr(_tls, "ring", None)


class step:
    """Context manager: one forward as one log-ring step on `device`."""

    def __init__(self, device: torch.device, discard: bool = False):
        self.ring = ring_for(device)
        self.discard = discard
        self.template: StepTemplate | None = None

    def __enter__(self):
        self.ring.begin(self.discard)
        _tls.ring = self.ring
        return self

    def __exit__(self, *exc):
        _tls.ring = None
        self.template = self.ring.end()
        return False


_unique_scratch_by_dev: dict = {}


def _unique_scratch(device) -> torch.Tensor:
    """Bitmap scratch of gm_unique_sum16, one per (stream, graph capture)
    (region.stream_key): calls on one stream are ordered, so one buffer
    serves them all, and concurrent streams or graphs never share one."""
    key = (device.index,) + stream_key(device)
    t = _unique_scratch_by_dev.get(key)
    if t is None:
        t = zeroed(nat.lib().gm_unique_sum16_scratch_bytes(), device)
        _unique_scratch_by_dev[key] = t
    return t


_hash_scratch_by_dev: dict = {}


def _hash_scratch(device, nbytes: int) -> torch.Tensor:
    """Per-device hash-set scratch of gm_unique_sum32_hash, zeroed once and
    kept: the bitmap pass clears what it read and the hash slots carry a
    call tag, so nothing is cleared per call.  A larger request allocates a
    larger buffer; the smaller ones stay alive for CUDA graphs that captured
    them.  One set per (stream, graph capture) (region.stream_key), so
    concurrent streams or graphs never share a table."""
    key = (device.index,) + stream_key(device)
    bufs = _hash_scratch_by_dev.setdefault(key, [])
    if not bufs or bufs[-1].numel() < nbytes:
        bufs.append(zeroed(nbytes, device))
    return bufs[-1]


class ModuleRuntime:
    """`__gm_rt` of a lowered module: its fused regions and replay sites."""

    def __init__(self, lowered):
        self.lowered = lowered
        self.regions = lowered.regions
        self.sites = lowered.sites
        self.immediate_replays = 0

    # -- fixed-shape replacements of dynamic-shape ops whose
    #    only consumer is a full sum (see lowering._lower_dynamic_shape)
    @staticmethod
    def call(mod, x):
        """`self.<sub>(x)`: an nn.Linear runs gemm.linear (fp32: cuBLASLt
        BF16x9 on the tensor cores), any other module as written."""
        return gemm.module_call(mod, x)

    @staticmethod
    def inlined_layer_norms(owner, names: tuple) -> None:
        """Guard of lowering._inline_layer_norms: every `self.<name>` the
        lowering inlined as F.layer_norm must still be a plain nn.LayerNorm
        (no forward hooks, a one-dimensional normalized_shape) — else the
        inlined statement would not be what `self.<name>(x)` computes, so
        raise instead of running it."""
        for n in names:
            m = getattr(owner, n, None)
            if (type(m) is not torch.nn.LayerNorm or m._forward_hooks or m._forward_pre_hooks
                    or len(m.normalized_shape) != 1):
                raise RuntimeError(f"self.{n} was lowered as F.layer_norm (an nn.LayerNorm built in __init__), "
                                   f"but is now a {type(m).__name__} with hooks or another shape")

    @staticmethod
    def matmul(a, b):
        """`a @ b` / torch.matmul(a, b): gemm.matmul."""
        return gemm.matmul(a, b)

    @staticmethod
    def linear(x, w, b=None):
        """torch.nn.functional.linear(x, w, b): gemm.linear."""
        return gemm.linear(x, w, b)

    @staticmethod
    def reshape(t, *shape):
        """`t.reshape(*shape)`: the view when one exists, else a packed copy —
        torch's semantics — made by gm_copy_strided when the innermost dim is
        contiguous (attention's head merge `ctx.transpose(1, 2).reshape(b, n,
        h)`), not torch's per-element permute copy."""
        if not torch.is_tensor(t):
            return t.reshape(*shape)
        try:
            return t.view(*shape)
        except RuntimeError:
            return gemm.contiguous(t).view(*shape)

    @staticmethod
    def contiguous(t):
        """`t.contiguous()` through gemm.contiguous."""
        return gemm.contiguous(t) if torch.is_tensor(t) else t.contiguous()

    @staticmethod
    def select_gemm(pred, kind, then_ops, else_ops):
        """The one GEMM a GEMM-bearing predicated block needs (gemm.select_gemm)."""
        return gemm.select_gemm(pred, kind, then_ops, else_ops)

    @staticmethod
    def linear_relu(mod, x):
        """relu(mod(x)).  For an nn.Linear with bias on a CUDA tensor: one
        GEMM with a RELU_BIAS epilogue (fp32: gemm.linear on cuBLASLt BF16x9;
        16-bit: torch._addmm_activation) instead of a GEMM and a separate
        relu launch — relu commutes with the rounding of the output, so the
        value is relu(Linear(x))."""
        if (type(mod) is torch.nn.Linear and not mod._forward_hooks and not mod._forward_pre_hooks
                and torch.is_tensor(x) and x.dtype == torch.float32 and x.is_cuda):
            return gemm.linear(x, mod.weight, mod.bias, relu=True)
        if (isinstance(mod, torch.nn.Linear) and mod.bias is not None and torch.is_tensor(x) and x.is_cuda
                and x.dim() >= 2 and x.dtype == mod.weight.dtype and x.shape[-1] == mod.in_features):
            y = torch._addmm_activation(mod.bias, x.reshape(-1, mod.in_features), mod.weight.t())
            return y.view(*x.shape[:-1], mod.out_features)
        return torch.relu(mod(x))

    @staticmethod
    def nonzero_sum(mask):
        """== torch.nonzero(mask).sum() (int64).  Inside a fused region this
        is a coordinate-sum reduction; here (unfused) it is computed without
        sizing a dynamic output: sum over dims of (coordinate * mask)."""
        m = mask != 0
        total = torch.zeros((), dtype=torch.int64, device=m.device)
        for d, n in enumerate(m.shape):
            shape = [1] * m.dim()
            shape[d] = n
            coord = torch.arange(n, device=m.device, dtype=torch.int64).view(shape)
            total = total + (coord * m).sum()
        return total

    @staticmethod
    def unique_sum(x):
        """== x.unique().sum() with fixed shapes (no host sync).  bf16/f16 on
        the GPU: one pass into a 65536-bit presence bitmap and a sum of the
        set bits (gm_unique_sum16); fp32 on the GPU: a presence bitmap over
        a 16-binade window (a hash set for the other values) and an exact
        fixed-point sum of the distinct values, rounded once
        (gm_unique_sum32_hash; GM_UNIQUE32=sort selects the radix-sort
        form gm_unique_sum32).  Otherwise (CPU tensors): sort, keep
        the first of each run of equal values, sum."""
        if x.is_cuda:
            nat.init(x.device.index if x.device.index is not None else torch.cuda.current_device())
        if x.is_cuda and x.dtype in (torch.bfloat16, torch.float16) and x.is_contiguous() \
                and x.data_ptr() % 16 == 0:
            out = torch.empty((), dtype=x.dtype, device=x.device)
            scratch = _unique_scratch(x.device)
            nat.count_launches(2)
            nat.check(nat.lib().gm_unique_sum16(
                ctypes.c_void_p(x.data_ptr()), x.numel(), nat.GM_BF16 if x.dtype == torch.bfloat16 else nat.GM_F16, ctypes.c_void_p(out.data_ptr()),
                ctypes.c_void_p(scratch.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)),
                "gm_unique_sum16")
            return out
        if x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and 0 < x.numel() < 2 ** 31 \
                and os.environ.get("GM_UNIQUE32", "hash") != "sort":
            out = torch.empty((), dtype=x.dtype, device=x.device)
            nb = nat.lib().gm_unique_sum32_hash_scratch_bytes(x.numel())
            scratch = _hash_scratch(x.device, nb)
            nat.count_launches(3)
            nat.check(nat.lib().gm_unique_sum32_hash(
                ctypes.c_void_p(x.data_ptr()), x.numel(), ctypes.c_void_p(out.data_ptr()),
                ctypes.c_void_p(scratch.data_ptr()), nb, ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)),
                "gm_unique_sum32_hash")
            return out
        if x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and 0 < x.numel() < 2 ** 31:
            out = torch.empty((), dtype=x.dtype, device=x.device)
            nb = nat.lib().gm_unique_sum32_scratch_bytes(x.numel())
            scratch = torch.empty(nb, dtype=torch.uint8, device=x.device)
            nat.count_launches(2)  # the two distinct-sum kernels (the CUB radix-sort passes are not counted)
            nat.check(nat.lib().gm_unique_sum32(
                ctypes.c_void_p(x.data_ptr()), x.numel(), ctypes.c_void_p(out.data_ptr()),
                ctypes.c_void_p(scratch.data_ptr()), nb, ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)),
                "gm_unique_sum32")
            return out
        s = x.reshape(-1).sort().values
        keep = torch.ones_like(s, dtype=torch.bool)
        if s.numel() > 1:
            keep[1:] = s[1:] != s[:-1]
        return torch.where(keep, s, torch.zeros((), dtype=s.dtype, device=s.device)).sum()

    def replay(self, site: int, callee, captured: tuple) -> None:
        ring = active_ring()
        if ring is None:
            self.immediate_replays += 1
            callee(*captured)
            return
        ring.record(site, callee, captured)

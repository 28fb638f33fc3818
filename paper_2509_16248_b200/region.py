"""Runtime side of a fused region: specialisation cache, launch, scratch.

A `Region` is created by the lowering (lowering.py) for one run of fusable
statements.  Calling it with the region's free values launches one
NVRTC-compiled sm_100a kernel (codegen.py + csrc/gm_region.cuh) on the
current CUDA stream and returns the live-out tensors.  Launches are
stream-ordered and graph-capturable; no call synchronises with the host.

When the arguments leave the fusable subset (integer tensors, CPU tensors,
shapes that do not broadcast to one iteration space, ...), the region runs
its original statements with PyTorch instead — the exact code the reference
transform emitted (`fallback`), on the device the tensors live on.  Every
such decision is recorded in `Region.stats` so tests can assert that the
fused kernel is what ran.  Missing native code is never a fallback: a
NativeError propagates.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import threading
from dataclasses import dataclass, field

import torch

from . import _native as nat
from .codegen import MODE_PERIODIC, MODE_STRIDED, Plan
from .ir import Graph, Node, Unsupported

SCRATCH_PARTIALS = 2432  # GM_SCRATCH_PARTIALS in csrc/gm_region.cuh
SCRATCH_STATS = 32      # GM_SCRATCH_STATS: u64 [speculative launches, mispredictions]
SCRATCH_PRED = 288      # GM_SCRATCH_PRED: int predicted decisions
_kernel_cache: dict[str, nat.CompiledRegion] = {}
_kernel_lock = threading.Lock()


PDL = os.environ.get("GM_PDL", "1") != "0"
KCACHE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_kcache")


def _skeleton_digest() -> str:
    """The cubin depends on the generated source AND on the skeleton header
    NVRTC includes, so both key the cache."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc", "gm_region.cuh")
    with open(path, "rb") as fh:
        return hashlib.sha1(fh.read()).hexdigest()


_SKELETON = _skeleton_digest()


def kcache_path(source: str, arch: str = "sm100a") -> str:
    key = hashlib.sha1((_SKELETON + "\n" + source).encode()).hexdigest()
    return os.path.join(KCACHE_DIR, f"{key}_{arch}.cubin")


def compiled_kernel(source: str, kernel: str) -> nat.CompiledRegion:
    """In-process cache, then the ahead-of-time cubin cache (filled by
    __graft_entry__.build() for the known workloads), then NVRTC."""
    with _kernel_lock:
        k = _kernel_cache.get(source)
        if k is None:
            path = kcache_path(source)
            cubin = None
            if os.path.exists(path):
                with open(path, "rb") as fh:
                    cubin = fh.read()
            k = nat.CompiledRegion(source, kernel, cubin=cubin)
            _kernel_cache[source] = k
        return k


def aot_compile(source: str) -> str:
    """NVRTC-compile `source` for sm_100a into the cubin cache (no GPU)."""
    path = kcache_path(source)
    if not os.path.exists(path):
        os.makedirs(KCACHE_DIR, exist_ok=True)
        cubin = nat.compile_cubin(source, (10, 0))
        tmp = path + ".tmp"
        with open(tmp, "wb") as fh:
            fh.write(cubin)
        os.replace(tmp, path)
    return path


def arg_key(a) -> tuple:
    if torch.is_tensor(a):
        return ("t", a.dtype, tuple(a.shape), tuple(a.stride()), a.device.type, a.device.index,
                a.data_ptr() % 16 == 0)
    if isinstance(a, (bool, int, float)):
        # bf16-exactness of a host scalar selects the packed bf16 code path
        f = torch.tensor(float(a), dtype=torch.float32)
        return ("h", type(a), bool(f.to(torch.bfloat16).float() == f))
    return ("o", type(a))


@dataclass
class RegionStats:
    launches: int = 0
    fallbacks: int = 0
    fallback_reasons: list = field(default_factory=list)


class _Spec:
    """A compiled specialisation plus its launch configuration."""

    def __init__(self, region: "Region", args: list):
        dev = next(a.device for a in args if torch.is_tensor(a) and a.device.type == "cuda")
        self.device = dev
        sms, smem_optin = nat.init(dev.index if dev.index is not None else torch.cuda.current_device())
        plan = Plan(region.graph, region.out_nodes, args, name=region.name, device_info=(sms, smem_optin))
        self.plan = plan
        self.kernel = compiled_kernel(plan.source, plan.kernel)
        n = plan.n
        nvec = -(-n // nat.VEC) if n else 0
        threads = plan.threads
        grid, smem = plan.grid, plan.smem_bytes
        vpc = plan.K
        if plan.reductions and grid > 1:
            # the grid barrier needs every CTA resident at once
            occ = self.kernel.occupancy(threads, smem)
            if occ * sms < grid:
                raise nat.NativeError(f"region {region.name}: {grid} CTAs not co-resident "
                                      f"({occ}/SM at {smem} B smem, {sms} SMs)")
        self.grid, self.vpc, self.smem, self.threads = grid, vpc, smem, threads
        self.nred = len(plan.reductions)
        self.nscal = len(plan.scalars)
        # scratch: counter/epoch/status/results (192 B, see gm_region.cuh) |
        # partials | scalar mirror (+1 KB: the GM_PROFILE timeline at scal_out + 64 u64)
        part_bytes = 8 * max(1, self.nred) * grid
        self.scratch = torch.zeros(SCRATCH_PARTIALS + part_bytes + 8 * 64 + 8 * 64 + 8 * max(1, self.nscal),
                                   dtype=torch.uint8, device=dev)
        base = self.scratch.data_ptr()
        P = nat.Params()
        P.n = n
        P.nvec = nvec
        P.vpc = vpc
        P.piece_vecs = 1  # (bulk-copy staging: gm_branch_select_f32 only)
        P.barrier = base
        P.status = base + 16
        P.partials = base + SCRATCH_PARTIALS
        P.scal_out = base + SCRATCH_PARTIALS + part_bytes
        self.template = P
        self.in_slots = []  # (slot, free_index, mode)
        for ip in plan.inputs:
            d = P.inp[ip.slot]
            d.smem_off = plan.smem_off.get(ip.slot, -1)
            if ip.mode == MODE_PERIODIC:
                t = args[ip.free_index]
                d.size[0] = t.numel()
            elif ip.mode == MODE_STRIDED:
                t = args[ip.free_index]
                S = tuple(plan.shape)
                ex = t.expand(S)
                if len(S) > nat.MAX_DIMS:
                    raise Unsupported("too many dims for a strided input")
                d.ndim = len(S)
                for j, (s, st) in enumerate(zip(S, ex.stride())):
                    d.size[j] = s
                    d.stride[j] = st
            self.in_slots.append((ip.slot, ip.free_index))
        self.hs_index = [node.value for node in plan.host_frees]
        # outputs
        self.out_specs = []  # (out position, kind, dtype, kernel slot or None)
        k = 0
        for j, o in enumerate(plan.outputs):
            if o.op == "free":
                self.out_specs.append((j, "alias", o.value, None))
            elif o.kind == "elem":
                self.out_specs.append((j, "elem", o.dtype, k))
                k += 1
            else:
                self.out_specs.append((j, "scalar", o.dtype, k))
                k += 1
        self.shape = tuple(plan.shape)

    def run(self, args: list, pdl: bool | None = None):
        """Launch on the current stream.  `pdl` (default: GM_PDL, on) makes it
        a programmatic dependent launch: the CTAs become resident while the
        previous kernel drains and wait (griddepcontrol.wait) for its results
        before reading anything."""
        P = nat.Params()
        ctypes.memmove(ctypes.byref(P), ctypes.byref(self.template), ctypes.sizeof(P))
        for slot, fi in self.in_slots:
            P.inp[slot].ptr = args[fi].data_ptr()
        for j, fi in enumerate(self.hs_index):
            P.hs[j] = float(args[fi])
        outs = [None] * len(self.out_specs)
        for j, kind, info, k in self.out_specs:
            if kind == "alias":
                outs[j] = args[info]
            elif kind == "elem":
                t = torch.empty(self.shape, dtype=info, device=self.device)
                P.out[k].ptr = t.data_ptr()
                outs[j] = t
            else:
                t = torch.empty((), dtype=info, device=self.device)
                P.out[k].ptr = t.data_ptr()
                outs[j] = t
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.kernel.launch(P, self.grid, self.threads, self.smem, stream, PDL if pdl is None else pdl)
        return outs

    def bytes_alg(self, args: list) -> int:
        """Compulsory HBM bytes of the path the last launch executed: every
        distinct input tensor the executed code reads, once, plus every
        output (counting only the selected arm's inputs)."""
        plan = self.plan
        vals = self.scalars()
        slot_of = plan.slot
        total = 0
        for ip in plan.inputs:
            t = args[ip.free_index]
            needed = False
            for p in range(plan.npass):
                nodes = plan._pass_nodes(p)
                if ip.node not in nodes:
                    continue
                dnf = plan._guards(p).get(ip.node.uid, frozenset({frozenset()}))
                for conj in dnf:
                    if all((vals[slot_of[uid]] != 0.0) == pol for uid, pol in conj):
                        needed = True
            if ip.node.kind == "dscalar":
                needed = True
            if needed:
                total += t.numel() * t.element_size()
        for j, kind, info, k in self.out_specs:
            if kind == "elem":
                total += int(torch.Size(self.shape).numel()) * torch.empty((), dtype=info).element_size()
        return total

    def timeline(self) -> list[int] | None:
        """GM_PROFILE builds: [start, pass0 end, pass0 barrier done, ...,
        end] in ns relative to the first CTA start (syncs; diagnostics)."""
        if not getattr(self.plan, "profiled", False):
            return None
        off = SCRATCH_PARTIALS + 8 * max(1, self.nred) * self.grid + 8 * 64
        v = self.scratch[off: off + 8 * 64].view(torch.int64).tolist()
        t0 = v[0]
        return [x - t0 if x and x < 2 ** 62 else 0 for x in v]

    def reset_timeline(self) -> None:
        off = SCRATCH_PARTIALS + 8 * max(1, self.nred) * self.grid + 8 * 64
        t = self.scratch[off: off + 8 * 64].view(torch.int64)
        t.zero_()
        t[0] = 2 ** 62
        t[32:40] = 2 ** 62   # per-pass earliest CTA finish (atomicMin)

    def spec_stats(self) -> tuple[int, int]:
        """(launches, mispredictions) of a speculative region (syncs; tests
        and bench)."""
        v = self.scratch[SCRATCH_STATS:SCRATCH_STATS + 16].view(torch.int64).tolist()
        return int(v[0]), int(v[1])

    def status(self) -> int:
        """Grid-barrier status word (syncs; diagnostics only)."""
        return int(self.scratch[16:20].view(torch.int32).item())

    def scalars(self) -> list[float]:
        """Scalar slots mirrored by CTA 0 of the last launch (syncs; tests)."""
        off = SCRATCH_PARTIALS + 8 * max(1, self.nred) * self.grid
        return self.scratch[off: off + 8 * self.nscal].view(torch.float64).tolist()


class Region:
    """One fused run of statements of a transformed forward."""

    def __init__(self, rid: int, name: str, graph: Graph, out_names: list[str], out_nodes: list[Node],
                 fallback, source: str):
        self.rid = rid
        self.name = name
        self.graph = graph
        self.out_names = out_names
        self.out_nodes = out_nodes
        self.fallback = fallback          # the original statements as a function
        self.source = source              # their text (for reports)
        self.specs: dict[tuple, object] = {}
        self.stats = RegionStats()
        self.last_spec: _Spec | None = None
        self.last_args: tuple | None = None
        # aot.py: when a list, every call's arguments are recorded here
        self.trace = None
        # optional (start, end) torch.cuda.Event(external=True) pair recorded
        # around the kernel launch; captured into a CUDA graph they time the
        # kernel inside every replay (bench.py's roofline measurement)
        self.probe = None

    def __call__(self, *args):
        if self.trace is not None:
            self.trace.append(args)
        key = tuple(arg_key(a) for a in args)
        spec = self.specs.get(key)
        if spec is None:
            spec = self._specialise(list(args))
            self.specs[key] = spec
        if isinstance(spec, str):
            self.stats.fallbacks += 1
            return self.fallback(*args)
        self.stats.launches += 1
        self.last_spec = spec
        self.last_args = args
        if self.probe is not None:
            self.probe[0].record()
        outs = spec.run(list(args))
        if self.probe is not None:
            self.probe[1].record()
        return outs[0] if len(outs) == 1 else tuple(outs)

    def _specialise(self, args: list):
        if not any(torch.is_tensor(a) and a.device.type == "cuda" for a in args):
            reason = "no CUDA tensor argument"
            self.stats.fallback_reasons.append(reason)
            return reason
        try:
            return _Spec(self, args)
        except Unsupported as exc:
            reason = str(exc)
            self.stats.fallback_reasons.append(reason)
            return reason

"""Runtime side of a fused region: specialisation cache, launch, scratch.

A `Region` is created by the lowering (lowering.py) for one run of fusable
statements.  Calling it with the region's free values launches one
NVRTC-compiled sm_100a kernel (codegen.py + csrc/gm_region.cuh) on the
current CUDA stream and returns the live-out tensors.  Launches are
stream-ordered and graph-capturable; no call synchronises with the host.

When the arguments leave the fusable subset (integer tensors, CPU tensors,
shapes that do not broadcast to one iteration space, ...), the call raises
`RegionUnsupported` — there is no silent fallback.  A caller that opts in
(`allow_eager=True`: `lowering.load(..., allow_eager=True)`, the CPU
equivalence tests) gets the region's original statements run with PyTorch
instead — the exact code the reference transform emitted (`fallback`), on
the device the tensors live on; every such decision is recorded in
`Region.stats`.  Missing native code is never a fallback: a NativeError
propagates.
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
from .ir import Graph, Node, Unsupported, fold_host_predicates
from .rowgen import RowPlan, has_row_ops
from .split import is_mixed
from .split import split as split_graph

SCRATCH_PARTIALS = 2432  # GM_SCRATCH_PARTIALS in csrc/gm_region.cuh
SCRATCH_STATS = 32      # GM_SCRATCH_STATS: u64 [launches, mispredictions, exact entries]
SCRATCH_CONF = 56       # GM_SCRATCH_CONF: int prediction confidence (adaptive speculation)
SCRATCH_FORCE = 60      # GM_SCRATCH_FORCE: diagnostics (flip decisions / force an entry)
FORCE_EXACT, FORCE_SPEC = 1 << 30, -(1 << 31)   # bits 30 / 31 of the (int32) force word
LIVE_BIT = 1 << 29      # bit 29: the grid kernels' live timer (GM_SCRATCH_LIVE)
SCRATCH_LIVE = 256      # GM_SCRATCH_LIVE: u64 [start ns, exits, sum of durations ns, launches]
SCRATCH_PRED = 288      # GM_SCRATCH_PRED: int predicted decisions
SCRATCH_SUBCNT = 384    # GM_SCRATCH_SUBCNT: arrival sub-counters
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


class RegionUnsupported(nat.NativeError):
    """The region's arguments leave the fused subset and the caller did not
    opt into running its statements with PyTorch (allow_eager)."""


_owner = threading.local()


class scratch_owner:
    """Context manager: launches inside it key their scratch by `owner`
    instead of by (stream, capture id).  B200Executor runs its last warm-up
    AND its capture under the entry as owner, so every buffer the captured
    graph uses is allocated and zeroed eagerly before the capture starts
    (nothing is allocated or filled while the stream captures) and belongs
    to that graph alone."""

    def __init__(self, owner):
        self.owner = owner

    def __enter__(self):
        self.prev = getattr(_owner, "v", None)
        _owner.v = self.owner
        return self

    def __exit__(self, *exc):
        _owner.v = self.prev
        return False


def stream_key(dev: torch.device) -> tuple:
    """The owner of a scratch buffer: the active scratch_owner, else
    (stream, capture id) of the current stream.  Eager launches on one
    stream are ordered; every CUDA-graph capture gets its own key, so two
    graphs (or two streams) replaying the same specialisation never share an
    arrival counter."""
    o = getattr(_owner, "v", None)
    if o is not None:
        return ("owner", id(o))
    s = torch.cuda.current_stream(dev).cuda_stream
    return s, nat.capture_id(s)


SLAB_BYTES = 16 << 20
_slabs: dict = {}


def _slab_take(nbytes: int, dev: torch.device) -> torch.Tensor | None:
    """A zeroed piece of the per-device slab (allocated and zeroed outside
    any capture by the first region specialisation)."""
    sl = _slabs.get(dev.index)
    if sl is None:
        return None
    t, off = sl
    n = (nbytes + 255) // 256 * 256
    if off + n > t.numel():
        return None
    _slabs[dev.index] = (t, off + n)
    return t[off: off + nbytes]


def ensure_slab(dev: torch.device) -> None:
    if dev.index not in _slabs and not torch.cuda.is_current_stream_capturing():
        _slabs[dev.index] = (torch.zeros(SLAB_BYTES, dtype=torch.uint8, device=dev), 0)


def zeroed(nbytes: int, dev: torch.device) -> torch.Tensor:
    """A zero-filled device buffer.  While the current stream captures a CUDA
    graph nothing may be allocated or filled outside it: small buffers come
    from the pre-zeroed slab; larger ones must have been created by an eager
    run under the same scratch_owner (B200Executor does this)."""
    if torch.cuda.is_current_stream_capturing():
        t = _slab_take(nbytes, dev)
        if t is None:
            raise nat.NativeError(
                f"a {nbytes}-byte scratch buffer is first needed inside a CUDA-graph capture; run the forward once "
                "eagerly under region.scratch_owner(<graph owner>) before capturing (B200Executor does)")
        return t
    return torch.zeros(nbytes, dtype=torch.uint8, device=dev)


# every (spec, scratch, status word) ever handed to a launch: check_status()
# reads their status words from the mapped page without synchronising
_status_owners: list = []


def _status_slot() -> int:
    n = len(_status_owners)
    if n >= nat.STATUS_WORDS:
        raise nat.NativeError("out of region status words")
    return n


def check_status() -> None:
    """Raise if any region launch hit the grid-barrier timeout (status = 1:
    CTAs were not co-resident, so partials may have been stale and the
    outputs of that launch are wrong).  Non-blocking when all is well (a read
    of mapped host memory); on an error the device is synchronised, the
    affected counters and status words are reset, and NativeError names the
    regions."""
    if not _status_owners:
        return
    page, _ = nat.status_page()
    bad = [o for o in _status_owners if page[o[2]]]
    if not bad:
        return
    torch.cuda.synchronize()
    names = []
    for spec, t, idx in bad:
        t[:SCRATCH_STATS].zero_()
        t[SCRATCH_SUBCNT:SCRATCH_PARTIALS].zero_()
        page[idx] = 0
        names.append(spec.name)
    torch.cuda.synchronize()
    raise nat.NativeError(f"grid-barrier timeout in region(s) {sorted(set(names))}: the CTAs were not co-resident; "
                          "the outputs of those launches are invalid (counters reset)")


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
        graph, outs = fold_host_predicates(region.graph, region.out_nodes, args)
        if any(o.op == "const" for o in outs):
            raise Unsupported("a live-out folds to a host constant")
        plan_cls = RowPlan if has_row_ops(outs) else Plan
        plan = plan_cls(graph, outs, args, name=region.name, device_info=(sms, smem_optin))
        self.plan = plan
        self.kernel = compiled_kernel(plan.source, plan.kernel)
        n = plan.n
        nvec = -(-n // nat.VEC) if n else 0
        threads = plan.threads
        grid, smem = plan.grid, plan.smem_bytes
        vpc = plan.K
        if getattr(plan, "persist", False):
            # a persistent row kernel loops over its row groups: one wave
            grid = max(1, min(grid, self.kernel.occupancy(threads, smem) * sms))
        if plan.reductions and grid > 1:
            # the grid barrier needs every CTA resident at once
            occ = self.kernel.occupancy(threads, smem)
            if occ * sms < grid:
                raise nat.NativeError(f"region {region.name}: {grid} CTAs not co-resident "
                                      f"({occ}/SM at {smem} B smem, {sms} SMs)")
        self.grid, self.vpc, self.smem, self.threads = grid, vpc, smem, threads
        self.nred = len(plan.reductions) + plan.extra_slots()
        self.nscal = len(plan.scalars)
        # scratch: counter/epoch/status/results (192 B, see gm_region.cuh) |
        # partials | scalar mirror (+1 KB: the GM_PROFILE timeline at scal_out + 64 u64);
        # one buffer per (stream, graph capture), see stream_key()
        part_bytes = 8 * max(1, self.nred) * grid
        self.part_bytes = part_bytes
        self.scratch_bytes = SCRATCH_PARTIALS + part_bytes + 8 * 64 + 8 * 64 + 8 * max(1, self.nscal)
        self.name = region.name
        self._scratches: dict = {}
        self.scratch: torch.Tensor | None = None
        self.status_idx = -1
        ensure_slab(dev)
        self.bind_scratch()
        P = nat.Params()
        P.n = n
        P.nvec = nvec
        P.vpc = vpc
        P.piece_vecs = 1  # (bulk-copy staging: gm_branch_select_f32 only)
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
                self.out_specs.append((j, "elem", (o.dtype, tuple(o.shape)), k))
                k += 1
            else:
                self.out_specs.append((j, "scalar", o.dtype, k))
                k += 1
        self.shape = tuple(plan.shape)

    def bind_scratch(self) -> torch.Tensor:
        """The scratch buffer of the current (stream, capture) — created
        zeroed on first use — made the one `scalars()` / `spec_stats()` read."""
        key = stream_key(self.device)
        sc = self._scratches.get(key)
        if sc is None:
            t = zeroed(self.scratch_bytes, self.device)
            idx = _status_slot()
            _status_owners.append((self, t, idx))
            sc = (t, idx)
            self._scratches[key] = sc
        self.scratch, self.status_idx = sc
        return self.scratch

    def run(self, args: list, pdl: bool | None = None):
        """Launch on the current stream.  `pdl` (default: GM_PDL, on) makes it
        a programmatic dependent launch: the CTAs become resident while the
        previous kernel drains and wait (griddepcontrol.wait) for its results
        before reading anything."""
        P = nat.Params()
        ctypes.memmove(ctypes.byref(P), ctypes.byref(self.template), ctypes.sizeof(P))
        base = self.bind_scratch().data_ptr()
        P.barrier = base
        P.status = nat.status_page()[1] + 4 * self.status_idx
        P.partials = base + SCRATCH_PARTIALS
        P.scal_out = base + SCRATCH_PARTIALS + self.part_bytes
        for slot, fi in self.in_slots:
            P.inp[slot].ptr = args[fi].data_ptr()
        for j, fi in enumerate(self.hs_index):
            P.hs[j] = float(args[fi])
        outs = [None] * len(self.out_specs)
        for j, kind, info, k in self.out_specs:
            if kind == "alias":
                outs[j] = args[info]
            elif kind == "elem":
                t = torch.empty(info[1], dtype=info[0], device=self.device)
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
                total += int(torch.Size(info[1]).numel()) * torch.empty((), dtype=info[0]).element_size()
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
        and bench).  Launches count both entries; see exact_entries()."""
        v = self.scratch[SCRATCH_STATS:SCRATCH_STATS + 16].view(torch.int64).tolist()
        return int(v[0]), int(v[1])

    def force(self, word: int) -> None:
        """Diagnostics: set the force word of the current scratch (bit j flips
        predicted decision j; FORCE_EXACT / FORCE_SPEC pick the entry); 0
        restores normal operation.  Stream-ordered, no sync."""
        self.scratch[SCRATCH_FORCE:SCRATCH_FORCE + 4].view(torch.int32).fill_(int(word))

    def set_live(self, on: bool) -> None:
        """Turn the in-kernel live timer on (zeroing its sums) or off in every
        scratch of this specialisation (each graph capture has its own).
        Grid-region kernels only; stream-ordered, no sync."""
        for t, _idx in self._scratches.values():
            word = t[SCRATCH_FORCE:SCRATCH_FORCE + 4].view(torch.int32)
            if on:
                t[SCRATCH_LIVE:SCRATCH_LIVE + 32].zero_()
                word.bitwise_or_(LIVE_BIT)
            else:
                word.bitwise_and_(~LIVE_BIT)

    def live_stats(self) -> tuple[int, int]:
        """(sum of kernel durations in ns, launches) the live timer recorded
        since set_live(True), over every scratch (syncs)."""
        tot, n = 0, 0
        for t, _idx in self._scratches.values():
            v = t[SCRATCH_LIVE:SCRATCH_LIVE + 32].view(torch.int64).tolist()
            tot += int(v[2])
            n += int(v[3])
        return tot, n

    def exact_entries(self) -> int:
        """Launches of a speculative region that took the exact entry (the
        confidence counter was below codegen.SPEC_CONFIDENT; syncs)."""
        return int(self.scratch[SCRATCH_STATS + 16:SCRATCH_STATS + 24].view(torch.int64).item())

    def status(self) -> int:
        """Grid-barrier status word of the current scratch (a read of mapped
        host memory: no sync; the launch it reports on may still be running)."""
        return int(nat.status_page()[0][self.status_idx])

    def scalars(self) -> list[float]:
        """Scalar slots mirrored by CTA 0 of the last launch (syncs; tests)."""
        off = SCRATCH_PARTIALS + 8 * max(1, self.nred) * self.grid
        return self.scratch[off: off + 8 * self.nscal].view(torch.float64).tolist()


class _SubRegion:
    """The graph of one kernel of a split region (split.py)."""

    def __init__(self, name: str, graph: Graph, outs: list[Node]):
        self.name, self.graph, self.out_nodes = name, graph, outs


class _SplitSpec:
    """A region over several iteration spaces (split.py): the side kernels
    run first and append their results to the argument list, then the main
    kernel.  Looks like the main kernel's _Spec to the bench and the tests
    (`plan`, `spec_stats`, `scalars`, ...); launch-wide queries (bytes,
    live timer) cover every kernel."""

    def __init__(self, region: "Region", graph: Graph, outs: list[Node], args: list, depth: int = 0):
        if depth > 8:
            raise Unsupported("shape split nested too deep")
        steps, (mg, mouts) = split_graph(graph, outs, args)
        ext = list(args)
        self.sides = []
        for i, (sg, souts, idx) in enumerate(steps):
            sub = _SubRegion(f"{region.name}/side{i}", sg, souts)
            sp = _SplitSpec(sub, sg, souts, ext, depth + 1) if is_mixed(sg, souts, ext) else _Spec(sub, ext)
            self.sides.append((sp, idx))
            probe = _probe_value(souts[0], ext)
            ext.append(probe)
        self.main = _Spec(_SubRegion(region.name, mg, mouts), ext)
        self.nargs = len(args)

    def __getattr__(self, name):
        return getattr(self.main, name)

    def run(self, args: list, pdl: bool | None = None):
        ext = list(args)
        for sp, _idx in self.sides:
            ext.append(sp.run(list(ext), pdl)[0])
        self._last_ext = ext
        return self.main.run(ext, pdl)

    _last_ext: list | None = None

    def all_specs(self):
        for sp, _ in self.sides:
            yield from (sp.all_specs() if isinstance(sp, _SplitSpec) else [sp])
        yield self.main

    def bytes_alg(self, args: list) -> int:
        """Every kernel's compulsory bytes (side results count as written by
        their kernel and read by the main one)."""
        ext = self._last_ext or list(args)
        total = 0
        for k, (sp, _idx) in enumerate(self.sides):
            total += sp.bytes_alg(ext[:self.nargs + k])
        return total + self.main.bytes_alg(ext)

    def set_live(self, on: bool) -> None:
        for sp in self.all_specs():
            sp.set_live(on)

    def live_stats(self) -> tuple[int, int]:
        tot, n = 0, 0
        for sp in self.all_specs():
            t, k = sp.live_stats()
            tot += t
            n = max(n, k)
        return tot, n


def _probe_value(node: Node, args: list):
    """A stand-in with the dtype / shape / device of a side result, so the
    main kernel is specialised for it (the real tensor arrives at run time;
    the specialisation key of the region covers its inputs only)."""
    dev = next(a.device for a in args if torch.is_tensor(a) and a.device.type == "cuda")
    return torch.empty(tuple(node.shape), dtype=node.dtype, device=dev)


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
        # run the original statements with PyTorch when specialisation fails
        # (opt-in; the default raises RegionUnsupported)
        self.allow_eager = False

    def __call__(self, *args):
        if self.trace is not None:
            self.trace.append(args)
        key = tuple(arg_key(a) for a in args)
        spec = self.specs.get(key)
        if spec is None:
            spec = self._specialise(list(args))
            self.specs[key] = spec
        if isinstance(spec, str):
            if not self.allow_eager:
                raise RegionUnsupported(f"region {self.name}: {spec} (the fused kernel cannot run these arguments; "
                                        f"load the program with allow_eager=True to run its statements with "
                                        f"PyTorch)")
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
            graph, outs = fold_host_predicates(self.graph, self.out_nodes, args)
            if is_mixed(graph, outs, args):
                return _SplitSpec(self, graph, outs, args)
            return _Spec(self, args)
        except Unsupported as exc:
            reason = str(exc)
            self.stats.fallback_reasons.append(reason)
            return reason

"""Bench: forward latency / throughput of a GraphMend-transformed program on
the B200 path (BASELINE.json metric; config 2 = BigBird-like layer, seq 1024,
batch 8, fp32 — the reference harness's own precision, runner.py:114-125 —
random-init weights, synthetic inputs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--dtype fp32|bf16]
    python bench.py --impl reference ...     # the reference's CPU path on the host cores

A step = one forward of the transformed program over one batch.  The
manifest's inputs (bigbird_like: seeds 63 / 61 / 62, whose branch decisions
differ) ROTATE through every timed loop, so speculation is measured with
changing decisions and the hit rate is reported.  `value` is whole-job
samples/s with inputs resident in HBM (graph replay only, device timed per
step with CUDA events, L2 flushed between steps); `e2e` is the same forward
through the public API (B200Executor) from pinned host buffers with the H2D
input copy and D2H output read inside the timed region.  `compile` is the
north_star comparator: the UNTRANSFORMED program under torch.compile
(default and reduce-overhead) on the same GPU and inputs.  Multi-GPU:
independent replicas (every predicate is a global reduction, so
the path does not shard), one process per GPU, gloo only for the timing
barrier and the max over ranks — no NCCL.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "p50 forward latency (ms) & samples/s per model; host syncs per forward"
WORKLOADS = {
    "bigbird_like": ("config 2: BigBird-RoBERTa-base-shaped layer, seq 1024, batch 8", None),
    "bart_step": ("config 4: BART-base-shaped decoder step, batch 32", None),
    "gemm_arms": ("config 2 variant: BigBird-shaped layer whose predicated arms each hold a GEMM", None),
    "bigbird_attn": ("config 2 with attention: BigBird-RoBERTa-base-shaped self-attention, 12 heads, "
                     "block-sparse / full softmax over [8,12,1024,1024] scores", None),
    "bigbird_layer": ("config 2 as a full encoder layer: BigBird-RoBERTa-base-shaped attention + FFN 3072 + "
                      "post-LayerNorms + GELU, block-sparse / full softmax", None),
    "phi4_like": ("config 5: corpus phi4_like at [8,1024,768]", [[8, 1024, 768]]),
    "qwen_audio_like": ("config 5: corpus qwen_audio_like at [8,1024,768]", [[8, 1024, 768]]),
    "longformer_like": ("config 3: corpus longformer_like at [4,4096,768]", [[4, 4096, 768]]),
    "biogpt_like": ("config 5: corpus biogpt_like at [8,1024,768]", [[8, 1024, 768]] * 2),
    "blenderbot_like": ("config 5: corpus blenderbot_like at [8,1024,768]", [[8, 1024, 768]]),
    "flan_t5_like": ("config 5: corpus flan_t5_like, [8192,768] @ [768,768]", [[8192, 768], [768, 768]]),
    "pegasus_like": ("config 5: corpus pegasus_like at [8,1024,768]", [[8, 1024, 768]]),
    "moe_minicpm_like": ("config 5: corpus moe_minicpm_like at [8,1024,768]", [[8, 1024, 768]]),
}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self) -> dict:
        rows = [r for r in self.rows if len(r) >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def max_over_ranks(x: float, dist_mod) -> float:
    """Max of a per-rank duration across replicas (gloo all-reduce MAX of a
    1-element CPU tensor: plumbing for the timing, not a data-path
    collective; no NCCL)."""
    if dist_mod is None or not dist_mod.is_initialized() or dist_mod.get_world_size() == 1:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    dist_mod.all_reduce(t, op=dist_mod.ReduceOp.MAX)
    return float(t)


def replica_value(batch: int, steps: int, world: int, max_seconds: float) -> float:
    """Whole-job samples/s of `world` independent replicas."""
    return world * batch * steps / max_seconds


def _ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu summary
    (profiles/*_ncu_regions.json, one `ncu --set full` capture), or None."""
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_regions.json"))):
        try:
            with open(path) as fh:
                rows = json.load(fh)
        except (OSError, ValueError):
            continue
        vals = [r["traffic_bytes"] for r in rows if r.get("kernel") == kernel and "traffic_bytes" in r]
        if vals:
            best = sum(vals) / len(vals)
    return best


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _transform_ms(workload: str):
    """The reference fix_file's one-time cost for this program (measured in
    the build container by oracle/time_transform.py; the reference is not on
    the GPU box)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "transform_times.json")) as fh:
            return json.load(fh)["ms"].get(workload)
    except (OSError, ValueError, KeyError):
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def _all_inputs(prog, shapes, dtype):
    """Every manifest input (runner.py:114-125 draws), in manifest order."""
    from paper_2509_16248_b200.harness import make_args

    return [make_args(spec["args"], spec["seed"], dtype, shapes) for spec in prog["inputs"]]


def _config(args, x0) -> dict:
    """Identical in both arms (the driver compares them)."""
    prog_inputs = _programs()[args.workload]["inputs"]
    return {"workload": f"{args.workload} ({WORKLOADS[args.workload][0]})", "batch": int(x0.shape[0]),
            "shape": list(x0.shape),
            "inputs": "manifest draws rotated every step: " + ", ".join(
                f"seed {sp['seed']} ({sp.get('note', '')})" for sp in prog_inputs)}


def _programs():
    from paper_2509_16248_b200.harness import programs

    return programs()


def _cpu_rate(prog, xs, dtype, budget_s: float, max_forwards: int = 100000):
    """The reference's CPU path — the reference-transformed program executed
    eagerly on CPU in the harness call shape (runner.py:154-157), all host
    threads — over the rotating inputs for `budget_s` seconds.
    Returns (samples/s, forwards, p50 ms, threads)."""
    import torch

    from oracle import executor as orc

    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    fn = orc.reference_callable(prog["transformed"], prog["callable"], dtype)
    orc.call_captured(fn, xs[0])
    times = []
    t_end = time.perf_counter() + budget_s
    k = 0
    while (time.perf_counter() < t_end or not times) and len(times) < max_forwards:
        t0 = time.perf_counter()
        orc.call_captured(fn, xs[k % len(xs)])
        times.append(time.perf_counter() - t0)
        k += 1
    batch = int(xs[0][0].shape[0])
    return batch * len(times) / sum(times), len(times), 1e3 * statistics.median(times), threads


def run_reference(args, ws, rank):
    """`--impl reference`: the reference's CPU path on the box's host cores,
    rank 0 only (the other ranks exit without work).  Each of the K timed
    steps is a bounded sample: eager forwards over the rotating inputs for
    ~30 s / K (of a sub-batch when one full-batch forward exceeds that), so
    the whole run is a ~30 s window."""
    if rank != 0:
        return
    import torch

    dtype = {"bf16": torch.bfloat16, "fp32": torch.float32}[args.dtype]
    prog = _programs()[args.workload]
    xs = _all_inputs(prog, WORKLOADS[args.workload][1], dtype)
    from oracle import executor as orc

    fn = orc.reference_callable(prog["transformed"], prog["callable"], dtype)
    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    batch = int(xs[0][0].shape[0])
    # size each step's sample: a forward of the whole batch when it fits the
    # step's share of the ~10 s window, else of its first `sub` samples (the
    # same program on the same data, fewer rows) — so a slow CPU forward
    # (the full bigbird_layer is ~2 s on 16 cores) keeps the run to minutes
    orc.call_captured(fn, xs[0])                 # first call: lazy initialisation
    t0 = time.perf_counter()
    orc.call_captured(fn, xs[1 % len(xs)])
    t_full = time.perf_counter() - t0
    per_step = 30.0 / max(1, args.steps)         # a ~30 s window over the K steps
    sub = max(1, min(batch, int(batch * per_step / max(t_full, 1e-9))))
    xsub = [[t[:sub] if torch.is_tensor(t) and t.dim() and t.shape[0] == batch else t for t in x] for x in xs]
    for k in range(args.warmup):
        orc.call_captured(fn, xsub[k % len(xsub)])
    total_s, forwards, step_ms, fwd_ms = 0.0, 0, [], []
    k = 0
    for _ in range(args.steps):
        t_step = time.perf_counter()
        while True:
            t0 = time.perf_counter()
            orc.call_captured(fn, xsub[k % len(xsub)])
            fwd_ms.append(1e3 * (time.perf_counter() - t0))
            k += 1
            forwards += 1
            if time.perf_counter() - t_step >= per_step:
                break
        dt = time.perf_counter() - t_step
        total_s += dt
        step_ms.append(1e3 * dt)
    value = sub * forwards / total_s
    p50s = [statistics.median(fwd_ms) * batch / sub]   # per full-batch forward
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(step_ms),
        "p50_ms": statistics.median(p50s), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": DATA,
        "config": _config(args, xs[0][0]),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
                         "cpu_model": _cpu_model(),
                         "sample": f"{args.steps} steps x ~{per_step:.2f} s: {forwards} eager forwards of the "
                                   f"reference-transformed program on {sub} of the batch's {batch} samples of the "
                                   f"rotating manifest inputs, torch CPU, {threads} threads"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


DATA = "synthetic inputs (manifest seeds/dists at the BASELINE shape, rotated), random-init weights (seed 0)"


def cpu_baseline(prog, shapes, dtype, budget_s=10.0):
    """Bounded CPU-oracle sample on the box's host cores (rank 0, N=1)."""
    import torch

    xs = _all_inputs(prog, shapes, dtype)
    v, n, p50, threads = _cpu_rate(prog, xs, dtype, budget_s)
    return {"value": v, "unit": "samples/s", "cores": threads, "kind": "port", "cpu_model": _cpu_model(),
            "sample": f"{n} eager forwards of the reference-transformed program over the rotating manifest inputs "
                      f"(~{budget_s:.0f} s), torch CPU, {threads} threads; p50 {p50:.2f} ms"}


def _wall_p50(fn, xs, iters: int, warm: int = 3) -> float:
    """p50 wall-clock ms of fn(*x) + synchronize, inputs rotating."""
    import torch

    for k in range(warm):
        fn(*xs[k % len(xs)])
    torch.cuda.synchronize()
    ts = []
    for k in range(iters):
        x = xs[k % len(xs)]
        t0 = time.perf_counter()
        fn(*x)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts)


def compile_comparator(prog, dtype, xs_dev, ex, iters: int) -> dict:
    """north_star's comparator: the UNTRANSFORMED original program under
    torch.compile (Inductor; default and reduce-overhead), same GPU, weights
    (seed 0) and rotating inputs, vs the B200 user-facing call
    (B200Executor(*device inputs): input copy + graph replay).  p50 of wall
    clock around a synchronised call; inference (no_grad) on both sides."""
    import logging

    import torch

    from oracle import executor as orc

    res = {"how": "p50 wall clock of call + cuda.synchronize, device-resident rotating inputs, warm; "
                  "untransformed original under torch.compile vs B200Executor(*inputs) on the transformed text"}
    logging.disable(logging.CRITICAL)
    try:
        with torch.no_grad():
            res["b200_call_p50_ms"] = _wall_p50(lambda *a: ex(*a), xs_dev, iters)
            ex.flush()
            for mode in ("default", "reduce-overhead"):
                torch._dynamo.reset()
                try:
                    fn = orc.reference_callable(prog["original"], prog["callable"], dtype)
                    if isinstance(fn, torch.nn.Module):
                        fn.to(xs_dev[0][0].device)
                    c = torch.compile(fn, mode=None if mode == "default" else mode)
                    t0 = time.perf_counter()
                    for x in xs_dev:
                        c(*x)
                    torch.cuda.synchronize()
                    res[f"{mode}_cold_ms"] = 1e3 * (time.perf_counter() - t0)
                    res[f"{mode}_p50_ms"] = _wall_p50(c, xs_dev, iters)
                except Exception as exc:  # report, keep the bench line
                    res[f"{mode}_error"] = repr(exc)[:300]
            torch._dynamo.reset()
    finally:
        logging.disable(logging.NOTSET)
    if res.get("default_p50_ms"):
        res["speedup_vs_compile"] = res["default_p50_ms"] / res["b200_call_p50_ms"]
    if res.get("reduce-overhead_p50_ms"):
        res["speedup_vs_compile_reduce_overhead"] = res["reduce-overhead_p50_ms"] / res["b200_call_p50_ms"]
    return res


def profile_syncs(ex, x_dev) -> dict:
    """torch.profiler count, inside one user-facing forward, of host-blocking
    CUDA calls and device-to-host copies."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    from torch.profiler import record_function

    ex(*x_dev)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        with record_function("gm_forward"):
            ex(*x_dev)
    torch.cuda.synchronize()
    evs = list(prof.events())
    fwd = [e for e in evs if e.name == "gm_forward"]
    lo, hi = fwd[0].time_range.start, fwd[0].time_range.end
    inside = [e for e in evs if e.device_type == torch.autograd.DeviceType.CPU
              and lo <= e.time_range.start <= hi]
    syncs = sum(1 for e in inside
                if e.name in ("cudaStreamSynchronize", "cudaDeviceSynchronize", "cudaEventSynchronize"))
    d2h = sum(1 for e in evs if ("DtoH" in e.name or "Device -> Pinned" in e.name or "Device -> Pageable" in e.name))
    return {"cuda_syncs": syncs, "d2h_copies": d2h, "how": "torch.profiler over one B200Executor call "
            "(device inputs): cudaStream/Device/EventSynchronize calls whose CPU start lies inside the "
            "forward's record_function range (the profiler's own stop-time cudaDeviceSynchronize is "
            "outside it), and DtoH memcpy events anywhere in the trace"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="bigbird_layer", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="fp32", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compile", action="store_true", help="skip the torch.compile comparator")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws, rank, local = _dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch

    from paper_2509_16248_b200 import compile_program, gemm
    from paper_2509_16248_b200.region import scratch_owner

    # one replica per GPU; on a box with fewer GPUs than ranks (the 1-GPU
    # test box) replicas share devices round-robin
    gpu = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    pg = None
    if ws > 1:
        # replicas only: gloo carries the timing barrier and the max over
        # ranks (CPU tensors) — there is no NCCL and no data-path collective
        import torch.distributed as dist

        dist.init_process_group("gloo")
        pg = dist
    dtype = {"bf16": torch.bfloat16, "fp32": torch.float32}[args.dtype]
    prog = _programs()[args.workload]
    shapes = WORKLOADS[args.workload][1]
    xs_host = [[t.pin_memory() for t in x] for x in _all_inputs(prog, shapes, dtype)]
    xs_dev = [[t.to(dev) for t in x] for x in xs_host]
    R = len(xs_host)
    batch = int(xs_host[0][0].shape[0])

    t0 = time.perf_counter()
    ex, mod, low = compile_program(prog["transformed"], prog["callable"], device=dev, dtype=dtype)
    entry = ex.prepare(*xs_dev[0])
    torch.cuda.synchronize(dev)
    cold_ms = 1e3 * (time.perf_counter() - t0)
    # the program's own regions and the row regions behind its module calls
    # (nn.LayerNorm, gemm.module_call)
    from paper_2509_16248_b200 import gemm as gemm_

    all_regions = list(low.regions) + gemm_.module_regions(getattr(mod, prog["callable"], None))
    info = entry.info
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    flush_rd = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.int64, device=dev)

    def flush_l2():
        """Write 256 MB (evicts everything), then read another 256 MB so the
        L2 holds only clean lines of the flush buffers: the next step starts
        cold and does not pay the flush's write-backs."""
        flush_buf.zero_()
        flush_rd.sum()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize(dev)

    def spec_totals():
        tot = [0, 0, 0]
        for r in all_regions:
            sp = r.last_spec
            if sp is not None and sp.plan.spec:
                a, b = sp.spec_stats()
                tot[0] += a
                tot[1] += b
                tot[2] += sp.exact_entries()
        return tot

    # ---- device-timed replay (inputs resident in HBM, rotating): before
    #      each step the step's input is copied into the graph's static
    #      buffers and the L2 is flushed, both outside the timed window
    for k in range(args.warmup):
        entry.load(xs_dev[k % R])
        entry.run()
    ex.flush()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    with ClockSampler(gpu) as clocks:
        # keep the GPU busy (untimed replays) until nvidia-smi has sampled it
        # under load, so the clock record covers the timed region
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.0 or len(clocks.rows) < 3:
            for _ in range(50):
                entry.run()
            torch.cuda.synchronize(dev)
            if time.perf_counter() - t_load > 5.0:
                break
        barrier()
        spec0 = spec_totals()
        fused_specs = [r.last_spec for r in all_regions if r.last_spec is not None]
        for sp in fused_specs:
            sp.set_live(True)        # grid kernels time themselves inside the graph
        for i in range(args.steps):
            entry.load(xs_dev[i % R])
            flush_l2()
            starts[i].record(stream)
            entry.run()
            ends[i].record(stream)
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    live_timer = {}
    for r in all_regions:
        if r.last_spec is not None:
            tot, n = r.last_spec.live_stats()
            r.last_spec.set_live(False)
            if n:
                live_timer[id(r)] = (tot / n / 1e6, n)
    spec1 = spec_totals()
    ex.flush()
    total_ms = max_over_ranks(sum(step_ms), pg)
    value = replica_value(batch, args.steps, ws, total_ms / 1e3)
    speculation = {"launches": spec1[0] - spec0[0], "mispredictions": spec1[1] - spec0[1],
                   "exact_entries": spec1[2] - spec0[2],
                   "how": f"speculative region launches in the timed loop, inputs rotating over {R} manifest draws"}
    if speculation["launches"]:
        speculated = speculation["launches"] - speculation["exact_entries"]
        speculation["speculated"] = speculated
        speculation["hit_rate"] = (1.0 - speculation["mispredictions"] / speculated) if speculated else None

    # ---- each fused kernel timed on its own stream, cold L2: a CUDA graph of
    #      R x [256 MB L2 flush, region launch] minus a graph of R x [flush],
    #      both replayed between CUDA events (no host work inside the window)
    fused = [r for r in all_regions if r.last_spec is not None]
    live = _live_kernel_ms(ex, fused, xs_dev, flush_l2, dev, args.steps)
    kernels = []
    for r in fused:
        spec = r.last_spec
        nbytes = spec.bytes_alg(list(r.last_args))
        if id(r) in live_timer:
            ms, how = live_timer[id(r)][0], (
                f"live, in-kernel: %globaltimer from CTA 0's start (after griddepcontrol.wait) to the last CTA's "
                f"exit, summed by the kernel over the {live_timer[id(r)][1]} launches of the timed loop itself, mean")
        else:
            ms, how = live.get(id(r), float("nan")), (
                "live: CUDA events captured around the launch inside the forward's graph, replayed over the "
                "rotating inputs with the L2 flushed before every step (the timed loop's conditions), mean")
        k = {"name": f"{spec.plan.kernel} ({r.name})", "ms": ms,
             "bytes": nbytes, "grid": spec.grid, "smem": spec.smem,
             "passes": spec.plan.npass, "speculative": spec.plan.spec,
             "how": how, "ms_events": live.get(id(r), float("nan")),
             "ms_isolated": _time_kernel_flushed(spec, list(r.last_args), flush_l2, dev),
             "isolated_how": "graph of 20 x (L2 flush + launch) minus 20 x flush; cold L2; one input"}
        if spec.plan.spec:
            k["ms_isolated"] = k["ms_isolated"]
            k["ms_spec_hit"] = k.pop("ms_isolated")
            k["ms_spec_miss"] = _time_kernel_flushed(spec, list(r.last_args), flush_l2, dev, mode="miss")
            k["ms_exact_entry"] = _time_kernel_flushed(spec, list(r.last_args), flush_l2, dev, mode="exact")
        kernels.append(k)
    dom = max(kernels, key=lambda k: k["ms"]) if kernels else None
    peak, peak_kind = _peaks()
    roofline = None
    if dom:
        achieved = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": _ncu_traffic(dom["name"].split(" ")[0]), "kernel": dom["name"],
                    "bytes_alg": dom["bytes"], "kernel_ms": dom["ms"],
                    "peak_kind": peak_kind, "share_of_step": dom["ms"] / statistics.mean(step_ms),
                    "traffic_how": "ncu dram__bytes_read+write per launch from the committed profiles/ capture",
                    # also against north_star's nominal 8 TB/s
                    "frac_nominal_8tbs": achieved / 8000.0,
                    "fused_kernels_frac": {k["name"].split(" ")[0]: round(k["bytes"] / (k["ms"] / 1e3) / 1e9 / peak, 3)
                                           for k in kernels if k["ms"] == k["ms"] and k["ms"] > 0}}

    # ---- end to end through the public API, host buffers in and out:
    # (a) single call latency: executor(*pinned host inputs) -> D2H into a
    #     pinned host tensor, synchronised; (b) throughput: the executor's
    #     pipelined host path (H2D / forward / D2H overlapped, 3 graph slots),
    #     inputs rotating so each slot's graph sees changing decisions
    h2d = sum(t.numel() * t.element_size() for t in xs_host[0])
    out0 = ex(*xs_host[0])
    out_pinned = torch.empty(out0.shape, dtype=out0.dtype, pin_memory=True)
    e2e_ms = []
    for i in range(args.steps + 3):
        e0 = time.perf_counter()
        out = ex(*xs_host[i % R])
        out_pinned.copy_(out, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        if i >= 3:
            e2e_ms.append(1e3 * (time.perf_counter() - e0))
    ex.flush()
    S = 3
    host_batches = [tuple(xs_host[(k // S) % R]) for k in range(args.steps)]
    # results land in a ring of 8 pinned host buffers (step k -> buffer k % 8:
    # the D2H copies into one buffer are ordered on the copy stream), so N
    # replicas do not pin N x steps x the output of host memory
    ring = [torch.empty(out0.shape, dtype=out0.dtype, pin_memory=True) for _ in range(min(8, args.steps))]
    outs = [ring[k % len(ring)] for k in range(args.steps)]
    ex.run_host_pipelined(host_batches[:4], out=outs[:4], slots=S)  # build the graph slots, warm
    ex.flush()
    barrier()
    t_e2e = time.perf_counter()
    ex.run_host_pipelined(host_batches, out=outs, slots=S)
    barrier()
    e2e_total = max_over_ranks(time.perf_counter() - t_e2e, pg)
    # the same pipelined H2D / D2H traffic with no forward: the PCIe
    # bound the end-to-end number sits against
    pcie_s = _copy_only_pipeline(list(host_batches[0]), outs, dev, args.steps)
    ex.flush()
    d2h = out_pinned.numel() * out_pinned.element_size()

    # our kernels per step, counted at their launch calls over one eager
    # forward (the graph replays what its capture launched)
    from paper_2509_16248_b200 import _native as nat_

    import contextlib
    import io
    import logging

    c0 = nat_.launch_count
    logging.disable(logging.CRITICAL)
    try:
        with torch.no_grad(), contextlib.redirect_stdout(io.StringIO()), scratch_owner(entry):
            ex.fn(*entry.static)
            torch.cuda.synchronize(dev)
    finally:
        logging.disable(logging.NOTSET)
    per_forward = nat_.launch_count - c0
    gpu_launches = args.steps * per_forward
    syncs = profile_syncs(ex, xs_dev[0])
    comparator = None
    if not args.no_compile and rank == 0:
        comparator = compile_comparator(prog, dtype, xs_dev, ex, iters=max(50, args.steps))
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "samples/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "p50_ms": statistics.median(step_ms),
        "cold_ms": cold_ms,
        "transform_ms_one_time": _transform_ms(args.workload),
        "host_syncs_per_forward": info.host_syncs,
        "host_syncs_profiler": syncs,
        "mode": info.mode,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": DATA,
        "config": _config(args, xs_host[0][0]),
        "parallelism": f"{ws} independent replicas (gloo timing barrier, no NCCL)" if ws > 1 else "single GPU",
        "l2": "flushed between timed steps: 256 MB write, then 256 MB read (cold, clean L2)",
        "speculation": speculation,
        "compile": comparator,
        "e2e": {"value": replica_value(batch, args.steps, ws, e2e_total), "unit": "samples/s",
                "how": "B200Executor.run_host_pipelined: pinned host inputs (rotating) -> H2D -> graph replay -> D2H "
                       "into pinned host outputs, 3 rotating graph slots; wall clock, max over ranks",
                "p50_ms_single_call": statistics.median(e2e_ms),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "copy_only_samples_per_s": replica_value(batch, args.steps, ws, pcie_s),
                "copy_only_how": "same pipeline (two copy streams, pinned buffers) with the forward removed"},
        "gpu_launches": gpu_launches,
        "gpu_launches_per_forward": per_forward,
        "gemm": {"backend": "cuBLASLt 12.9 BF16x9 emulation (fp32)" if args.dtype == "fp32" else "torch cuBLAS",
                 "calls": dict(gemm.stats)},
        "roofline": roofline,
        "kernels": kernels,
        "clocks": clocks.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(prog, shapes, dtype)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def _copy_only_pipeline(x_host, outs, dev, steps: int) -> float:
    """Wall time of `steps` H2D input copies + D2H output copies over 3
    rotating buffers (no forward), the same streams/events pattern as
    B200Executor.run_host_pipelined."""
    import torch

    S = 3
    dst = [[torch.empty_like(t, device=dev) for t in x_host] for _ in range(S)]
    src = [torch.empty(o.shape, dtype=o.dtype, device=dev) for o in outs[:S]]
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    loaded = [torch.cuda.Event() for _ in range(S)]
    free = [torch.cuda.Event() for _ in range(S)]
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for k in range(steps):
        s = k % S
        with torch.cuda.stream(h2d):
            if k >= S:
                h2d.wait_event(free[s])
            for d, h in zip(dst[s], x_host):
                d.copy_(h, non_blocking=True)
            loaded[s].record(h2d)
        with torch.cuda.stream(d2h):
            d2h.wait_event(loaded[s])
            outs[k].copy_(src[s], non_blocking=True)
            free[s].record(d2h)
    d2h.synchronize()
    h2d.synchronize()
    return time.perf_counter() - t0


def _live_kernel_ms(ex, regions, xs_dev, flush, dev, steps: int) -> dict:
    """Per-region kernel duration (ms, mean) inside the forward's own CUDA
    graph under the timed loop's conditions: a fresh graph slot is captured
    with a pair of external CUDA events around every region launch, then
    replayed `steps` times over the rotating inputs with the L2 flushed
    before each step; the events are read after each replay."""
    import torch

    for r in regions:
        r.probe = (torch.cuda.Event(enable_timing=True, external=True),
                   torch.cuda.Event(enable_timing=True, external=True))
    try:
        entry = ex.prepare(*xs_dev[0], slot="probe")
    finally:
        probes = {id(r): r.probe for r in regions}
        for r in regions:
            r.probe = None
    acc = {rid: [] for rid in probes}
    R = len(xs_dev)
    for i in range(steps):
        entry.load(xs_dev[i % R])
        flush()
        entry.run()
        torch.cuda.synchronize(dev)
        if i < 3:
            continue   # the slot's first launches (its confidence counters start at 0)
        for rid, (a, b) in probes.items():
            acc[rid].append(a.elapsed_time(b))
    ex.flush()
    return {rid: statistics.mean(v) for rid, v in acc.items() if v}


def _time_kernel_flushed(spec, args, flush, dev, reps: int = 20, trials: int = 5, mode: str = "hit") -> float:
    """Average duration (ms) of one region launch with a cold L2.  For a
    speculative region `mode` picks the path every launch takes through the
    scratch's diagnostics word: "hit" (speculation on the predicted
    decisions — the sampled or the last launch's, both right here), "miss"
    (speculation on every decision flipped, then the restart) or "exact"
    (the exact entry)."""
    import torch

    nd = len(spec.plan.decisions) if spec.plan.spec else 0
    from paper_2509_16248_b200.region import FORCE_EXACT, FORCE_SPEC, SCRATCH_FORCE, SCRATCH_PRED, scratch_owner

    owner = object()   # this measurement's own barrier scratch, zeroed before the captures
    want_pred = want_force = None
    if nd:
        vals = spec.scalars()
        dec = [1 if vals[spec.plan.slot[d.uid]] != 0.0 else 0 for d in spec.plan.decisions]
        want_pred = torch.tensor(dec, dtype=torch.int32, device=dev)   # history predictor: right
        word = {"hit": FORCE_SPEC, "miss": FORCE_SPEC | ((1 << nd) - 1), "exact": FORCE_EXACT}[mode]
        want_force = torch.tensor([word], dtype=torch.int32, device=dev)

    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side), scratch_owner(owner):
        spec.run(args, pdl=False)  # warm (allocator, module, this owner's scratch)
        pred = spec.scratch[SCRATCH_PRED: SCRATCH_PRED + 4 * nd].view(torch.int32) if nd else None
        fw = spec.scratch[SCRATCH_FORCE: SCRATCH_FORCE + 4].view(torch.int32) if nd else None
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize(dev)
    g_both, g_flush = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    keep = []

    def force():
        if want_pred is not None:
            pred.copy_(want_pred)
            fw.copy_(want_force)

    with torch.cuda.graph(g_both), scratch_owner(owner):
        for _ in range(reps):
            flush()
            force()
            keep.append(spec.run(args, pdl=False))  # the kernel's own duration
    with torch.cuda.graph(g_flush):
        for _ in range(reps):
            flush()
            force()

    def t(g):
        g.replay()
        torch.cuda.synchronize(dev)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        return s.elapsed_time(e)

    diffs = [(t(g_both) - t(g_flush)) / reps for _ in range(trials)]
    return statistics.median(diffs)


if __name__ == "__main__":
    main()

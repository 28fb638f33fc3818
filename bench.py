"""Bench: forward latency / throughput of a GraphMend-transformed program on
the B200 path (BASELINE.json metric; config 2 = BigBird-like layer, seq 1024,
batch 8, bf16, random-init weights, synthetic inputs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--dtype bf16|fp32]
    python bench.py --impl reference ...     # the reference's CPU path on the host cores

A step = one forward of the transformed program over one batch.  `value` is
whole-job samples/s with inputs resident in HBM (graph replay only, device
timed per step with CUDA events, L2 flushed between steps); `e2e` is the same
forward through the public API (B200Executor.__call__) from pinned host
buffers with the H2D input copy and D2H output read inside the timed region.
Multi-GPU: independent replicas (every predicate is a global
reduction, so the path does not shard), one process per GPU; the timing is
the max over ranks.
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


def max_over_ranks(x: float, dist_mod, device=None) -> float:
    """Max of a per-rank duration across replicas (all-reduce MAX on a 1-elem
    tensor: plumbing for the timing, not a data-path collective)."""
    if dist_mod is None or not dist_mod.is_initialized() or dist_mod.get_world_size() == 1:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=device or "cpu")
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


def _inputs(prog, shapes, dtype):
    from paper_2509_16248_b200.harness import make_args

    spec = prog["inputs"][0]
    return make_args(spec["args"], spec["seed"], dtype, shapes)


def run_reference(args, ws, rank):
    """The reference's CPU path: the reference-transformed program executed
    eagerly on CPU (harness call shape, runner.py:154-157) with all host
    threads; rank 0 only."""
    if rank != 0:
        return
    import torch

    from oracle import executor as orc
    from paper_2509_16248_b200.harness import programs

    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    dtype = {"bf16": torch.bfloat16, "fp32": torch.float32}[args.dtype]
    prog = programs()[args.workload]
    shapes = WORKLOADS[args.workload][1]
    x = _inputs(prog, shapes, dtype)
    fn = orc.reference_callable(prog["transformed"], prog["callable"], dtype)
    for _ in range(args.warmup):
        orc.call_captured(fn, x)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.call_captured(fn, x)
        times.append(time.perf_counter() - t0)
    batch = int(x[0].shape[0])
    total = sum(times)
    value = batch * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "p50_ms": 1e3 * statistics.median(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (manifest seed/dist), random-init weights",
        "config": {"workload": f"{args.workload} ({WORKLOADS[args.workload][0]})", "batch": batch,
                   "shape": list(x[0].shape)},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port", "cpu_model": _cpu_model(),
                         "sample": f"{len(times)} full forwards of the reference-transformed program, eager "
                                   f"torch CPU, {threads} threads"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(prog, shapes, dtype, budget_s=10.0):
    """Bounded CPU-oracle sample on the box's host cores (rank 0, N=1)."""
    import torch

    from oracle import executor as orc

    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    x = _inputs(prog, shapes, dtype)
    fn = orc.reference_callable(prog["transformed"], prog["callable"], dtype)
    orc.call_captured(fn, x)
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end and len(times) < 2000:
        t0 = time.perf_counter()
        orc.call_captured(fn, x)
        times.append(time.perf_counter() - t0)
    batch = int(x[0].shape[0])
    return {"value": batch * len(times) / sum(times), "unit": "samples/s", "cores": threads, "kind": "port",
            "cpu_model": _cpu_model(),
            "sample": f"{len(times)} forwards of the reference-transformed program (same inputs), eager torch "
                      f"CPU, {threads} threads; p50 {1e3 * statistics.median(times):.2f} ms"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="bigbird_like", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    ws, rank, local = _dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch

    from paper_2509_16248_b200 import compile_program
    from paper_2509_16248_b200.harness import programs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    dtype = {"bf16": torch.bfloat16, "fp32": torch.float32}[args.dtype]
    prog = programs()[args.workload]
    shapes = WORKLOADS[args.workload][1]
    x_host = [t.pin_memory() for t in _inputs(prog, shapes, dtype)]
    batch = int(x_host[0].shape[0])

    t0 = time.perf_counter()
    ex, mod, low = compile_program(prog["transformed"], prog["callable"], device=dev, dtype=dtype)
    entry = ex.prepare(*[t.to(dev) for t in x_host])
    torch.cuda.synchronize(dev)
    cold_ms = 1e3 * (time.perf_counter() - t0)
    entry.load([t.to(dev) for t in x_host])
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

    # ---- device-timed replay (inputs resident in HBM)
    for _ in range(args.warmup):
        entry.run()
    ex.flush()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clocks:
        # keep the GPU busy (untimed replays) until nvidia-smi has sampled it
        # under load, so the clock record covers the timed region
        t_load = time.perf_counter()
        while time.perf_counter() - t_load < 1.0 or len(clocks.rows) < 3:
            for _ in range(200):
                entry.run()
            torch.cuda.synchronize(dev)
            if time.perf_counter() - t_load > 5.0:
                break
        barrier()
        for i in range(args.steps):
            flush_l2()
            starts[i].record(stream)
            entry.run()
            ends[i].record(stream)
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ex.flush()
    total_ms = max_over_ranks(sum(step_ms), pg, dev)
    value = replica_value(batch, args.steps, ws, total_ms / 1e3)

    # ---- each fused kernel timed on its own stream, cold L2: a CUDA graph of
    #      R x [256 MB L2 flush, region launch] minus a graph of R x [flush],
    #      both replayed between CUDA events (no host work inside the window)
    fused = [r for r in low.regions if r.last_spec is not None]
    kernels = []
    for r in fused:
        spec = r.last_spec
        ms = _time_kernel_flushed(spec, list(r.last_args), flush_l2, dev)
        k = {"name": f"{spec.plan.kernel} ({r.name})", "ms": ms,
             "bytes": spec.bytes_alg(list(r.last_args)), "grid": spec.grid, "smem": spec.smem,
             "passes": spec.plan.npass, "speculative": spec.plan.spec,
             "how": "graph of 20 x (L2 flush + launch) minus 20 x flush; cold L2"}
        if spec.plan.spec:
            launches, misses = spec.spec_stats()
            k["spec_launches"], k["spec_misses"] = launches, misses
            k["ms_mispredicted"] = _time_kernel_flushed(spec, list(r.last_args), flush_l2, dev, mispredict=True)
        kernels.append(k)
    dom = max(kernels, key=lambda k: k["ms"]) if kernels else None
    peak, peak_kind = _peaks()
    roofline = None
    if dom:
        achieved = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": _ncu_traffic(dom["name"].split(" ")[0]), "kernel": dom["name"],
                    "bytes_alg": dom["bytes"], "kernel_ms": dom["ms"],
                    "peak_kind": peak_kind, "share_of_step": dom["ms"] / statistics.mean(step_ms)}

    # ---- end to end through the public API, host buffers in and out:
    # (a) single call latency: executor(*pinned host inputs) -> D2H into a
    #     pinned host tensor, synchronised; (b) throughput: the executor's
    #     pipelined host path (H2D / forward / D2H overlapped, 3 graph slots).
    h2d = sum(t.numel() * t.element_size() for t in x_host)
    out0 = ex(*x_host)
    out_pinned = torch.empty(out0.shape, dtype=out0.dtype, pin_memory=True)
    e2e_ms = []
    for i in range(args.steps + 3):
        e0 = time.perf_counter()
        out = ex(*x_host)
        out_pinned.copy_(out, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        if i >= 3:
            e2e_ms.append(1e3 * (time.perf_counter() - e0))
    ex.flush()
    host_batches = [tuple(x_host)] * args.steps
    # results land in a ring of 8 pinned host buffers (step k -> buffer k % 8:
    # the D2H copies into one buffer are ordered on the copy stream), so N
    # replicas do not pin N x steps x 12.6 MB of host memory
    ring = [torch.empty(out0.shape, dtype=out0.dtype, pin_memory=True) for _ in range(min(8, args.steps))]
    outs = [ring[k % len(ring)] for k in range(args.steps)]
    ex.run_host_pipelined(host_batches[:4], out=outs[:4])  # build the graph slots, warm
    ex.flush()
    barrier()
    t_e2e = time.perf_counter()
    ex.run_host_pipelined(host_batches, out=outs)
    barrier()
    e2e_total = max_over_ranks(time.perf_counter() - t_e2e, pg, dev)
    # the same pipelined H2D / D2H traffic with no forward: the PCIe
    # bound the end-to-end number sits against
    pcie_s = _copy_only_pipeline(x_host, outs, dev, args.steps)
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
        with torch.no_grad(), contextlib.redirect_stdout(io.StringIO()):  # its deferred prints run now
            ex.fn(*entry.static)
            torch.cuda.synchronize(dev)
    finally:
        logging.disable(logging.NOTSET)
    gpu_launches = args.steps * (nat_.launch_count - c0)
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
        "mode": info.mode,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic inputs (manifest seed/dist at the BASELINE shape), random-init weights (seed 0)",
        "config": {"workload": f"{args.workload} ({WORKLOADS[args.workload][0]})", "batch": batch,
                   "shape": list(x_host[0].shape), "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "l2": "flushed between timed steps: 256 MB write, then 256 MB read (cold, clean L2)"},
        "e2e": {"value": replica_value(batch, args.steps, ws, e2e_total), "unit": "samples/s",
                "how": "B200Executor.run_host_pipelined: pinned host inputs -> H2D -> graph replay -> D2H into "
                       "pinned host outputs, 3 rotating graph slots; wall clock, max over ranks",
                "p50_ms_single_call": statistics.median(e2e_ms),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "copy_only_samples_per_s": replica_value(batch, args.steps, ws, pcie_s),
                "copy_only_how": "same pipeline (two copy streams, pinned buffers) with the forward removed"},
        "gpu_launches": gpu_launches,
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


def _time_kernel_flushed(spec, args, flush, dev, reps: int = 20, trials: int = 5, mispredict: bool = False) -> float:
    """Average duration (ms) of one region launch with a cold L2.  With
    `mispredict`, every launch of a speculative region is handed the wrong
    predictions (the exact fallback path runs)."""
    import torch

    nd = len(spec.plan.decisions) if spec.plan.spec else 0
    from paper_2509_16248_b200.region import SCRATCH_PRED

    pred = spec.scratch[SCRATCH_PRED: SCRATCH_PRED + 4 * nd].view(torch.int32) if nd else None
    wrong = None
    if mispredict and nd:
        vals = spec.scalars()
        wrong = torch.tensor([0 if vals[spec.plan.slot[d.uid]] != 0.0 else 1 for d in spec.plan.decisions],
                             dtype=torch.int32, device=dev)

    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        spec.run(args, pdl=False)  # warm (allocator, module)
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize(dev)
    g_both, g_flush = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    keep = []
    with torch.cuda.graph(g_both):
        for _ in range(reps):
            flush()
            if wrong is not None:
                pred.copy_(wrong)
            keep.append(spec.run(args, pdl=False))  # the kernel's own duration
    with torch.cuda.graph(g_flush):
        for _ in range(reps):
            flush()
            if wrong is not None:
                pred.copy_(wrong)

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

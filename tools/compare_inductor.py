"""Comparator (SURVEY §8d / BASELINE.md §3): the UNTRANSFORMED original
program under torch.compile (Inductor, default and reduce-overhead) on the
same GPU, inputs and weights, vs the B200 path on the transformed program.

    python tools/compare_inductor.py [--workloads bigbird_like,phi4_like] [--dtype bf16]

Prints one JSON line per workload with p50 forward latency (ms, wall clock
around a synchronised forward, warm) for: original eager, original
torch.compile default, original torch.compile reduce-overhead, transformed
eager (PyTorch ops, no fusion), the B200 path (graph replay alone, and the
user-facing call that also copies the inputs in), and the transformed program
under torch.compile with this package as the backend.  The speed-up is taken
against the user-facing call.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {
    "bigbird_like": None, "bart_step": None, "toy": None, "bigbird_attn": None, "bigbird_layer": None, "gemm_arms": None,
    "phi4_like": [[8, 1024, 768]], "qwen_audio_like": [[8, 1024, 768]], "biogpt_like": [[8, 1024, 768]] * 2,
    "blenderbot_like": [[8, 1024, 768]], "pegasus_like": [[8, 1024, 768]],
    "flan_t5_like": [[8192, 768], [768, 768]], "longformer_like": [[4, 4096, 768]],
    "moe_minicpm_like": [[8, 1024, 768]],
}


def p50(fn, iters=50, warm=5):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts)


def main():
    import logging

    import torch

    from oracle import executor as orc
    from paper_2509_16248_b200 import compile_program
    from paper_2509_16248_b200.harness import make_args, programs

    logging.disable(logging.CRITICAL)
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="bigbird_like,bart_step,phi4_like,qwen_audio_like,biogpt_like")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    dtype = {"bf16": torch.bfloat16, "fp32": torch.float32}[args.dtype]
    dev = torch.device("cuda", 0)
    P = programs()
    for name in args.workloads.split(","):
        prog = P[name]
        spec = prog["inputs"][0]
        x = [t.to(dev) for t in make_args(spec["args"], spec["seed"], dtype, SHAPES[name])]
        res = {"workload": name, "dtype": args.dtype, "shape": list(x[0].shape)}

        def load(text):
            fn = orc.reference_callable(text, prog["callable"], dtype)
            if isinstance(fn, torch.nn.Module):
                fn.to(dev)
            return fn

        orig = load(prog["original"])
        trans = load(prog["transformed"])
        with torch.no_grad():
            res["original_eager_ms"] = p50(lambda: orig(*x), args.iters)
            res["transformed_eager_ms"] = p50(lambda: trans(*x), args.iters)
            for mode in ("default", "reduce-overhead"):
                torch._dynamo.reset()
                try:
                    c = torch.compile(load(prog["original"]), mode=None if mode == "default" else mode)
                    t0 = time.perf_counter()
                    c(*x)
                    torch.cuda.synchronize()
                    res[f"original_compile_{mode}_cold_ms"] = 1e3 * (time.perf_counter() - t0)
                    res[f"original_compile_{mode}_ms"] = p50(lambda: c(*x), args.iters)
                except Exception as exc:  # report, keep going
                    res[f"original_compile_{mode}_error"] = repr(exc)[:200]
        ex, _mod, _low = compile_program(prog["transformed"], prog["callable"], device=dev, dtype=dtype)
        t0 = time.perf_counter()
        entry = ex.prepare(*x)
        torch.cuda.synchronize()
        res["b200_cold_ms"] = 1e3 * (time.perf_counter() - t0)
        res["b200_mode"] = entry.info.mode
        res["b200_host_syncs"] = entry.info.host_syncs
        res["b200_ms"] = p50(lambda: entry.run(), args.iters)
        # the user-facing call: copies the inputs into the graph's static
        # buffers, replays, enqueues the deferred calls
        res["b200_call_ms"] = p50(lambda: ex(*x), args.iters)
        ex.flush()
        # the same transformed program through torch.compile with this
        # package as the Dynamo backend
        try:
            import paper_2509_16248_b200.dynamo  # noqa: F401

            torch._dynamo.reset()
            from paper_2509_16248_b200.dynamo import gm_compile

            cb = gm_compile(load(prog["transformed"]))
            with torch.no_grad():
                cb(*x)
                res["gm_compile_backend_ms"] = p50(lambda: cb(*x), args.iters)
        except Exception as exc:  # report, keep going
            res["gm_compile_backend_error"] = repr(exc)[:200]
        ref = res.get("original_compile_default_ms")
        if ref:
            res["speedup_vs_compile_default"] = ref / res["b200_call_ms"]
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

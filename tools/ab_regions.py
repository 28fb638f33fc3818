"""A/B timing of region-kernel code-generation variants in one process.

    python tools/ab_regions.py --workload bigbird_like --dtype bf16 \
        --variant base: --variant nodefer:GM_DEFER_STORES=0 --rounds 7

Every variant is a set of environment overrides read by codegen.Plan.  The
workload runs once to record each region's arguments; then, per round and
variant (interleaved, so drift hits every variant alike), each region kernel
is timed as bench.py does: a CUDA graph of 20 x (L2 flush + launch) minus a
graph of 20 x flush.  Prints the median per variant and region (us).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import WORKLOADS, _all_inputs, _time_kernel_flushed
    from paper_2509_16248_b200 import compile_program
    from paper_2509_16248_b200 import region as reg
    from paper_2509_16248_b200.harness import programs

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bigbird_like")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--variant", action="append", default=[])
    ap.add_argument("--rounds", type=int, default=7)
    a = ap.parse_args()
    dtype = {"bf16": torch.bfloat16, "fp32": torch.float32}[a.dtype]
    prog = programs()[a.workload]
    x = [t.cuda() for t in _all_inputs(prog, WORKLOADS[a.workload][1], dtype)[0]]
    ex, mod, low = compile_program(prog["transformed"], prog["callable"], dtype=dtype)
    ex(*x)
    ex.flush()
    torch.cuda.synchronize()
    dev = x[0].device
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    flush_rd = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.int64, device=dev)

    def flush():
        flush_buf.zero_()
        flush_rd.sum()

    variants = {}
    for v in a.variant or ["base:"]:
        name, _, envs = v.partition(":")
        env = dict(e.split("=", 1) for e in envs.split(",") if e)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            specs = []
            for r in low.regions:
                if r.last_spec is None:
                    continue
                s = reg._Spec(r, list(r.last_args))
                for _ in range(3):   # learn the predictions
                    s.run(list(r.last_args))
                specs.append((r.name, s, list(r.last_args)))
        finally:
            for k, val in old.items():
                if val is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = val
        variants[name] = specs
    torch.cuda.synchronize()
    res = {n: {rn: [] for rn, _, _ in sp} for n, sp in variants.items()}
    for _ in range(a.rounds):
        for n, sp in variants.items():
            for rn, s, args in sp:
                res[n][rn].append(1e3 * _time_kernel_flushed(s, args, flush, dev, trials=3))
    out = {n: {rn: round(statistics.median(v), 2) for rn, v in d.items()} for n, d in res.items()}
    print(json.dumps({"workload": a.workload, "dtype": a.dtype, "us_median": out}))


if __name__ == "__main__":
    main()

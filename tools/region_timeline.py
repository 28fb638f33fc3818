"""Per-pass timeline of the fused region kernels of a workload (GM_PROFILE=1).

    GM_PROFILE=1 python tools/region_timeline.py --workload bigbird_like --dtype bf16

Speculative regions: GM_SPEC_CONFIDENT=99 times the exact entry, =0 the
speculative sweep (the input repeats, so every launch hits).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("GM_PROFILE", "1")


def main():
    import torch

    from bench import WORKLOADS, _all_inputs
    from paper_2509_16248_b200 import compile_program
    from paper_2509_16248_b200.harness import programs

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bigbird_like")
    ap.add_argument("--dtype", default="bf16")
    a = ap.parse_args()
    dtype = {"bf16": torch.bfloat16, "fp32": torch.float32}[a.dtype]
    prog = programs()[a.workload]
    x = [t.cuda() for t in _all_inputs(prog, WORKLOADS[a.workload][1], dtype)[0]]
    ex, mod, low = compile_program(prog["transformed"], prog["callable"], dtype=dtype)
    ex(*x)
    torch.cuda.synchronize()
    for r in low.regions:
        spec = r.last_spec
        if spec is None:
            continue
        rows = []
        for it in range(5):
            spec.reset_timeline()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            spec.run(list(r.last_args))
            e.record()
            torch.cuda.synchronize()
            tl = spec.timeline()
            rows.append({"event_us": 1e3 * s.elapsed_time(e), "timeline_ns": [v for v in tl[:32] if v], "first_cta_done_ns": [v for v in tl[32:40] if v],
                         "barrier_ns (per reduce: last CTA before arrival, arrival done, poll done, combine done)": [v for v in tl[40:63] if v]})
        print(json.dumps({"region": r.name, "grid": spec.grid, "smem": spec.smem, "passes": spec.plan.npass,
                          "runs": rows[-2:]}))


if __name__ == "__main__":
    main()

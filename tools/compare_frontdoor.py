"""p50 of the torch.compile front door (dynamo.gm_compile -> gm_b200 backend)
against the direct path (compile_program -> B200Executor) on every workload,
same GPU, inputs and weights.  Prints one JSON line per
workload x dtype."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import WORKLOADS, _all_inputs
from paper_2509_16248_b200 import compile_program
from paper_2509_16248_b200.dynamo import gm_compile
from paper_2509_16248_b200.harness import programs


def p50(fn, xs, iters=100):
    for x in xs:
        fn(*x)
    torch.cuda.synchronize()
    ts = []
    for i in range(iters):
        t0 = time.perf_counter()
        fn(*xs[i % len(xs)])
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts)


def main():
    progs = programs()
    dtypes = [torch.float32, torch.bfloat16]
    for name in sorted(WORKLOADS):
        for dtype in dtypes:
            torch._dynamo.reset()
            from torch._dynamo.utils import counters

            counters.clear()
            prog = progs[name]
            xs = [[t.cuda() for t in x] for x in _all_inputs(prog, WORKLOADS[name][1], dtype)]
            ex, mod, low = compile_program(prog["transformed"], prog["callable"], dtype=dtype)
            with torch.no_grad():
                direct = p50(lambda *a: ex(*a), xs)
                ex.flush()
                ns = {}
                exec(compile(prog["transformed"], prog["callable"], "exec"), ns)
                fn = ns[prog["callable"]]
                if isinstance(fn, torch.nn.Module):
                    fn.to("cuda", dtype)
                c = gm_compile(fn)
                try:
                    front = p50(c, xs)
                    err = None
                except Exception as exc:  # report, keep going
                    front, err = float("nan"), repr(exc)[:200]
            from torch._dynamo.utils import counters

            print(json.dumps({"workload": name, "dtype": str(dtype)[6:], "direct_p50_ms": direct,
                              "gm_compile_p50_ms": front, "ratio": front / direct,
                              "fx_graphs": counters["stats"].get("unique_graphs"), "error": err}), flush=True)


if __name__ == "__main__":
    main()

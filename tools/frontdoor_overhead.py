"""Where the torch.compile front door's per-call time goes (gm_compile ->
gm_b200 backend -> B200Executor) against the direct path, on one workload:
host-timed p50 of each layer with a synchronize after every call.

  direct            ex(*x)                            (compile_program)
  direct+flush      ex(*x); ex.flush()
  backend           the backend's `run` called with Dynamo's own arguments
  backend, no clone the same with static outputs
  gm_compile        the full front door (Dynamo guards + backend)
"""
import functools
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import WORKLOADS, _all_inputs
from paper_2509_16248_b200 import compile_program, dynamo
from paper_2509_16248_b200.harness import programs


def p50(fn, iters=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e6 * (time.perf_counter() - t0))
    return statistics.median(ts)


def main():
    names = sys.argv[1:] or ["phi4_like", "bigbird_layer"]
    progs = programs()
    for name in names:
        for dtype in (torch.float32, torch.bfloat16):
            prog = progs[name]
            x = [t.cuda() for t in _all_inputs(prog, WORKLOADS[name][1], dtype)[0]]
            ex, _, _ = compile_program(prog["transformed"], prog["callable"], dtype=dtype)
            res = {"workload": name, "dtype": str(dtype)[6:]}
            with torch.no_grad():
                res["direct_us"] = p50(lambda: ex(*x))
                res["direct_flush_us"] = p50(lambda: (ex(*x), ex.flush()))
                seen = {}

                def backend(gm, example_inputs):
                    run = dynamo.gm_b200_backend(gm, example_inputs)

                    def rec(*args):
                        seen["args"], seen["run"] = args, run
                        return run(*args)
                    return rec

                torch._dynamo.reset()
                torch._dynamo.config.capture_scalar_outputs = True
                torch._dynamo.config.capture_dynamic_output_shape_ops = True
                ns = {}
                exec(compile(prog["transformed"], prog["callable"], "exec"), ns)
                fn = ns[prog["callable"]]
                if isinstance(fn, torch.nn.Module):
                    fn.to("cuda", dtype)
                c = torch.compile(fn, backend=backend)
                c(*x)
                run, args = seen["run"], seen["args"]
                res["n_graph_args"] = len(args)
                res["backend_us"] = p50(lambda: run(*args))
                ex2 = run.executor
                res["backend_executor_flush_us"] = p50(lambda: (ex2(*args), ex2.flush()))
                res["executor_only_us"] = p50(lambda: ex2(*args))
                res["gm_compile_us"] = p50(lambda: c(*x))
                for tag, env in (("gm_compile_clone_us", "0"), ("gm_compile_slots_us", "2")):
                    os.environ["GM_OUTPUT_SLOTS"] = env
                    torch._dynamo.reset()
                    cc = torch.compile(fn, backend="gm_b200")
                    cc(*x)
                    res[tag] = p50(lambda: cc(*x))
                os.environ.pop("GM_OUTPUT_SLOTS")
                torch._dynamo.reset()
                cs = torch.compile(fn, backend=functools.partial(dynamo.gm_b200_backend, static_outputs=True))
                cs(*x)
                res["gm_compile_static_us"] = p50(lambda: cs(*x))
                # Dynamo's own per-call floor: the same program and guards,
                # a backend that returns precomputed outputs without any work
                outs = run(*args)

                def noop_backend(gm, example_inputs):
                    return lambda *a: outs

                torch._dynamo.reset()
                c0 = torch.compile(fn, backend=noop_backend)
                c0(*x)
                res["dynamo_noop_backend_us"] = p50(lambda: c0(*x))
                res["sync_only_us"] = p50(lambda: None)
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

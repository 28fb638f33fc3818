"""Where the first call of a workload goes (compile_program + first
prepare, as bench.py's cold_ms): cProfile of the cold path, top entries by
cumulative time, in a fresh process."""
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import WORKLOADS, _all_inputs
from paper_2509_16248_b200 import compile_program
from paper_2509_16248_b200.harness import programs

name = sys.argv[1] if len(sys.argv) > 1 else "bigbird_layer"
prog = programs()[name]
dev = torch.device("cuda", 0)
xs = [[t.to(dev) for t in x] for x in _all_inputs(prog, WORKLOADS[name][1], torch.float32)]
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
ex, mod, low = compile_program(prog["transformed"], prog["callable"], device=dev, dtype=torch.float32)
t1 = time.perf_counter()
entry = ex.prepare(*xs[0])
torch.cuda.synchronize()
pr.disable()
t2 = time.perf_counter()
print(f"{name}: compile_program {1e3 * (t1 - t0):.1f} ms, first prepare {1e3 * (t2 - t1):.1f} ms, "
      f"build_s {entry.info.build_s:.3f}")
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(45)
print(s.getvalue())
# second workload instance in the same process (warm caches): what is per-program
t0 = time.perf_counter()
ex2, _, _ = compile_program(prog["transformed"], prog["callable"], device=dev, dtype=torch.float32)
ex2.prepare(*xs[0])
torch.cuda.synchronize()
print(f"second instance, same process: {1e3 * (time.perf_counter() - t0):.1f} ms")

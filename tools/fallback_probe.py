import sys, torch
sys.path.insert(0, '/root/repo')
from bench import WORKLOADS, _all_inputs
from paper_2509_16248_b200 import compile_program
from paper_2509_16248_b200.harness import programs
progs = programs()
for name in sorted(WORKLOADS) + ['toy']:
    for dt in (torch.float32, torch.bfloat16):
        prog = progs[name]
        shapes = WORKLOADS.get(name, (None, None))[1]
        x = [t.cuda() for t in _all_inputs(prog, shapes, dt)[0]]
        ex, mod, low = compile_program(prog['transformed'], prog['callable'], dtype=dt)
        ex(*x); ex.flush()
        print(name, str(dt)[6:], [(r.name, r.stats.launches, r.stats.fallbacks, r.stats.fallback_reasons[:1]) for r in low.regions], flush=True)

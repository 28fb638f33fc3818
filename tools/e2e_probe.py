import sys, time, torch
sys.path.insert(0, '/root/repo')
from bench import _inputs
from paper_2509_16248_b200 import compile_program
from paper_2509_16248_b200.harness import programs
prog = programs()['bigbird_like']
x_host = [t.pin_memory() for t in _inputs(prog, None, torch.bfloat16)]
ex, mod, low = compile_program(prog['transformed'], prog['callable'], dtype=torch.bfloat16)
out0 = ex(*x_host); ex.flush()
steps = 200
outs = [torch.empty(out0.shape, dtype=out0.dtype, pin_memory=True) for _ in range(steps)]
batches = [tuple(x_host)] * steps
ex.run_host_pipelined(batches[:4], out=outs[:4]); ex.flush()
torch.cuda.synchronize()
t0 = time.perf_counter()
orig = torch.cuda.Stream.synchronize
issue_end = []
def sync(self):
    issue_end.append(time.perf_counter())
    return orig(self)
torch.cuda.Stream.synchronize = sync
ex.run_host_pipelined(batches, out=outs)
t1 = time.perf_counter()
torch.cuda.Stream.synchronize = orig
print(f"total {1e3*(t1-t0):.1f} ms for {steps} steps ({1e6*(t1-t0)/steps:.0f} us/step); issue loop {1e3*(issue_end[0]-t0):.1f} ms ({1e6*(issue_end[0]-t0)/steps:.0f} us/step)")
ex.flush()

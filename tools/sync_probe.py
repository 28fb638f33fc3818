"""Which CUDA API calls does one B200Executor call make (profiler)?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2509_16248_b200 import compile_program
from paper_2509_16248_b200.harness import make_args, programs

p = programs()["bigbird_like"]
x = [t.cuda() for t in make_args(p["inputs"][0]["args"], p["inputs"][0]["seed"], torch.float32)]
ex, mod, low = compile_program(p["transformed"], p["callable"], dtype=torch.float32)
ex(*x)
ex(*x)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True) as prof:
    ex(*x)
torch.cuda.synchronize()
for e in prof.events():
    if e.name.startswith("cuda") or "Memcpy" in e.name:
        stack = [s for s in (e.stack or []) if "site-packages/torch" not in s][:8]
        print(e.name, stack)

"""Where does the host-fed pipeline (B200Executor.run_host_pipelined) lose
against the copy-only bound?  Variants over 300 steps of BigBird-like bf16:
the real pipeline (3 and 4 slots), the same stream/event chain with the
forward replaced by nothing, and bench.py's copy-only pipeline.  Also the
host issue time of the real loop."""
import sys
import time

import torch

sys.path.insert(0, '/root/repo')
from bench import _copy_only_pipeline, _all_inputs  # noqa: E402
from paper_2509_16248_b200 import compile_program  # noqa: E402
from paper_2509_16248_b200.harness import programs  # noqa: E402

prog = programs()['bigbird_like']
x_host = [t.pin_memory() for t in _all_inputs(prog, None, torch.bfloat16)[0]]
ex, mod, low = compile_program(prog['transformed'], prog['callable'], dtype=torch.bfloat16)
out0 = ex(*x_host)
ex.flush()
steps = 300
ring = [torch.empty(out0.shape, dtype=out0.dtype, pin_memory=True) for _ in range(8)]
outs = [ring[k % 8] for k in range(steps)]
batches = [tuple(x_host)] * steps
dev = out0.device


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for slots in (3, 4, 3, 4):
    ex.run_host_pipelined(batches[:6], out=outs[:6], slots=slots)
    t = timed(lambda: ex.run_host_pipelined(batches, out=outs, slots=slots))
    print(f"pipeline slots={slots}: {1e6 * t / steps:.1f} us/step")
    ex.flush()

# the same chain (h2d -> comp -> d2h events) with no forward
S = 3
dst = [[torch.empty_like(t, device=dev) for t in x_host] for _ in range(S)]
src = [torch.empty(out0.shape, dtype=out0.dtype, device=dev) for _ in range(S)]


def chain(forward, own_stream: bool = False, chunks: int = 1):
    comp = torch.cuda.Stream(dev) if own_stream else torch.cuda.current_stream(dev)
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    free = [torch.cuda.Event() for _ in range(S)]
    loaded = [torch.cuda.Event() for _ in range(S)]
    done = [torch.cuda.Event() for _ in range(S)]
    for k in range(steps):
        s = k % S
        with torch.cuda.stream(h2d):
            if k >= S:
                h2d.wait_event(free[s])
            for d, h in zip(dst[s], x_host):
                for dc, hc in zip(d.view(-1).chunk(chunks), h.view(-1).chunk(chunks)):
                    dc.copy_(hc, non_blocking=True)
            loaded[s].record(h2d)
        comp.wait_event(loaded[s])
        if forward:
            with torch.cuda.stream(comp):
                if forward is True:
                    src[s].add_(1)  # one small kernel on the compute stream
                else:
                    torch.cuda._sleep(forward)  # a kernel spinning `forward` cycles
        done[s].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done[s])
            for oc, sc in zip(outs[k].view(-1).chunk(chunks), src[s].view(-1).chunk(chunks)):
                oc.copy_(sc, non_blocking=True)
            free[s].record(d2h)
    d2h.synchronize()


print("current stream:", torch.cuda.current_stream(dev), "null:", torch.cuda.current_stream(dev).cuda_stream == 0)
for fwd, own, ch in ((False, False, 1), (80000, True, 1), (80000, True, 4), (80000, True, 16), (80000, True, 1),
                     (80000, True, 4), (False, False, 4)):
    t = timed(lambda: chain(fwd, own, ch))
    print(f"event chain, forward={fwd if fwd is not True else 'add_'}, comp={'own stream' if own else 'current'}, "
          f"chunks={ch}: {1e6 * t / steps:.1f} us/step")
with torch.cuda.stream(torch.cuda.Stream(dev)):
    for slots in (3, 3):
        ex.run_host_pipelined(batches[:6], out=outs[:6], slots=slots)
        t = timed(lambda: ex.run_host_pipelined(batches, out=outs, slots=slots))
        print(f"pipeline on a side stream, slots={slots}: {1e6 * t / steps:.1f} us/step")
        ex.flush()
t = _copy_only_pipeline(x_host, outs, dev, steps)
print(f"copy-only (bench): {1e6 * t / steps:.1f} us/step")
# H2D alone and D2H alone
t = timed(lambda: [dst[k % S][0].copy_(x_host[0], non_blocking=True) for k in range(steps)])
print(f"H2D alone: {1e6 * t / steps:.1f} us/step ({x_host[0].numel() * 2 * steps / t / 1e9:.1f} GB/s)")
t = timed(lambda: [outs[k].copy_(src[k % S], non_blocking=True) for k in range(steps)])
print(f"D2H alone: {1e6 * t / steps:.1f} us/step")


# per-slot streams: step k runs H2D -> forward -> D2H on stream k % S, so
# stream order alone guards slot reuse (no cross-stream events)
def per_slot(n_slots: int, forward: bool):
    streams = [torch.cuda.Stream(dev) for _ in range(n_slots)]
    entries = [ex.prepare(*[b.to(dev) for b in batches[0]], slot=s) for s in range(n_slots)]
    for k in range(steps):
        s = k % n_slots
        e = entries[s]
        with torch.cuda.stream(streams[s]):
            for st, a in zip(e.static, batches[k]):
                if torch.is_tensor(st):
                    st.copy_(a, non_blocking=True)
            o = e.run() if forward else e.outputs
            outs[k].copy_(o, non_blocking=True)
    for st in streams:
        st.synchronize()


for n_slots in (3, 4, 3, 4):
    for fwd in (True, False):
        per_slot(n_slots, fwd)
        t = timed(lambda: per_slot(n_slots, fwd))
        print(f"per-slot streams x{n_slots}, forward={fwd}: {1e6 * t / steps:.1f} us/step")
        ex.flush()


# do kernels slow the copies at all?  copy-only pipeline with an independent
# stream kept busy by spin kernels (no memory traffic) / by the forward graph
def copy_with_background(kind: str):
    bg = torch.cuda.Stream(dev)
    with torch.cuda.stream(bg):
        for _ in range(steps // 2):
            if kind == "spin":
                torch.cuda._sleep(200000)
            else:
                ex.entries[next(iter(ex.entries))].graph.replay()
    return _copy_only_pipeline(x_host, outs, dev, steps)


for kind in ("spin", "forward"):
    torch.cuda.synchronize()
    t = copy_with_background(kind)
    torch.cuda.synchronize()
    print(f"copy-only with a busy background stream ({kind}): {1e6 * t / steps:.1f} us/step")


# software-pipelined issue order: H2D of step k+L is issued before the D2H of
# step k, so a D2H waiting on its forward never sits ahead of later H2Ds in a
# copy queue
def lookahead(L: int, n_slots: int = 3):
    entries = [ex.prepare(*[b.to(dev) for b in batches[0]], slot=s) for s in range(n_slots)]
    comp = torch.cuda.current_stream(dev)
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    free = [torch.cuda.Event() for _ in range(n_slots)]
    loaded = [torch.cuda.Event() for _ in range(n_slots)]
    done = [torch.cuda.Event() for _ in range(n_slots)]

    def load(j):
        s = j % n_slots
        with torch.cuda.stream(h2d):
            if j >= n_slots:
                h2d.wait_event(free[s])
            for st, a in zip(entries[s].static, batches[j]):
                if torch.is_tensor(st):
                    st.copy_(a, non_blocking=True)
            loaded[s].record(h2d)

    for j in range(min(L, steps)):
        load(j)
    for k in range(steps):
        if k + L < steps:
            load(k + L)
        s = k % n_slots
        comp.wait_event(loaded[s])
        o = entries[s].run()
        done[s].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done[s])
            outs[k].copy_(o, non_blocking=True)
            free[s].record(d2h)
    d2h.synchronize()


for L, S in ((1, 3), (2, 3), (1, 4), (2, 4), (3, 4), (1, 3), (2, 4)):
    lookahead(L, S)
    t = timed(lambda: lookahead(L, S))
    print(f"lookahead L={L} slots={S}: {1e6 * t / steps:.1f} us/step")
    ex.flush()

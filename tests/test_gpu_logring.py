"""The record-level log ring (include/gm_b200.h):
gm_logring_capture / gm_logring_end_step on the device, gm_logring_drain
with a C callback on the host, and torch.ops.gm.log_capture inside a
Dynamo-traced graph."""

import ctypes

import pytest
import torch

from paper_2509_16248_b200 import _native as nat
from paper_2509_16248_b200 import logring


def _summary(t: torch.Tensor) -> torch.Tensor:
    """The elements torch's repr reads (edgeitems 3 when numel > 1000)."""
    counts, heads = logring.summary_plan(tuple(t.shape))
    idx = []
    for d, (c, h, s) in enumerate(zip(counts, heads, t.shape)):
        idx.append(torch.tensor([k if k < h else s - c + k for k in range(c)]))
    return t[torch.meshgrid(*idx, indexing="ij")] if idx else t


@pytest.mark.gpu
def test_capture_and_drain_through_the_c_callback():
    """Records are delivered by gm_logring_drain, through a C function
    pointer, in commit order; the data are exactly the summarised
    elements; a step without records launches nothing."""
    nat.init(0)
    h = ctypes.c_void_p()
    nat.check(nat.lib().gm_logring_open(64 << 16, ctypes.byref(h)))
    got = []

    @nat.RECORD_CB
    def cb(rec_p, user):
        r = rec_p.contents
        shape = tuple(r.shape[i] for i in range(r.ndim))
        counts = tuple(r.counts[i] for i in range(r.ndim))
        got.append((r.record_id, r.step, r.dtype, shape, counts, ctypes.string_at(r.data, r.bytes)))
        return 0

    torch.manual_seed(0)
    xs = [torch.randn(50, 40, device="cuda"), torch.randn(5, 7, device="cuda").t(),
          torch.randn(3000, device="cuda").to(torch.bfloat16)]
    s = torch.cuda.current_stream().cuda_stream
    lib = nat.lib()
    for step, ts in enumerate([xs[:2], xs[2:], []]):
        nat.check(lib.gm_logring_begin_step(h))
        for j, t in enumerate(ts):
            code = {torch.float32: nat.GM_F32, torch.bfloat16: nat.GM_BF16}[t.dtype]
            shape = (ctypes.c_int64 * t.dim())(*t.shape)
            stride = (ctypes.c_int64 * t.dim())(*t.stride())
            nat.check(lib.gm_logring_capture(h, ctypes.c_void_p(t.data_ptr()), shape, stride, t.dim(), code,
                                             100 * step + j, ctypes.c_void_p(s)))
        tid = ctypes.c_uint32()
        nat.check(lib.gm_logring_end_step(h, ctypes.c_void_p(s), ctypes.byref(tid)))
        if not ts:
            assert tid.value == nat.LOGRING_NO_TEMPLATE
    torch.cuda.synchronize()
    assert lib.gm_logring_drain(h, cb, None) == 2      # two committing steps
    assert [g[0] for g in got] == [0, 1, 100] and [g[1] for g in got] == [1, 1, 2]
    for (rid, step, code, shape, counts, data), t in zip(got, xs):
        want = _summary(t.cpu())
        assert shape == tuple(t.shape) and counts == tuple(want.shape)
        back = torch.frombuffer(bytearray(data), dtype=t.dtype).reshape(counts)
        assert torch.equal(back, want.contiguous())
    assert lib.gm_logring_drain(h, cb, None) == 0      # nothing new
    lib.gm_logring_close(h)


@pytest.mark.gpu
def test_drain_is_graph_replayable():
    """A captured step replays its gathers and its commit; every replay is
    drained as a new step with the replayed data."""
    ring = logring.LogRing(torch.device("cuda", 0), slot_bytes=1 << 16)
    x = torch.zeros(4, 5, device="cuda")
    seen = []
    tmpl_holder = {}
    logring.on_record(424242, lambda t: seen.append(t.clone()))
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g):
        ring.begin()
        ring.capture(x, 424242)
        tmpl_holder["t"] = ring.end()
    for k in range(3):
        x.fill_(k)
        g.replay()
        ring.enqueue(tmpl_holder["t"])
    ring.flush()
    assert [float(t[0, 0]) for t in seen] == [0.0, 1.0, 2.0]
    ring.close()


@pytest.mark.gpu
def test_log_capture_op_in_a_dynamo_graph():
    """torch.ops.gm.log_capture stays inside a fullgraph Dynamo trace
    (ordered effectful op) and, through the gm_b200 backend, inside the CUDA
    graph: every call's tensor arrives at the registered handler."""
    from paper_2509_16248_b200 import dynamo  # noqa: F401

    torch._dynamo.reset()
    got = []
    logring.on_record(777, lambda t: got.append(t))

    def f(x):
        h = x * 2
        torch.ops.gm.log_capture(h, 777)
        return h + 1

    c = torch.compile(f, backend="gm_b200", fullgraph=True)
    with torch.no_grad():
        for v in (1.0, 2.0):
            x = torch.full((64, 64), v, device="cuda")
            out = c(x)
            torch.cuda.synchronize()
            assert torch.equal(out.cpu(), torch.full((64, 64), 2 * v + 1))
    logring.ring_for(torch.device("cuda", 0)).flush()
    assert [float(t[0, 0]) for t in got] == [2.0, 4.0], got
    assert all(t.shape == (64, 64) for t in got)

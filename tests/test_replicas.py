"""N>1 path on CPU (gloo, world_size 2): replicas are independent, the
timing is the max over ranks and `value` is the whole-job aggregate
(the path does not shard, so there is no data-path collective)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ws, r, local = bench._dist()
        assert (ws, r, local) == (world, rank, rank)
        # rank-dependent local durations: the slowest replica sets the clock
        local_s = 0.5 + rank
        m = bench.max_over_ranks(local_s, dist)
        out[rank] = (m, bench.replica_value(8, 100, ws, m))
        # each replica runs its own independent forward on its own batch; the
        # lowered CPU program needs no collective to agree with the oracle
        from oracle import executor as orc
        from paper_2509_16248_b200 import lowering
        from paper_2509_16248_b200.harness import programs

        p = programs()["phi4_like"]
        spec = p["inputs"][rank % len(p["inputs"])]
        args = orc.make_args(spec["args"], spec["seed"])
        mod, _ = lowering.load(p["transformed"], allow_eager=True)
        ref, _ = orc.run_reference(p["transformed"], p["callable"], args)
        assert torch.equal(getattr(mod, p["callable"])(*args), ref)
    finally:
        dist.destroy_process_group()


def test_two_replicas_gloo():
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == pytest.approx(1.5)
    # 2 replicas x 8 samples x 100 steps in 1.5 s
    assert res[0][1] == pytest.approx(2 * 8 * 100 / 1.5)

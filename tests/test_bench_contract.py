"""bench.py's one-line JSON contract (the driver parses it): the reference
arm on the CPU, the B200 arm on a GPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"])
    assert d["impl"] == "reference"
    assert d["unit"] == "samples/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("bigbird_layer") and d["dtype"] == "fp32"
    assert set(d["config"]) == {"workload", "batch", "shape", "inputs"}   # identical keys in both arms


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run(["--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-compile"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "speculation"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["dtype"] == "fp32"
    assert set(d["config"]) == {"workload", "batch", "shape", "inputs"}
    assert d["host_syncs_per_forward"] == 0 and d["mode"] == "graph"
    assert d["host_syncs_profiler"]["cuda_syncs"] == 0 and d["host_syncs_profiler"]["d2h_copies"] == 0
    # config 2 as a full encoder layer: the predicate's grid region, the
    # softmax row region, the residual adds, GELU, the two LayerNorm row
    # regions, the head split / merge gathers and the fp32 GEMMs (BF16x9)
    assert d["gpu_launches_per_forward"] >= 12 and d["gpu_launches"] == 5 * d["gpu_launches_per_forward"]
    sp = d["speculation"]
    assert sp["launches"] == 0 and sp["mispredictions"] == 0   # a one-pass predicate feeding a row kernel
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 8 * 1024 * 768 * 4
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert r["kernel"].startswith("gm_row_")          # the softmax arms dominate
    # grid and row kernels time themselves inside the timed loop (in-kernel
    # %globaltimer, one launch per step and region), never longer than CUDA
    # events around their launch in a replay of the same graph
    for k in d["kernels"]:
        assert k["name"].startswith(("gm_region_", "gm_row_")), k["name"]
        assert k["how"].startswith("live, in-kernel") and "over the 5 launches" in k["how"], k["how"]
        assert 0 < k["ms"] <= k["ms_events"] * 1.05, (k["ms"], k["ms_events"])
    assert set(r["fused_kernels_frac"]) == {k["name"].split(" ")[0] for k in d["kernels"]}
    assert 0 < r["frac_nominal_8tbs"] < r["frac"]


@pytest.mark.gpu
def test_two_replicas_end_to_end():
    """bench.py --gpus 2 under torchrun, as the driver launches the scaling
    run: two independent replica processes (sharing the GPU on a 1-GPU box),
    gloo for the timing barrier only, the max over ranks, ONE JSON line from
    rank 0 whose value aggregates both replicas' samples."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-compile"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["steps"] == 5
    assert d["host_syncs_per_forward"] == 0 and d["mode"] == "graph"
    # value = both replicas' samples over the max-over-ranks time
    assert d["value"] == pytest.approx(2 * d["config"]["batch"] * 5 / (d["ms_per_step"] * 5 / 1e3), rel=1e-6)

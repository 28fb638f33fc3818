"""GraphMend-transformed programs on the B200 path vs the reference's CPU
eager execution of the same text (the oracle), through the harness call
shape (runner.py:154-157): outputs within the north_star tolerance, side
effect text identical and in order, fused regions actually launched, zero
host syncs inside the forward when the reference reports 0 residual breaks."""

import pytest
import torch

from oracle import executor as orc
from paper_2509_16248_b200 import harness
from parity import has_row_reduction, rowop_fp64_reference, assert_parity, check_scalars, has_dense_contraction, torch_cuda_reference

CORPUS = ["biogpt_like", "blenderbot_like", "flan_t5_like", "longformer_like", "moe_minicpm_like",
          "pegasus_like", "phi4_like", "qwen_audio_like"]
WORKLOADS = ["toy", "bigbird_like", "bart_step", "gemm_arms", "bigbird_attn", "bigbird_layer"]


def _run(programs, name, idx, dtype=None, scaled=False):
    prog = programs[name]
    spec = prog["inputs"][idx]
    shapes = prog.get("scaled_shapes") if scaled else None
    args = orc.make_args(spec["args"], spec["seed"], dtype, shapes)
    ref_out, ref_text = orc.run_reference(prog["transformed"], prog["callable"], args, dtype)
    ex, mod, low, _ = harness.b200_program(name, dtype=dtype)
    out, text = harness.call_captured(ex, [a.cuda() for a in args])
    # branch decisions = the oracle's; predicate statistics within tolerance
    check_scalars(low, prog["transformed"], prog["callable"], args, dtype, what=f"{name}[{idx}]")
    noise = []
    if isinstance(ref_out, torch.Tensor) and has_dense_contraction(prog["transformed"]):
        noise.append(torch_cuda_reference(prog["transformed"], prog["callable"], args, dtype))
    if isinstance(ref_out, torch.Tensor) and has_row_reduction(prog["transformed"]):
        noise.append(rowop_fp64_reference(prog["transformed"], prog["callable"], args, dtype))
    return prog, ref_out, ref_text, out, text, ex, low, noise


def _check(prog, name, ref_out, ref_text, out, text, ex, low, dtype, noise=None):
    if isinstance(ref_out, torch.Tensor):
        assert_parity(out, ref_out, dtype or torch.float32, what=name, noise=noise)
    if prog.get("compare_output_text", True):
        assert text == ref_text, (name, text, ref_text)
    info = ex.info()[0]
    # every corpus program and stand-in is sync-free on the B200 path — the
    # 15 dynamic-shape sites of moe_minicpm_like and the 3 .item() reads of
    # longformer_like included, although the
    # reference reports them unfixable (its counts stay the parity target)
    assert info.mode == "graph", (name, info)
    assert info.host_syncs == 0, (name, info)
    # every region of every program runs the sm_100a kernel (no region of
    # the corpus or the stand-ins falls back to PyTorch ops)
    for r in low.regions:
        assert r.stats.launches > 0 and r.stats.fallbacks == 0, (name, r.name, r.stats.fallback_reasons)
    return info


@pytest.mark.gpu
@pytest.mark.parametrize("name", CORPUS)
def test_corpus_manifest_shapes(programs, name):
    """Every manifest input at the corpus' own shapes (latency-bound)."""
    for idx in range(len(programs[name]["inputs"])):
        prog, ref_out, ref_text, out, text, ex, low, noise = _run(programs, name, idx)
        _check(prog, name, ref_out, ref_text, out, text, ex, low, None, noise)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("name", CORPUS)
def test_corpus_baseline_shapes(programs, name, dtype):
    """Config 3/5: corpus programs with every tensor at the BASELINE shape."""
    prog = programs[name]
    for idx in range(len(prog["inputs"])):
        prog, ref_out, ref_text, out, text, ex, low, noise = _run(programs, name, idx, dtype, scaled=True)
        _check(prog, name, ref_out, ref_text, out, text, ex, low, dtype, noise)
        fused = [r for r in low.regions if r.stats.launches > 0]
        assert fused, f"{name}: no fused region launched ({[r.stats.fallback_reasons for r in low.regions]})"


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["fp32", "bf16"])
@pytest.mark.parametrize("name", WORKLOADS)
def test_workloads(programs, name, dtype):
    """Configs 1, 2, 4: the BASELINE-shaped stand-ins."""
    prog = programs[name]
    for idx in range(len(prog["inputs"])):
        prog, ref_out, ref_text, out, text, ex, low, noise = _run(programs, name, idx, dtype)
        _check(prog, name, ref_out, ref_text, out, text, ex, low, dtype, noise)


@pytest.mark.gpu
def test_host_pipeline_matches_single_calls(programs):
    """B200Executor.run_host_pipelined (pipelined H2D / replay / D2H over rotating graph slots)
    returns, batch by batch, exactly what single calls return."""
    prog = programs["bigbird_like"]
    ex, mod, low, _ = harness.b200_program("bigbird_like", dtype=torch.bfloat16)
    batches = []
    for spec in prog["inputs"]:
        args = orc.make_args(spec["args"], spec["seed"], torch.bfloat16)
        batches.append(tuple(a.pin_memory() for a in args))
    singles = [ex(*b).cpu().clone() for b in batches]
    outs = ex.run_host_pipelined(batches * 3)
    ex.flush()
    for k, o in enumerate(outs):
        assert torch.equal(o, singles[k % len(batches)]), k


@pytest.mark.gpu
def test_aot_cubins_are_used(programs):
    """build() precompiled the BASELINE workloads' regions: the GPU run finds
    the same specialisations in the cubin cache (no NVRTC at first call)."""
    import os

    from paper_2509_16248_b200 import region as reg

    prog = programs["bigbird_like"]
    spec = prog["inputs"][0]
    args = orc.make_args(spec["args"], spec["seed"], torch.bfloat16)
    if not any(os.path.exists(p) for p in [reg.KCACHE_DIR]):
        pytest.skip("no AOT cache (build() not run)")
    ex, mod, low, _ = harness.b200_program("bigbird_like", dtype=torch.bfloat16)
    ex(*[a.cuda() for a in args])
    ex.flush()
    for r in low.regions:
        assert r.last_spec is not None and r.last_spec.kernel.from_cache, r.name


@pytest.mark.gpu
def test_bound_entry_reads_inputs_in_place(programs):
    """B200Executor.bind: the graph is captured on the caller's tensors; a
    serving loop refills them in place and replays with no input copy —
    each replay equals a fresh call on the same values."""
    prog = programs["bigbird_like"]
    ex, mod, low, _ = harness.b200_program("bigbird_like", dtype=torch.bfloat16)
    specs = prog["inputs"]
    first = orc.make_args(specs[0]["args"], specs[0]["seed"], torch.bfloat16)[0].cuda()
    entry = ex.bind(first)
    assert entry.info.mode == "graph"
    for spec in specs:
        x = orc.make_args(spec["args"], spec["seed"], torch.bfloat16)[0].cuda()
        first.copy_(x)
        out = entry.run().clone()
        ex.flush()
        ref = ex(x).clone()
        ex.flush()
        assert torch.equal(out, ref)

"""Generate tests/golden/ from the reference (build container only).

    python oracle/gen_fixtures.py            # needs /root/reference

1. programs.json — for the 8 corpus cases (pkg/corpus/*) and this repo's
   BASELINE-shaped stand-ins (workloads/*): the original text, the text the
   reference `fix_file` returns (transform.py:822-936), its FileOutcome
   (found / fixed / skipped / unfixable / predicted_residual, per-site status,
   transform.py:778-819), the manifest fields the harness reads
   (runner.py:56-75) and, for the sweep, the BASELINE shapes.
2. corpus_harness.json — the reference harness's own results on the corpus
   (runner.py:180-238, run_suite :291-353): per input the output tensor and
   side-effect lines of the transformed program, plus measured break counts.
   These are the golden vectors the oracle executor is pinned against.

Nothing here runs on the GPU box: /root/reference does not exist there.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg")
REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"

# BASELINE shapes for the 8-model sweep (config 5) and longformer (config 3)
BB = [8, 1024, 768]
SCALED = {
    "biogpt_like": [BB, BB],
    "blenderbot_like": [BB],
    "flan_t5_like": [[8192, 768], [768, 768]],
    "longformer_like": [[4, 4096, 768]],
    "moe_minicpm_like": [BB],
    "pegasus_like": [BB],
    "phi4_like": [BB],
    "qwen_audio_like": [BB],
}


def _outcome(o) -> dict:
    return {
        "status": o.status,
        "found": o.found,
        "fixed": o.fixed,
        "skipped": o.skipped_count,
        "unfixable": o.unfixable,
        "predicted_residual": o.predicted_residual,
        "sites": [
            {"line": s.line, "col": s.col, "kind": s.kind, "status": s.status, "reason": s.reason,
             "runtime_effective": s.runtime_effective}
            for s in o.sites
        ],
    }


def _tensor_json(t):
    import torch

    if not isinstance(t, torch.Tensor):
        return {"python": repr(t)}
    return {"dtype": str(t.dtype), "shape": list(t.shape),
            "values": [float.hex(float(v)) for v in t.detach().double().reshape(-1).tolist()]}


def main() -> None:
    sys.path.insert(0, str(REF / "src"))
    sys.path.insert(0, str(REF / "harness" / "src"))
    from graphmend import SourceModule, fix_file
    from graphmend_harness import runner

    programs = {}
    for case in sorted(p.parent.name for p in (REF / "corpus").glob("*/manifest.json")):
        d = REF / "corpus" / case
        man = json.loads((d / "manifest.json").read_text())
        text = (d / "original.py").read_text()
        new_text, outcome = fix_file(SourceModule.from_text(f"corpus/{case}/original.py", text))
        programs[case] = {
            "kind": "corpus",
            "config": 3 if case == "longformer_like" else 5,
            "callable": man["callable"],
            "inputs": man["inputs"],
            "explain_input": man.get("explain_input", 0),
            "expected_breaks_before": man["expected_breaks_before"],
            "expected_breaks_after": man["expected_breaks_after"],
            "compare_output_text": man.get("compare_output_text", True),
            "expected_output_text": man.get("expected_output_text"),
            "expected_tags": json.loads((d / "expected_tags.json").read_text()),
            "scaled_shapes": SCALED[case],
            "original": text,
            "transformed": new_text,
            "outcome": _outcome(outcome),
        }
    for wd in sorted((REPO / "workloads").glob("*/spec.json")):
        spec = json.loads(wd.read_text())
        text = (wd.parent / "program.py").read_text()
        new_text, outcome = fix_file(SourceModule.from_text(f"workloads/{spec['name']}/program.py", text))
        programs[spec["name"]] = {
            "kind": "workload",
            "config": spec["config"],
            "callable": spec["callable"],
            "inputs": spec["inputs"],
            "explain_input": 0,
            "expected": spec["expected"],
            "original": text,
            "transformed": new_text,
            "outcome": _outcome(outcome),
        }
    # the reference's unit fixtures (pkg/tests/fixtures/units/*.py): the
    # rewrite shapes its own tests pin (test_transform.py), run through the
    # B200 path by tests/test_gpu_units.py on branch-forcing inputs
    for up in sorted((REF / "tests" / "fixtures" / "units").glob("*.py")):
        text = up.read_text()
        new_text, outcome = fix_file(SourceModule.from_text(f"units/{up.name}", text))
        programs[f"unit:{up.stem}"] = {
            "kind": "unit",
            "original": text,
            "transformed": new_text,
            "outcome": _outcome(outcome),
        }
    GOLDEN.mkdir(parents=True, exist_ok=True)
    (GOLDEN / "programs.json").write_text(json.dumps(programs, indent=1, sort_keys=True) + "\n")

    # reference harness on the corpus (its own code path, in a temp workdir)
    with tempfile.TemporaryDirectory() as tmp:
        env_path = os.environ.get("PYTHONPATH", "")
        os.environ["PYTHONPATH"] = f"{REF / 'src'}:{REF / 'harness' / 'src'}:{env_path}"
        summary = runner.run_suite(REF / "corpus", Path(tmp) / "summary.json", Path(tmp) / "cases")
        golden = {"suite": {k: summary[k] for k in ("passed", "failed", "agreement", "fully_clean", "partial",
                                                    "unchanged")},
                  "cases": {}}
        for c in summary["cases"]:
            golden["cases"][c["name"]] = {k: c[k] for k in ("breaks_before", "breaks_after", "pass",
                                                             "predicted_residual", "primary_fixed",
                                                             "primary_unfixable", "max_rel_diff")}
        for case in sorted(programs):
            p = programs[case]
            if p["kind"] != "corpus":
                continue
            case_dir = Path(tmp) / "cases" / case
            fc = runner.FixtureCase.from_manifest(case_dir)
            mod = runner._load_module(fc.transformed_path, f"{case}_golden")
            fn = getattr(mod, fc.callable_name)
            runs = []
            for spec in fc.inputs:
                args = runner._make_args(spec.args, spec.seed)
                out, text = runner._call_captured(fn, args)
                runs.append({"note": spec.note, "seed": spec.seed, "output": _tensor_json(out), "text": text})
            golden["cases"][case]["runs"] = runs
    (GOLDEN / "corpus_harness.json").write_text(json.dumps(golden, indent=1, sort_keys=True) + "\n")
    print(f"wrote {GOLDEN / 'programs.json'} ({len(programs)} programs) and corpus_harness.json")


if __name__ == "__main__":
    main()

"""ORACLE — test infrastructure only.

CPU restatement of the reference's hot path: the GraphMend-transformed
program executed eagerly on CPU through the harness call shape
(pkg/harness/src/graphmend_harness/runner.py:105-177).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this package, and only as the checker or the timed CPU baseline;
the product (paper_2509_16248_b200/) never does.

Pinning: the transformed programs and their break counts come from the
reference's own `fix_file` (transform.py:822-936), generated in the build
container by oracle/gen_fixtures.py into tests/golden/programs.json, and are
checked against the reference's sidecars (corpus/*/expected_tags.json), its
fix-rate table (tests/test_acceptance.py:33-42), the manifests' expected
break counts and expected log text, and the reference harness's own outputs
on the corpus (tests/golden/corpus_harness.json).  The arithmetic itself is
PyTorch's CPU kernels (third-party, torch 2.11.0 in this image), which is
exactly what the reference harness runs.
"""

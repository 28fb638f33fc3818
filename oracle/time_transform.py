"""One-time cost of the reference transform ("Transform
(`fix_file`) time is reported separately as a one-time cost").

Runs the reference's own `fix_file` (transform.py:822-936) on every program
of tests/golden/programs.json that came from a source file (corpus cases and
the BASELINE stand-ins), 20 times each after one warm-up, and writes the
median milliseconds to tests/golden/transform_times.json.  Test
infrastructure: it imports the reference from /root/reference, which exists
only in the build container — bench.py reports the committed numbers.

    python oracle/time_transform.py
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.gen_fixtures import REF  # noqa: E402


def main() -> None:
    sys.path.insert(0, str(REF / "src"))
    from graphmend import SourceModule, fix_file

    progs = json.load(open(os.path.join(ROOT, "tests", "golden", "programs.json")))
    out = {}
    for name, p in sorted(progs.items()):
        if name.startswith("unit:") or "original" not in p:
            continue
        src = SourceModule.from_text(f"{name}.py", p["original"])
        fix_file(src)
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            fix_file(src)
            ts.append(time.perf_counter() - t0)
        out[name] = round(1e3 * statistics.median(ts), 3)
    with open(os.path.join(ROOT, "tests", "golden", "transform_times.json"), "w") as fh:
        json.dump({"how": "reference fix_file (transform.py:822-936), median of 20 after 1 warm-up, "
                          "build container CPU, one-time per program", "ms": out}, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

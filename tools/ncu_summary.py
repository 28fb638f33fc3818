"""Summarise an ncu capture into profiles/ (run in the build container).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_regions.json

Per kernel launch: duration, DRAM bytes read/written (the `traffic` the bench
line reports), achieved DRAM throughput, SM throughput, registers, occupancy
and the top warp-stall reasons."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "warp_instructions",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
              "msecond": 1e6, "ms": 1e6}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * UNIT_SCALE.get(units[i], 1)
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i])))
                except ValueError:
                    pass
        stalls.sort(key=lambda x: -x[1])
        d["top_stalls"] = stalls[:5]
        if "dram_read" in d:
            d["traffic_bytes"] = d["dram_read"] + d.get("dram_write", 0.0)
        res.append(d)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    for d in res:
        print(d["kernel"][:40], {k: d.get(k) for k in ("duration_ns", "traffic_bytes", "dram_pct", "sm_pct")})


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

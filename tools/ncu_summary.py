"""Summarises ncu --set full reports of the step kernel into profiles/ (JSON + markdown rows).

usage: python tools/ncu_summary.py OUT.json name=path.ncu-rep|raw.csv [...] [--bnode 304 --nodes N]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "registers": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "msecond": 1e3, "usecond": 1.0,
        "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3}


def read(path):
    """path[@k]: the k-th profiled launch of the report (default the first)."""
    k = 0
    if "@" in path:
        path, k = path.rsplit("@", 1)
        k = int(k)
    if path.endswith(".csv"):  # an exported `ncu -i REP --page raw --csv` page
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2 + k]
    rec = {"kernel": v[h.index("Kernel Name")]}
    for k, m in KEYS.items():
        if m in h:
            i = h.index(m)
            val = float(v[i].replace(",", ""))
            unit = u[i]
            if k.endswith("_bytes"):
                val *= UNIT.get(unit, 1.0)
            if k == "duration_us":
                val *= UNIT.get(unit, 1.0)
            rec[k] = val
    stalls = []
    for i, name in enumerate(h):
        if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
            try:
                stalls.append((float(v[i]), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    rec["top_stalls_pct"] = {n: round(100 * s / tot, 1) for s, n in sorted(stalls, reverse=True)[:5]}
    rec["dram_bytes_per_launch"] = rec.get("dram_read_bytes", 0) + rec.get("dram_write_bytes", 0)
    return rec


if __name__ == "__main__":
    out = sys.argv[1]
    res = {}
    for arg in sys.argv[2:]:
        name, path = arg.split("=", 1)
        res[name] = read(path)
        print(name, json.dumps(res[name]))
    json.dump(res, open(out, "w"), indent=1)

#!/usr/bin/env python
"""Summarise ncu --set full captures into profiles/ (measurement tool).

    python tools/ncu_summary.py OUT.md NAME=path.ncu-rep[:algorithmic_bytes] ...

Writes one markdown table (metric rows x capture columns) plus, per capture,
the raw page as CSV next to OUT.md (OUT_<NAME>_raw.csv), and updates
profiles/ncu_traffic.json entries given as NAME=...@workload:nN.
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("Kernel Name", None),
    ("gpu__time_duration.sum", None),
    ("dram__bytes_read.sum", None),
    ("dram__bytes_write.sum", None),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", None),
    ("launch__registers_per_thread", None),
    ("launch__grid_size", None),
    ("launch__block_size", None),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", None),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", None),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    ("smsp__inst_executed.sum", None),
    ("sm__cycles_elapsed.avg.per_second", None),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2], out


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def to_seconds(v, unit):
    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}.get(unit, 1e-9)
    return float(v.replace(",", "")) * scale


def main():
    out_md = sys.argv[1]
    caps = []
    for arg in sys.argv[2:]:
        name, rest = arg.split("=", 1)
        key = None
        if "@" in rest:
            rest, key = rest.split("@", 1)
        path, _, algo = rest.partition(":")
        hdr, units, vals, text = raw(path)
        base = os.path.splitext(out_md)[0]
        with open(f"{base}_{name}_raw.csv", "w") as f:
            f.write(text)
        caps.append((name, dict(zip(hdr, zip(vals, units))), float(algo) if algo else None, key))
    lines = ["| metric | " + " | ".join(c[0] for c in caps) + " |", "|---|" + "---|" * len(caps)]
    for m, _ in METRICS:
        cells = []
        for _, d, _, _ in caps:
            v, u = d.get(m, ("", ""))
            cells.append((v[:70] if m == "Kernel Name" else f"{v} {u}").strip())
        lines.append(f"| `{m}` | " + " | ".join(cells) + " |")
    derived = []
    for name, d, algo, key in caps:
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        t = to_seconds(*d["gpu__time_duration.sum"])
        line = f"* **{name}**: DRAM traffic {(rd + wr) / 1e9:.4f} GB per launch, {(rd + wr) / t / 1e9:.0f} GB/s under ncu"
        if algo:
            line += f"; algorithmic {algo / 1e9:.4f} GB -> traffic / algorithmic = {(rd + wr) / algo:.4f}"
        derived.append(line)
        if key:
            tj = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
            db = json.load(open(tj)) if os.path.exists(tj) else {}
            db[key] = {"dram_bytes_per_launch": int(round(rd + wr)), "kernel": d["Kernel Name"][0][:80],
                       "source": os.path.basename(f"{os.path.splitext(out_md)[0]}_{name}_raw.csv")}
            json.dump(db, open(tj, "w"), indent=1)
    with open(out_md, "w") as f:
        f.write("\n".join(lines + [""] + derived) + "\n")
    print(open(out_md).read())


if __name__ == "__main__":
    main()

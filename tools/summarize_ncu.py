"""Summaries for profiles/: per-kernel launch shares from an `ncu --metrics
gpu__time_duration.sum --csv` log, and key metrics from an `ncu --set full` report."""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            nm = d["Kernel Name"].split("(")[0].replace("void ", "")
            agg[nm][0] += 1
            agg[nm][1] += float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
    tot = sum(v for _, v in agg.values()) or 1
    out = ["| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {c} | {v:.1f} | {100 * v / tot:.1f}% |")
    return "\n".join(out)


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Achieved Occupancy",
        "Registers Per Thread", "Executed Ipc Active", "Grid Size", "Block Size", "Compute (SM) Throughput"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h = rows[0]
    per = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in WANT:
            key = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", ""))
            per[key][d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    dram = {}
    if rr:
        hh = rr[0]
        for r in rr[2:]:
            d = dict(zip(hh, r))
            try:
                rd = float(d.get("dram__bytes_read.sum", "nan").replace(",", ""))
                wr = float(d.get("dram__bytes_write.sum", "nan").replace(",", ""))
                dram[d["ID"]] = (rd, wr, hh)
            except ValueError:
                pass
    out = []
    for (i, k), m in sorted(per.items(), key=lambda x: int(x[0][0])):
        extra = ""
        if i in dram:
            extra = f"; dram read {dram[i][0]:.3g} + write {dram[i][1]:.3g} (units per ncu raw page)"
        out.append(f"- `{k}` (ID {i}): " + "; ".join(f"{a} {b}" for a, b in m.items()) + extra)
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))

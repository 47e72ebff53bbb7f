"""Markdown tables of a tools/sweep.py result: M txn/s per (n, theta) for each strategy.
   python tools/sweep_table.py gpurun_out/sweep.json"""
import json
import sys

d = json.load(open(sys.argv[1]))
rows = d["rows"]
thetas = sorted({r["theta"] for r in rows})
ns = sorted({r["n"] for r in rows})
strats = []
for r in rows:
    if r["strategy"] not in strats:
        strats.append(r["strategy"])
cell = {(r["n"], r["theta"], r["strategy"]): r for r in rows}
print(f"{d['config']}; median of {d['steps']} bulks; M txn/s (submit + execute, device-resident)\n")
print("| n | " + " | ".join(f"θ={t}: " + " / ".join(strats) for t in thetas) + " |")
print("|---|" + "---|" * len(thetas))
for n in ns:
    out = []
    for t in thetas:
        vals = []
        for s in strats:
            r = cell.get((n, t, s))
            if not r:
                vals.append("—")
            elif r["result"] != "ok":
                vals.append("t/o")
            else:
                v = f"{r['txn_per_s'] / 1e6:.1f}"
                if s == "auto":
                    v += f"({r.get('chose', '?')[0]})"
                vals.append(v)
        out.append(" / ".join(vals))
    print(f"| 2^{n.bit_length() - 1} | " + " | ".join(out) + " |")
print("\nK-SET depth d (rank passes) per point:\n")
print("| n | " + " | ".join(f"θ={t}" for t in thetas) + " |")
print("|---|" + "---|" * len(thetas))
for n in ns:
    out = []
    for t in thetas:
        r = cell.get((n, t, "kset"))
        out.append(f"{r['depth']} ({r['rank_passes']})" if r and r["result"] == "ok" else "—")
    print(f"| 2^{n.bit_length() - 1} | " + " | ".join(out) + " |")

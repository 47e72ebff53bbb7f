"""Top SASS instructions by warp-stall samples from an ncu report (source page).
   python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
h = r[1]
idx = {k: i for i, k in enumerate(h)}
rows = [x for x in r[2:] if len(x) == len(h)]
key = "Warp Stall Sampling (All Samples)"
f = lambda x, k: float((x[idx[k]] or "0").replace(",", ""))
tot = sum(f(x, key) for x in rows) or 1
print("total samples", tot, "instructions executed", sum(f(x, "Instructions Executed") for x in rows))
for x in sorted(rows, key=lambda x: -f(x, key))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{x[idx['Address']]:>8} {100 * f(x, key) / tot:5.1f}%  ex={x[idx['Instructions Executed']]:>10}  {x[idx['Source']][:100]}")

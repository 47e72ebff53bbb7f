"""Per-bulk kernel durations (us) from an ncu --metrics gpu__time_duration.sum launch list:
the last bulk's launches (from the last fill_multi before the last ingest)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
ing = [i for i, d in enumerate(data) if d["Kernel Name"].startswith("void ingest_kernel")]
start = ing[-1] - 1 if len(ing) else 0
tot = 0.0
for d in data[start:]:
    us = float(d["Metric Value"].replace(",", "")) / 1e3
    tot += us
    print(f"{us:8.1f}  {d['Kernel Name'][:70]}")
print(f"{tot:8.1f}  total, {len(data) - start} launches")

"""Record DRAM traffic per launch from an `ncu --set full` capture into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).

  python tools/ncu_traffic.py <workload> <report.ncu-rep> [<kernel-name-prefix> ...]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3}


def raw_csv(path):
    if path.endswith(".csv"):                 # a raw page already exported on the GPU box
        return open(path).read()
    return subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout


def rows(raw):
    r = list(csv.reader(raw.splitlines()))
    h, u = r[0], r[1]
    for v in r[2:]:
        yield {k: (x, uu) for k, x, uu in zip(h, v, u)}


def main():
    wl, path = sys.argv[1], sys.argv[2]
    prefixes = sys.argv[3:]
    out_p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    db = json.load(open(out_p)) if os.path.exists(out_p) else {}
    agg = {}
    raw = raw_csv(path)
    # the raw page (every metric of every captured launch) is kept under profiles/
    keep = os.path.join(ROOT, "profiles", "ncu_raw_" + os.path.basename(path).replace(".ncu-rep", ".csv"))
    open(keep, "w").write(raw)
    for d in rows(raw):
        name = d["Kernel Name"][0].split("(")[0].split("<")[0].replace("void ", "").replace("gputx::", "")
        if prefixes and not any(name.startswith(p) for p in prefixes):
            continue
        val = lambda k: float(d[k][0].replace(",", "")) * SCALE.get(d[k][1], 1)
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        a[2] += val("gpu__time_duration.sum")
        a[3] += float(d["lts__t_sector_hit_rate.pct"][0])
    for name, (c, b, t, hit) in agg.items():
        db.setdefault(wl, {})[name] = {"dram_bytes_per_launch": b / c, "ncu_us_per_launch": t / c,
                                       "l2_hit_pct": hit / c, "launches": c,
                                       "source": os.path.relpath(keep, ROOT)}
        print(wl, name, db[wl][name])
    json.dump(db, open(out_p, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

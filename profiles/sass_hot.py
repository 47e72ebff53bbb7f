"""Summarise an `ncu --page source --csv --print-source sass` dump: hottest SASS
instructions by warp-stall samples, plus the stall-reason columns."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    samp = idx["Warp Stall Sampling (All Samples)"]
    data = []
    for r in rows[2:]:
        if len(r) < len(h) - 1:
            continue
        try:
            v = float(r[samp])
        except ValueError:
            continue
        data.append((v, r[idx["Address"]][-5:], r[idx["Source"]].strip()))
    tot = sum(d[0] for d in data) or 1
    print(f"total samples {tot:.0f}")
    for v, a, s in sorted(data, reverse=True)[:top]:
        print(f"{100 * v / tot:5.1f}%  {a}  {s[:90]}")
    # stall reason columns
    reasons = [k for k in h if k.startswith("stall_") or "Stall" in k and "Sampling" not in k]
    agg = {}
    for k in reasons:
        s = 0.0
        for r in rows[2:]:
            try:
                s += float(r[idx[k]])
            except (ValueError, IndexError):
                pass
        agg[k] = s
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        if v:
            print(f"  {k}: {v:.0f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

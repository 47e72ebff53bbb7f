"""Diagnostics: TM-1 K-SET rank / exec phase times for NURand and uniform subscriber draws."""
import sys

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

dims = W.Tm1Dims(1_000_000)
image = W.make_db(W.TM1, dims, seed=1)
for dist in ("nurand", "uniform"):
    bulk = W.make_bulk(W.TM1, dims, 1_000_000, seed=2, dist=dist)
    db = Database(W.TM1, dims.dims, 1_000_000, image, insert_capacity=8)
    ms = []
    for it in range(6):
        db.submit(bulk)
        st = db.execute("kset")
        ms.append((st["ms_sort"], st["ms_rank"], st["ms_group"], st["ms_exec"]))
    best = [min(m[i] for m in ms[2:]) for i in range(4)]
    print(f"{dist}: ksets {st['ksets']} sort {best[0]:.3f} rank {best[1]:.3f} group {best[2]:.3f} exec {best[3]:.3f} ms")
    db.close()

"""Diagnostics: TM-1 PART phase times vs partition size (subscribers per partition)."""
import sys

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

dims = W.Tm1Dims(1_000_000)
image = W.make_db(W.TM1, dims, seed=1)
bulk = W.make_bulk(W.TM1, dims, 1_000_000, seed=2, dist="nurand")
for ps in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,4,16,128").split(",")]:
    db = Database(W.TM1, dims.dims, 1_000_000, image, insert_capacity=8, part_size=ps)
    best = None
    for it in range(5):
        db.submit(bulk)
        st = db.execute("part")
        t = (st["ms_total"], st["ms_emit"], st["ms_sort"], st["ms_exec"], st["max_chain"])
        best = t if best is None or t[0] < best[0] else best
    print(f"part_size {ps}: total {best[0]:.3f} emit {best[1]:.3f} sort {best[2]:.3f} exec {best[3]:.3f} ms, max chain {best[4]}")
    db.close()

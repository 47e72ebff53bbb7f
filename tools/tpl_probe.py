"""TPL timing on one workload (for wait-policy experiments)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "tpcb"]
strategies = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tpl"]
dims, image, bulks = bench.make_inputs(wl, 0, 1, 2, 1)
db = Database(wl["schema"], dims.dims, wl["n"], image, insert_capacity=4)
for s in strategies:
    for k in range(3):
        db.reset()
        db.submit(bulks[0])
        st = db.execute(s)
    print(f"{sys.argv[1]} {s}: exec_ms {st['ms_exec']:.3f} total_ms {st['ms_total']:.3f}", flush=True)

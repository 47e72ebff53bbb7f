"""Run one warm-up and one measured bulk of a bench workload (for ncu captures)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "tm1"]
strategy = sys.argv[2] if len(sys.argv) > 2 else "kset"
dims, image, bulks = bench.make_inputs(wl, 0, 1, 2, 1)
db = Database(wl["schema"], dims.dims, wl["n"], image, insert_capacity=4, packed_out=True)   # as bench.py
for b in bulks[:2]:
    db.submit(b)
    st = db.execute(strategy)
print({k: st[k] for k in ("ms_sort", "ms_rank", "ms_group", "ms_exec", "rank_passes", "ksets")})

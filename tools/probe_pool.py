"""Diagnostics: per-tick costs of the streaming K-SET pool (submit, step, read) on TM-1."""
import sys
import time

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

per = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
dist = sys.argv[2] if len(sys.argv) > 2 else "nurand"
dims = W.Tm1Dims(1_000_000)
image = W.tm1_db(dims, seed=1)
arr = W.tm1_bulk(dims, per * 20, seed=11, dist=dist)
db = Database(W.TM1, dims.dims, 1 << 22, image, insert_capacity=1)
db.pool_submit(arr.slice(0, 1000)); db.pool_step(); db.reset()
for k in range(20):
    t0 = time.perf_counter()
    db.pool_submit(arr.slice(k * per, (k + 1) * per))
    t1 = time.perf_counter()
    s = db.pool_step()
    t2 = time.perf_counter()
    db.pool_read()
    t3 = time.perf_counter()
    print(f"tick {k}: pool_before {db.pool_pending() + s['executed']} executed {s['executed']} "
          f"submit {1e3*(t1-t0):.2f} ms step {1e3*(t2-t1):.2f} ms (dev zs {s['ms_rank']:.3f} exec {s['ms_exec']:.3f} "
          f"compact {s['ms_merge']:.3f}) read {1e3*(t3-t2):.2f} ms", flush=True)

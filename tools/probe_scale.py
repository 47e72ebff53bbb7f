"""K-SET executor per-round cost vs table size (TLB / cache footprint probe)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

for P in [int(x) for x in sys.argv[1:]] or [100_000, 1_000_000]:
    dims = W.Tm1Dims(P)
    db = Database(W.TM1, dims.dims, 1_000_000, W.tm1_db(dims, seed=1))
    bulk = W.tm1_bulk(dims, 1_000_000, seed=2, dist="uniform")
    db.trace_rounds(True)
    for _ in range(3):
        db.submit(bulk)
        s = db.execute("kset")
    raw = db.round_ns(s["ksets"]).astype(np.int64)
    dt = np.diff(raw[:, 0]) / 1e3
    print(f"P={P}: ksets {s['ksets']} exec_ms {s['ms_exec']:.3f} round us {np.round(dt[:6], 1)} "
          f"cta0 work us {np.round((raw[:6, 6] - raw[:6, 0]) / 1e3, 1)}")
    db.close()

"""Latency of single transactions in the K-SET executor on an idle GPU."""
import sys
import numpy as np
sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

dims = W.TpccDims(64, 10, 3000, 100_000)
db = Database(W.TPCC, dims.dims, 100_000, W.tpcc_db(dims, seed=1))
db.trace_rounds(True)
for n in (1, 1, 8, 64, 600):
    bulk = W.tpcc_bulk(dims, n, seed=n, mix=(1, 0))          # NewOrders only
    db.submit(bulk)
    s = db.execute("kset")
    raw = db.round_ns(s["ksets"]).astype(np.int64)
    sl = raw[:, 3]
    print(f"n={n}: ksets {s['ksets']} exec_ms {s['ms_exec']:.3f} slowest txn us {np.round((sl >> 24) / 1e3, 1)[:4]} "
          f"round us {np.round(np.diff(raw[:, 0]) / 1e3, 1)[:4]} cta0 work {np.round((raw[:4, 6] - raw[:4, 0]) / 1e3, 1)}")

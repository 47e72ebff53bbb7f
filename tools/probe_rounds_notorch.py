"""Diagnostics: per-round K-SET executor timing and k-set size distribution."""
import sys
import time

import numpy as np


sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "tm1"
if wl == "tm1":
    schema, dims, n, kw = W.TM1, W.Tm1Dims(1_000_000), 1_000_000, dict(dist="nurand")
elif wl == "tpcb":
    schema, dims, n, kw = W.TPCB, W.TpcbDims(1000, 10, 100_000), 4_000_000, dict(remote_pct=15.0)
else:
    schema, dims, n, kw = W.TPCC, W.TpccDims(64, 10, 3000, 100_000), 1_000_000, {}
image = W.make_db(schema, dims, seed=1)
bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
db = Database(schema, dims.dims, n, image, insert_capacity=8)
db.trace_rounds(True)
for it in range(3):
    db.submit(bulk)
    st = db.execute("kset")
nk = st["ksets"]
raw = db.round_ns(nk).astype(np.int64)
tr = raw[:, :4]
spins = np.zeros((nk, 4), np.int64)
spins[:-1, 1] = raw[1:, 4]
spins[:-1, 3] = raw[1:, 5]
ns = tr[:, 0]
d = db.depths()
sizes = np.bincount(d, minlength=nk)
dt = np.diff(ns)
print(f"{wl}: ksets {nk} exec_ms {st['ms_exec']:.3f} rank_ms {st['ms_rank']:.3f} passes {st['rank_passes']}")
print("round start span ms", (ns[-1] - ns[0]) / 1e6)
order = np.argsort(-dt)[:15]
for k in order:
    c1 = f"cta1 start {(tr[k, 2] - ns[k]) / 1e3:8.2f} sig {(tr[k, 3] - ns[k]) / 1e3:8.2f}" if tr[k, 2] else ""
    half = (raw[k + 1, 6] - ns[k]) / 1e3 if k + 1 < nk and raw[k + 1, 6] else -1
    print(f"  round {k:5d} size {sizes[k]:8d} dt_us {dt[k] / 1e3:8.2f} cta0 sig {(tr[k, 1] - ns[k]) / 1e3:8.2f} {c1} spins {spins[k, 1]} {spins[k, 3]} cta0 saw-first-signal {half:8.2f}")
for lo, hi in [(0, 1), (1, 33), (33, 1025), (1025, 10**9)]:
    m = (sizes[:-1] >= lo) & (sizes[:-1] < hi)
    if m.any():
        print(f"  size [{lo},{hi}): rounds {m.sum():6d} total_us {dt[m].sum() / 1e3:9.1f} mean_us {dt[m].mean() / 1e3:7.2f}")

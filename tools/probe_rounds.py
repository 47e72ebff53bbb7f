"""Diagnostics: per-round K-SET executor timing and k-set size distribution."""
import sys
import time

import numpy as np
import torch

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
order = np.argsort(-dt)[:12]
for k in order:
    st = raw[k, 5] - ns[k]; wk = raw[k, 7] - ns[k]
    print(f"  round {k:5d} size {sizes[k]:8d} dt_us {dt[k] / 1e3:8.2f} cta0 work {(raw[k, 6] - ns[k]) / 1e3:7.2f} "
          f"last start {st / 1e3:7.2f} last work-done {wk / 1e3:7.2f} cta0 polls {raw[k + 1, 4] if k + 1 < nk else 0}")
    sl = int(raw[k, 3]); sidx = sl & 0xFFFFFF; sdur = (sl >> 24) / 1e3
    print(f"        slowest txn {sidx} type {bulk.type[sidx]} {sdur:.1f} us params {bulk.params(sidx)[:8]}")
w = np.where(raw[:, 6] > 0, raw[:, 6] - ns, 0)[:-1]
s1 = np.where(raw[:, 1] > 0, raw[:, 1] - ns, 0)[:-1]
print(f"  mean us: work-issued {w.mean() / 1e3:.2f} signalled {s1.mean() / 1e3:.2f} round {dt.mean() / 1e3:.2f}")
lstart = np.where(raw[:, 5] > 0, raw[:, 5] - ns, 0)[:-1]
lwork = np.where(raw[:, 7] > 0, raw[:, 7] - ns, 0)[:-1]
for lo, hi in [(0, 1), (1, 9), (9, 33), (33, 129), (129, 1025), (1025, 10**9)]:
    m = (sizes[:-1] >= lo) & (sizes[:-1] < hi)
    if m.any():
        print(f"  size [{lo},{hi}): rounds {m.sum():6d} total_us {dt[m].sum() / 1e3:9.1f} mean_us {dt[m].mean() / 1e3:7.2f}"
              f"  cta0 issued {w[m].mean() / 1e3:6.2f} signalled {s1[m].mean() / 1e3:6.2f} last start"
              f" {lstart[m].mean() / 1e3:6.2f} last issued {lwork[m].mean() / 1e3:6.2f}")
print("  k, size, dt_us (every few rounds):")
step = max(1, nk // 40)
print("  " + " ".join(f"{k}:{sizes[k]}:{dt[k] / 1e3:.2f}" for k in range(0, nk - 1, step)))

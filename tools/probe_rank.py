"""Diagnostics: per-pass phase times of the K-SET rank fixpoint (gputx_read_rank_ns)."""
import sys

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
P = min(int(st["rank_passes"]), 1024)
r = db.rank_ns(P).astype(np.int64)
t0 = r[0, 0]
print(f"{wl}: rank_ms {st['ms_rank']:.3f} passes {st['rank_passes']} sort_ms {st['ms_sort']:.3f} "
      f"exec_ms {st['ms_exec']:.3f} ksets {st['ksets']}")
print(" pass   A_us  bar1_us   D_us  bar2_us  total_us  swept  sweeps")
tot = np.zeros(4)
for p in range(P):
    a = (r[p, 1] - r[p, 0]) / 1e3
    b1 = (r[p, 2] - r[p, 1]) / 1e3
    d = (r[p, 3] - r[p, 2]) / 1e3
    b2 = (r[p, 4] - r[p, 3]) / 1e3
    tot += [a, b1, d, b2]
    if p < 12 or p >= P - 3 or p % max(1, P // 20) == 0:
        print(f"{p:5d} {a:7.1f} {b1:7.1f} {d:7.1f} {b2:7.1f} {(r[p, 4] - r[p, 0]) / 1e3:9.1f} {r[p, 5]:6d} {r[p, 6]:6d}")
print(f"sum us: A {tot[0]:.1f} bar1 {tot[1]:.1f} D {tot[2]:.1f} bar2 {tot[3]:.1f}; span {(r[P - 1, 4] - t0) / 1e3:.1f}")

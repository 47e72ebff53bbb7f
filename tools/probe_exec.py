"""Diagnostics: K-SET exec / total ms of one workload (env knobs apply: GPUTX_KSET_Q, ...)."""
import os
import sys

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "tpcb"
strategy = sys.argv[2] if len(sys.argv) > 2 else "kset"
if wl == "tpcb":
    schema, dims, n, kw = W.TPCB, W.TpcbDims(1000, 10, 100_000), 4_000_000, dict(remote_pct=15.0)
elif wl == "tm1":
    schema, dims, n, kw = W.TM1, W.Tm1Dims(1_000_000), 1_000_000, dict(dist="nurand")
else:
    schema, dims, n, kw = W.TPCC, W.TpccDims(64, 10, 3000, 100_000), 1_000_000, {}
image = W.make_db(schema, dims, seed=1)
bulk = W.make_bulk(schema, dims, n, seed=2, **kw)
db = Database(schema, dims.dims, n, image, insert_capacity=8)
best = None
for it in range(4):
    db.submit(bulk)
    st = db.execute(strategy)
    if best is None or st["ms_total"] < best["ms_total"]:
        best = st
    db.reset()
env = {k: v for k, v in os.environ.items() if k.startswith("GPUTX_")}
print(f"{wl} {strategy} {env}: total {best['ms_total']:.3f} rank {best['ms_rank']:.3f} exec {best['ms_exec']:.3f} ms")

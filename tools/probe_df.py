"""K-SET executor comparison: rounds (GPUTX_KSET_DF=0) vs dataflow (=1) on the bench configs."""
import os
import sys

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
import bench  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

MICRO = dict(schema=W.MICRO, dims=W.MicroDims(8_000_000, 8, 1), n=1 << 20, kw=dict(alpha=0.01))
for name in sys.argv[1:] or ["tpcb", "tpcc", "tpcb_add", "tpcc_add", "tpcb_hot_add"]:
    wl = MICRO if name == "micro" else bench.WORKLOADS[name]
    image = W.make_db(wl["schema"], wl["dims"], seed=1)
    bulk = W.make_bulk(wl["schema"], wl["dims"], wl["n"], 2, **wl["kw"])
    for df in ("0", "1"):
        os.environ["GPUTX_KSET_DF"] = df
        db = Database(wl["schema"], wl["dims"].dims, wl["n"], image, insert_capacity=6, add_rule=wl.get("add_rule", False))
        best = None
        for it in range(4):
            db.reset()
            db.submit(bulk)
            st = db.execute("kset")
            if best is None or st["ms_exec"] < best["ms_exec"]:
                best = st
        print(f"{name:14s} df={df}: exec {best['ms_exec']:8.3f} ms  total {best['ms_total']:8.3f} ms  depth {best['depth']}",
              flush=True)
        db.close()

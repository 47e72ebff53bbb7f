"""Diagnostics: median per-phase device times of one bench workload (device-resident
bulks, K-SET unless argv[2] names another strategy)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tm1"
strategy = sys.argv[2] if len(sys.argv) > 2 else "kset"
wl = bench.WORKLOADS[name]
dims, image, bulks = bench.make_inputs(wl, 0, 1, 3, 1)
db = Database(wl["schema"], dims.dims, wl["n"], image, insert_capacity=40, packed_out=True)
if len(sys.argv) > 3:                                  # executor grid cap (CTAs)
    db.set_launch(exec_grid=int(sys.argv[3]))
dev = torch.device("cuda:0")
dbk = [(torch.from_numpy(b.type).to(dev), torch.from_numpy(b.param_off.view(np.int32)).to(dev),
        torch.from_numpy(b.param_words.view(np.int32)).to(dev)) for b in bulks]
keys = ["ms_ingest", "ms_emit", "ms_sort", "ms_rank", "ms_group", "ms_exec", "ms_total"]
rows = []
for it in range(10):
    t, o, w = dbk[it % 3]
    db.submit(type=t, param_off=o, param_words=w, on_device=True)
    st = db.execute(strategy)
    rows.append([st[k] for k in keys])
    if it % 3 == 2:
        db.reset()
m = np.median(np.array(rows[3:]), axis=0)
print(name, strategy, " ".join(f"{k[3:]} {v:.3f}" for k, v in zip(keys, m)))

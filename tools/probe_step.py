"""Diagnostics: host vs device time of one device-resident submit + execute step (TM-1)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

dims = W.Tm1Dims(1_000_000)
image = W.make_db(W.TM1, dims, seed=1)
bulk = W.make_bulk(W.TM1, dims, 1_000_000, seed=2, dist="nurand")
dev = torch.device("cuda:0")
tt = torch.from_numpy(bulk.type).to(dev)
po = torch.from_numpy(bulk.param_off.view(np.int32)).to(dev)
pw = torch.from_numpy(bulk.param_words.view(np.int32)).to(dev)
strategy = sys.argv[1] if len(sys.argv) > 1 else "kset"
db = Database(W.TM1, dims.dims, 1_000_000, image, insert_capacity=8, packed_out=True)
stream = torch.cuda.current_stream()
rows = []
for it in range(12):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e0.record(stream)
    db.submit(type=tt, param_off=po, param_words=pw, on_device=True)
    h1 = time.perf_counter()
    e1.record(stream)
    st = db.execute(strategy)
    h2 = time.perf_counter()
    e2.record(stream)
    e2.synchronize()
    rows.append((e0.elapsed_time(e1), e1.elapsed_time(e2), (h1 - h0) * 1e3, (h2 - h1) * 1e3, st["ms_ingest"], st["ms_total"]))
r = np.array(rows[4:])
m = np.median(r, axis=0)
print(f"{strategy}: dev submit {m[0]:.3f} execute {m[1]:.3f} | host submit {m[2]:.3f} execute {m[3]:.3f} | "
      f"ingest {m[4]:.3f} ms_total {m[5]:.3f}  step {m[0] + m[1]:.3f} ms")

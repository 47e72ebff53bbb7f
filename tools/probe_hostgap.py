"""Diagnostics: is the device-resident TM-1 step host-bound?  Times one step (submit +
execute_async) (a) as bench.py does, from an idle stream, and (b) with a 3 ms device sleep
queued before the start event so every launch is enqueued before the GPU reaches it
(GPU-only time); (c) the host's enqueue time of the step."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tm1"
wl = bench.WORKLOADS[name]
dims, image, bulks = bench.make_inputs(wl, 0, 1, 3, 1)
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
db = Database(wl["schema"], dims.dims, wl["n"], image, insert_capacity=40, packed_out=True, deferred_check=True,
              stream=stream.cuda_stream)
dbk = [(torch.from_numpy(b.type).to(dev), torch.from_numpy(b.param_off.view(np.int32)).to(dev),
        torch.from_numpy(b.param_words.view(np.int32)).to(dev)) for b in bulks]
res = {"idle": [], "queued": [], "host_ms": []}
for it in range(24):
    t, o, w = dbk[it % 3]
    if it % 3 == 0:
        db.reset()
    mode = "queued" if it % 2 else "idle"
    torch.cuda.synchronize()
    if mode == "queued":
        torch.cuda._sleep(3_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    db.submit(type=t, param_off=o, param_words=w, on_device=True)
    db.execute_async("kset")
    h1 = time.perf_counter()
    e1.record(stream)
    db.wait()
    e1.synchronize()
    if it >= 6:
        res[mode].append(e0.elapsed_time(e1))
        res["host_ms"].append((h1 - h0) * 1e3)
print(name, " ".join(f"{k} {statistics.median(v):.3f}" for k, v in res.items()))

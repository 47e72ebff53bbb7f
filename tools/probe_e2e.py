"""Diagnostics: where the e2e pipeline (gputx_run_bulks) spends its time on TM-1."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "tm1"]
dims, image, bulks = bench.make_inputs(wl, 0, 1, 3, 1)
db = Database(wl["schema"], dims.dims, wl["n"], image, insert_capacity=60, packed_out=True)


def pin(a):
    return torch.from_numpy(a.view(np.uint8)).pin_memory().numpy().view(a.dtype)


class HB:
    def __init__(self, b):
        self.type, self.param_off, self.param_words = pin(b.type), pin(b.param_off), pin(b.param_words)


hb = [HB(b) for b in bulks]
n = wl["n"]
st2 = [pin(np.zeros(n, np.uint8)) for _ in range(2)]
out2 = [pin(np.zeros((n, db.stride), np.uint8)) for _ in range(2)]
K = 10
seq = [hb[k % 3] for k in range(K)]
for label, st, out in [("status+out", st2, out2), ("status", st2, None), ("none", None, None)]:
    db.run_bulks(seq[:2], "kset", [st2[k % 2] for k in range(2)] if st else None, [out2[k % 2] for k in range(2)] if out else None)
    t0 = time.perf_counter()
    db.run_bulks(seq, "kset", [st2[k % 2] for k in range(K)] if st else None, [out2[k % 2] for k in range(K)] if out else None)
    print(f"run_bulks {label}: {1e3 * (time.perf_counter() - t0) / K:.3f} ms/bulk", flush=True)
t0 = time.perf_counter()
for k in range(K):
    db.submit(seq[k])
    db.execute_nostats("kset")
print(f"host submit+execute (sync H2D inside submit): {1e3 * (time.perf_counter() - t0) / K:.3f} ms/bulk")
dev = [bench_t for bench_t in []]
t = [torch.from_numpy(b.type).cuda() for b in bulks]
o = [torch.from_numpy(b.param_off.view(np.int32)).cuda() for b in bulks]
w = [torch.from_numpy(b.param_words.view(np.int32)).cuda() for b in bulks]
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(K):
    db.submit(type=t[k % 3], param_off=o[k % 3], param_words=w[k % 3], on_device=True)
    db.execute_nostats("kset")
print(f"device-resident submit+execute: {1e3 * (time.perf_counter() - t0) / K:.3f} ms/bulk")
hbuf = out2[0]
dbuf = torch.empty(hbuf.nbytes, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(K):
    torch.from_numpy(hbuf.view(np.uint8).reshape(-1)).copy_(dbuf, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H {hbuf.nbytes / 1e6:.0f} MB alone: {1e3 * (time.perf_counter() - t0) / K:.3f} ms")

"""Diagnostics: per-phase device times of gputx_run_bulks bulks with / without the result D2H."""
import sys

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
K = 8
seq = [hb[k % 3] for k in range(K)]
keys = ["ms_ingest", "ms_emit", "ms_sort", "ms_rank", "ms_group", "ms_exec"]
for label, st, out in [("status+out", st2, out2), ("none", None, None), ("status+out", st2, out2)]:
    sts = db.run_bulks(seq, "kset", [st2[k % 2] for k in range(K)] if st else None,
                       [out2[k % 2] for k in range(K)] if out else None, stats=True)
    for s in sts[2:5]:
        print(label, {k: round(s[k], 3) for k in keys}, flush=True)

"""Diagnostics: timeline of a pipelined gputx_run_bulks run (GPUTX_PIPE_TRACE): per bulk the
exec start / exec end / D2H end times, with and without the result copies."""
import os
import sys

import numpy as np
import torch

os.environ["GPUTX_PIPE_TRACE"] = "1"
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

wl = bench.WORKLOADS["tm1"]
dims, image, bulks = bench.make_inputs(wl, 0, 1, 3, 1)
dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
db = Database(wl["schema"], dims.dims, wl["n"], image, packed_out=True, deferred_check=True, stream=stream.cuda_stream)


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
for label, withres in [("warm", True), ("results", True), ("no results", False)]:
    print(label, flush=True)
    sys.stderr.flush()
    db.run_bulks(seq, "kset", [st2[k % 2] for k in range(K)] if withres else None,
                 [out2[k % 2] for k in range(K)] if withres else None)
    torch.cuda.synchronize()

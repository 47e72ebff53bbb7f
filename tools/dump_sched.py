"""Write the real TM-1 k-set schedule (off[k*T+t], g[k]) for tools/execrepro."""
import sys
import numpy as np
sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

dims = W.Tm1Dims(1_000_000)
image = W.tm1_db(dims, seed=1)
bulk = W.tm1_bulk(dims, 1_000_000, seed=2, dist="nurand")
db = Database(W.TM1, dims.dims, bulk.n, image)
db.submit(bulk)
db.execute("kset")
d = db.depths().astype(np.int64)
T = 7
key = d * T + bulk.type.astype(np.int64)
nk = int(d.max()) + 1
cnt = np.bincount(key, minlength=nk * T)
off = np.zeros(nk * T + 1, np.uint32)
off[1:] = np.cumsum(cnt)
sizes = np.bincount(d, minlength=nk)
G, Q = int(sys.argv[1]) if len(sys.argv) > 1 else 2, 256
g = np.clip((sizes + Q - 1) // Q, 1, G).astype(np.uint16)
with open("gpurun_out/sched.bin", "wb") as f:
    np.array([nk], np.uint32).tofile(f)
    off.tofile(f)
    g.tofile(f)
print("nk", nk, "g>1 rounds", int((g > 1).sum()))

"""Sharded bench path in one process (G handles on one GPU, LocalShards exchange):
   python tools/repro_shard.py <workload> [G] [steps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402
from paper_1103_3105_b200.shard import LocalShards  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1]]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
strats = (sys.argv[4] if len(sys.argv) > 4 else "kset").split(",")
n = wl["n"]
ins = [bench.make_inputs(wl, r, G, steps, 1) for r in range(G)]
dims, image = ins[0][0], ins[0][1]
dbs = [Database(wl["schema"], dims.dims, min(1 << 24, n + n // 2 + 1024), image, shard=r, nshards=G,
                insert_capacity=3 * steps + 8, add_rule=wl.get("add_rule", False)) for r in range(G)]
ls = LocalShards(dbs)
for k in range(steps * len(strats)):
    strategy = strats[k // steps]
    homes = [ins[r][2][k % len(ins[r][2])] for r in range(G)]
    for r, h in enumerate(homes):
        t = h.ts.astype(np.int64)
        print(f"step {k} rank {r}: n {h.n} ts [{t.min()}, {t.max()}] strictly increasing {bool((np.diff(t) > 0).all())}")
    try:
        st = ls.step(homes, strategy)
        print("  ok", strategy, [(s["n"], s["depth"], s["rank_passes"]) for s in st])
    except Exception as e:
        print("  FAILED", e)
        break

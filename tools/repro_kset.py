"""Reproduce / bisect a K-SET parity failure on the smoke() TM-1 config.
usage: python tools/repro_kset.py [reps] [schema]   (env knobs GPUTX_KSET_* apply)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
which = sys.argv[2] if len(sys.argv) > 2 else "tm1"
strategy = sys.argv[3] if len(sys.argv) > 3 else "kset"
cfg = {"tm1": (W.TM1, W.Tm1Dims(4096), 8192), "tpcb": (W.TPCB, W.TpcbDims(4, 10, 1000), 4096),
       "tpcc": (W.TPCC, W.TpccDims(2, 10, 3000, 10_000), 2048)}[which]
schema, dims, n = cfg
image = W.make_db(schema, dims, seed=1)
bulk = W.make_bulk(schema, dims, n, seed=2)
ref = oracle.run(schema, dims.dims, image, bulk)
bad = 0
for r in range(reps):
    with Database(schema, dims.dims, n, image, device=0) as db:
        db.submit(bulk)
        stats = db.execute(strategy)
        st, out = db.read_results()
        got = db.read_image(image)
        msgs = []
        if not np.array_equal(st, ref.status):
            msgs.append(f"status {np.flatnonzero(st != ref.status)[:10]}")
        o = out.reshape(n, -1)
        ro = ref.out.reshape(n, -1)
        rows = np.flatnonzero((o != ro).any(axis=1))
        if len(rows):
            types = bulk.type[rows]
            msgs.append(f"out rows {len(rows)} first {rows[:10]} types {np.bincount(types, minlength=7)}")
            if r == 0 and which == "tm1":
                d = db.depths()
                nbr = {int(v): k for k, v in enumerate(image["sub_nbr"])}
                for i in rows[:6]:
                    if bulk.type[i] != 0:
                        continue
                    s_ = int(bulk.params(i)[0]) - 1
                    gv = int(o[i][20:24].copy().view(np.uint32)[0])
                    wv = int(ro[i][20:24].copy().view(np.uint32)[0])
                    uls = [(j, int(d[j]), int(bulk.params(j)[2])) for j in range(n) if bulk.type[j] == 4
                           and nbr.get(int(bulk.params(j)[0]) | (int(bulk.params(j)[1]) << 32)) == s_]
                    msgs.append(f"  GSD {i} depth {d[i]} s {s_} got vlr {gv} want {wv} init {int(image['sub_vlr'][s_])} ULs {uls}")
            if r == 0:
                d = db.depths()
                for i in rows[:5]:
                    msgs.append(f"  txn {i} type {bulk.type[i]} depth {d[i]} got {o[i][:24]} want {ro[i][:24]}")
        if strategy == "kset":
            want_d = oracle.depths(schema, dims.dims, image, bulk)
            gd = db.depths()
            if not np.array_equal(gd, want_d):
                bad_d = np.flatnonzero(gd != want_d)
                msgs.append(f"depths differ at {len(bad_d)}: {bad_d[:8]} got {gd[bad_d[:8]]} want {want_d[bad_d[:8]]}")
        for k in image:
            if not np.array_equal(got[k], ref.db[k]):
                msgs.append(f"col {k} diff {int((got[k] != ref.db[k]).sum())}")
        if msgs:
            bad += 1
            print(f"rep {r}: MISMATCH depth={stats['depth']}", *msgs, sep="\n  ")
print(f"{which} {strategy}: {bad}/{reps} bad", flush=True)
sys.exit(1 if bad else 0)

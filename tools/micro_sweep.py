"""Micro-benchmark sweeps (App. F.1): the trends of
Figures 3, 4, 5, 6, 12, 13 and 14 on B200, plus the grouping calibration of App. D
(PAPER.md:400-404).  Every point is one bulk of the micro schema (N tuples, T types, x units
of 100 sin calls, lock skew alpha) executed through the C ABI; device times from the
library's CUDA events (gputx_stats).  Bulk 0 of every configuration is first checked against
the oracle (bit-exact) -- a sweep that fails parity aborts.

usage: python tools/micro_sweep.py [fig3,fig4,fig5,fig6,fig12,fig13,fig14,calib] [--out profiles/x.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

STRATS = ("tpl", "part", "kset")


def check_parity(d, image, bulk, strategy, db, p=0):
    import oracle
    ref = oracle.run(W.MICRO, d.dims, image, bulk)
    db.reset()
    db.set_grouping(p)
    db.submit(bulk)
    db.execute(strategy)
    st, out = db.read_results()
    got = db.read_column("tuple").view(np.uint32)
    ok = np.array_equal(st, ref.status) and np.array_equal(out, ref.out) and np.array_equal(got, ref.db["tuple"])
    if not ok:
        raise SystemExit(f"PARITY FAILURE micro {d} {strategy} p={p}")
    db.reset()


def measure(db, bulk, strategy, reps=3, p=0, part_size=None):
    """median over reps of (stats of one bulk); the DB is reset before each run."""
    db.set_grouping(p)
    res = []
    for _ in range(reps):
        db.reset()
        db.submit(bulk)
        res.append(db.execute(strategy))
    res.sort(key=lambda s: s["ms_total"])
    s = res[len(res) // 2]
    s["txn_per_s"] = bulk.n / (s["ms_total"] / 1e3)
    return s


def pick(s, keys=("ms_total", "ms_sort", "ms_rank", "ms_group", "ms_exec", "depth", "zero_set", "max_chain",
                  "txn_per_s")):
    return {k: s[k] for k in keys}


def fig3(args):
    """Branch divergence: throughput with and without grouping on the transaction types,
    T = 1..32, x = 1 (L) and 16 (H); grouping = the calibrated p (best of 2^k <= T)."""
    rows = []
    n = args.n
    for x in (1, 16):
        for T in (1, 2, 4, 8, 16, 32):
            d = W.MicroDims(8_000_000, T, x)
            image = W.micro_db(d, seed=1)
            bulk = W.micro_bulk(d, n, seed=2)
            db = Database(W.MICRO, d.dims, n, image)
            check_parity(d, image, bulk, "kset", db, p=1)
            base = measure(db, bulk, "kset", p=1)
            best, bp = None, None
            for p in [q for q in (1, 2, 4, 8, 16, 32) if q <= T]:
                s = measure(db, bulk, "kset", p=p)
                if best is None or s["ms_group"] + s["ms_exec"] < best["ms_group"] + best["ms_exec"]:
                    best, bp = s, p
            db.close()
            rows.append({"x": x, "T": T, "no_grouping_txn_per_s": n / ((base["ms_group"] + base["ms_exec"]) / 1e3),
                         "grouping_txn_per_s": n / ((best["ms_group"] + best["ms_exec"]) / 1e3),
                         "calibrated_p": bp, "no_grouping": pick(base), "grouping": pick(best)})
            print(json.dumps(rows[-1]), flush=True)
    return rows


def calib(args):
    """App. D / Fig. 12: x = 32, T = 16, type groups p = 1..16: grouping vs execution time;
    the calibrated p minimises their sum."""
    d = W.MicroDims(8_000_000, 16, 32)
    n = args.n
    image = W.micro_db(d, seed=1)
    bulk = W.micro_bulk(d, n, seed=2)
    db = Database(W.MICRO, d.dims, n, image)
    check_parity(d, image, bulk, "kset", db, p=4)
    rows = []
    for p in (1, 2, 4, 8, 16):
        s = measure(db, bulk, "kset", p=p)
        rows.append({"p": p, "ms_group": s["ms_group"], "ms_exec": s["ms_exec"],
                     "ms_group_plus_exec": s["ms_group"] + s["ms_exec"]})
        print(json.dumps(rows[-1]), flush=True)
    db.close()
    best = min(rows, key=lambda r: r["ms_group_plus_exec"])
    return {"rows": rows, "calibrated_p": best["p"]}


def fig4(args):
    """Throughput of the three strategies vs bulk size (8M tuples, x = 16, T = 8, uniform)."""
    d = W.MicroDims(8_000_000, 8, 16)
    image = W.micro_db(d, seed=1)
    rows = []
    nmax = 1 << 22
    db = Database(W.MICRO, d.dims, nmax, image)
    for lg in range(10, 23, 2):
        n = 1 << lg
        bulk = W.micro_bulk(d, n, seed=lg)
        if lg == 10:
            for s_ in STRATS:
                check_parity(d, image, bulk, s_, db)
        row = {"n": n}
        for s_ in STRATS:
            row[s_] = pick(measure(db, bulk, s_))
        rows.append(row)
        print(json.dumps({"n": n, **{s_: "%.3g" % row[s_]["txn_per_s"] for s_ in STRATS}}), flush=True)
    db.close()
    return rows


def fig5(args):
    """Time breakdown (bulk generation = emit + sort + rank + group vs execution) at ~16M
    transactions."""
    n = 1 << 24
    d = W.MicroDims(8_000_000, 8, 16)
    image = W.micro_db(d, seed=1)
    bulk = W.micro_bulk(d, n, seed=3)
    db = Database(W.MICRO, d.dims, n, image)
    out = {}
    for s_ in STRATS:
        s = measure(db, bulk, s_, reps=2)
        gen = s["ms_emit"] + s["ms_sort"] + s["ms_rank"] + s["ms_group"]
        out[s_] = {"ms_generation": gen, "ms_exec": s["ms_exec"], "generation_share": gen / (gen + s["ms_exec"]),
                   "txn_per_s": s["txn_per_s"]}
        print(s_, json.dumps(out[s_]), flush=True)
    db.close()
    return out


def fig6(args):
    """Throughput vs lock skew alpha (tuple 0 with probability alpha),
    x = 1 so the deep chains stay measurable (bulk 64k)."""
    d = W.MicroDims(8_000_000, 8, 1)
    image = W.micro_db(d, seed=1)
    n = 1 << 16
    db = Database(W.MICRO, d.dims, n, image)
    rows = []
    for a in (0.0, 0.001, 0.01, 0.05, 0.1, 0.2, 0.4):
        bulk = W.micro_bulk(d, n, seed=5, alpha=a)
        if a == 0.01:
            for s_ in STRATS:
                check_parity(d, image, bulk, s_, db)
        row = {"alpha": a}
        for s_ in STRATS:
            row[s_] = pick(measure(db, bulk, s_))
        rows.append(row)
        print(json.dumps({"alpha": a, "depth": row["kset"]["depth"],
                          **{s_: "%.3g" % row[s_]["txn_per_s"] for s_ in STRATS}}), flush=True)
    db.close()
    return rows


def fig13(args):
    """PART throughput vs partition size (x = 16, optimum 128 there)."""
    d = W.MicroDims(8_000_000, 8, 16)
    image = W.micro_db(d, seed=1)
    n = 1 << 20
    bulk = W.micro_bulk(d, n, seed=7)
    rows = []
    for ps in (16, 32, 64, 128, 256, 512, 1024, 4096):
        db = Database(W.MICRO, d.dims, n, image, part_size=ps)
        if ps == 128:
            check_parity(d, image, bulk, "part", db)
        s = measure(db, bulk, "part")
        rows.append({"part_size": ps, **pick(s)})
        print(json.dumps({"part_size": ps, "txn_per_s": "%.3g" % s["txn_per_s"], "max_chain": s["max_chain"]}),
              flush=True)
        db.close()
    return rows


def fig14(args):
    """Throughput vs relation cardinality (bulk 256k, x = 16)."""
    n = 1 << 18
    rows = []
    for lg in (10, 12, 14, 16, 18, 20, 23):
        d = W.MicroDims(1 << lg, 8, 16)
        image = W.micro_db(d, seed=1)
        bulk = W.micro_bulk(d, n, seed=lg)
        db = Database(W.MICRO, d.dims, n, image)
        if lg == 14:
            for s_ in STRATS:
                check_parity(d, image, bulk, s_, db)
        row = {"tuples": 1 << lg}
        for s_ in STRATS:
            row[s_] = pick(measure(db, bulk, s_, reps=2))
        rows.append(row)
        print(json.dumps({"tuples": 1 << lg, "depth": row["kset"]["depth"],
                          **{s_: "%.3g" % row[s_]["txn_per_s"] for s_ in STRATS}}), flush=True)
        db.close()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("figs", nargs="?", default="fig3,calib,fig4,fig5,fig6,fig13,fig14")
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = {"device": None, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    try:
        import torch
        res["device"] = torch.cuda.get_device_name(0)
    except Exception:
        pass
    fns = {"fig3": fig3, "calib": calib, "fig4": fig4, "fig5": fig5, "fig6": fig6, "fig13": fig13, "fig14": fig14}
    for f in args.figs.split(","):
        t0 = time.time()
        print(f"== {f}", flush=True)
        res[f] = fns[f](args)
        res[f + "_wall_s"] = time.time() - t0
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

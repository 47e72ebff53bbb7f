"""Streaming K-SET measurements:

  resp  : response time vs throughput (PAPER.md:286 Fig. 9 on TM-1, :497 Fig. 15):
          transactions arrive uniformly at rate LAMBDA; every interval t the system takes the
          pool's arrivals and either (stream) runs ONE streaming K-SET step -- the pool's 0-set
          (gputx_pool_step) -- or (bulk) executes all of them as one K-SET bulk.  Virtual
          clock: a tick starts at max(k*t, end of the previous tick) and lasts the measured
          wall time of its library calls; response = completion - arrival.
  skew  : throughput vs lock skew alpha (Fig. 6, micro benchmark x = 1): chunks
          of arrivals, one streaming step per chunk (executed transactions per second, with
          the backlog left in the pool) against executing every chunk as a bulk.

usage: python tools/pool_bench.py [resp,skew] [--out profiles/x.json]
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


def resp(args):
    dims = W.Tm1Dims(1_000_000)
    image = W.tm1_db(dims, seed=1)
    lam = args.rate
    rows = []
    for t_ms in (0.02, 0.05, 0.1, 0.2, 0.5, 1.0, 2.0):
        per = max(1, int(lam * t_ms / 1e3))
        ticks = max(8, min(200, int(200e3 / per)))
        total = per * ticks
        arr = W.tm1_bulk(dims, total, seed=11, dist="nurand")
        arrival = (np.arange(total) + 0.5) / lam                       # seconds, uniform
        for mode in ("stream", "stream_drain", "bulk"):
            db = Database(W.TM1, dims.dims, 1 << 23, image, insert_capacity=1)
            done_t = np.full(total, np.nan)
            clock = 0.0
            warm = arr.slice(0, min(per, 1000))
            db.submit(warm)
            db.execute("kset")
            db.reset()
            db.pool_submit(warm)                      # first pool use allocates its buffers
            db.pool_step()
            db.reset()
            for k in range(ticks + 200):
                start = max((k + 1) * t_ms / 1e3, clock)
                lo, hi = k * per, min((k + 1) * per, total)
                t0 = time.perf_counter()
                if mode.startswith("stream"):
                    # stream: ONE 0-set per tick; stream_drain: 0-sets while they are at
                    # least 1% of a tick's arrivals (the deep tail waits for later ticks)
                    if lo < hi:
                        db.pool_submit(arr.slice(lo, hi))
                    parts = []
                    while True:
                        ex = db.pool_step()["executed"]
                        t_, _, _ = db.pool_read()
                        parts.append(t_.astype(np.int64))
                        if mode == "stream" or ex * 100 < per or not db.pool_pending():
                            break
                    ts = np.concatenate(parts)
                elif lo < hi:
                    first = db.submit(arr.slice(lo, hi))
                    db.execute_nostats("kset")
                    st, _ = db.read_results()
                    ts = first + np.arange(hi - lo)
                else:
                    ts = np.zeros(0, np.int64)
                clock = start + (time.perf_counter() - t0)
                done_t[ts] = clock
                if hi >= total and (mode == "bulk" or db.pool_pending() == 0):
                    break
            ok = ~np.isnan(done_t)
            r = done_t[ok] - arrival[ok]
            rows.append({"interval_ms": t_ms, "mode": mode, "per_tick": per, "completed": int(ok.sum()),
                         "throughput_txn_per_s": float(ok.sum() / clock), "mean_response_ms": float(r.mean() * 1e3),
                         "p99_response_ms": float(np.percentile(r, 99) * 1e3)})
            print(json.dumps(rows[-1]), flush=True)
            db.close()
    return rows


def skew(args):
    d = W.MicroDims(8_000_000, 8, 1)
    image = W.micro_db(d, seed=1)
    chunk, steps = 1 << 16, 24
    rows = []
    for a in (0.0, 0.01, 0.05, 0.1, 0.2, 0.4):
        arr = W.micro_bulk(d, chunk * steps, seed=5, alpha=a)
        res = {"alpha": a}
        for mode in ("stream", "bulk"):
            db = Database(W.MICRO, d.dims, 1 << 23, image)
            warm = arr.slice(0, 1000)
            db.pool_submit(warm)                      # first pool use allocates its buffers
            db.pool_step()
            db.reset()
            db.submit(warm)
            db.execute("kset")
            db.reset()
            executed, secs = 0, 0.0
            for k in range(steps):
                sl = arr.slice(k * chunk, (k + 1) * chunk)
                t0 = time.perf_counter()
                if mode == "stream":
                    db.pool_submit(sl)
                    executed += db.pool_step()["executed"]
                else:
                    db.submit(sl)
                    executed += db.execute("kset")["n"]
                secs += time.perf_counter() - t0
            res[mode] = {"txn_per_s": executed / secs, "executed": executed,
                         "backlog": db.pool_pending() if mode == "stream" else 0}
            db.close()
        rows.append(res)
        print(json.dumps(rows[-1]), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="?", default="resp,skew")
    ap.add_argument("--rate", type=float, default=2e8, help="arrival rate (txn/s) of the response-time runs")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = {}
    for w in args.what.split(","):
        print(f"== {w}", flush=True)
        res[w] = {"resp": resp, "skew": skew}[w](args)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

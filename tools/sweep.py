"""BASELINE config 5: bulk-size and contention sweep across TPL / PART / K-SET.

TPC-B, 1,000 branches (the single-type workload is the clean
contention axis), bulk n in {2^10 .. 2^22} (2^24 with --max-log2 24), branch skew
Zipf(theta), theta in {0, 0.3, 0.6, 0.9, 1.2}.  Device-resident bulks, one warm-up and
--steps timed bulks per point (CUDA events around submit + execute), median reported.
A point whose first timed bulk exceeds --cap seconds is reported as "timeout" and the
larger bulks of that (theta, strategy) are skipped.  One GPU (G = 1): the multi-GPU
columns of config 5 need the 8-GPU step (bench.py --gpus N covers the sharded path).

    python tools/sweep.py [--max-log2 22] [--steps 3] [--out profiles/round1_sweep.json]
"""
import argparse
import json
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=22)
    ap.add_argument("--thetas", default="0,0.3,0.6,0.9,1.2")
    ap.add_argument("--strategies", default="kset,part,tpl")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--cap", type=float, default=60.0)
    ap.add_argument("--branches", type=int, default=1000)
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    args = ap.parse_args()
    dims = W.TpcbDims(args.branches, 10, 100_000)
    image = W.tpcb_db(dims)
    nmax = 1 << args.max_log2
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)          # one stream for the engine and the events
    torch.cuda.set_stream(stream)
    db = Database(W.TPCB, dims.dims, nmax, image, stream=stream.cuda_stream,
                  insert_capacity=2)
    thetas = [float(x) for x in args.thetas.split(",")]
    strategies = args.strategies.split(",")
    rows = []
    dead = set()
    for lg in range(args.min_log2, args.max_log2 + 1):
        n = 1 << lg
        for th in thetas:
            t0 = time.time()
            bulk = W.tpcb_bulk(dims, n, seed=lg * 101 + int(th * 10), zipf_theta=th)
            gen_s = time.time() - t0
            t = torch.from_numpy(bulk.type).to(dev)
            o = torch.from_numpy(bulk.param_off.view(np.int32)).to(dev)
            w = torch.from_numpy(bulk.param_words.view(np.int32)).to(dev)
            top = float(np.bincount(bulk.param_words[2::4], minlength=dims.branches).max()) / n
            for s in strategies:
                row = {"n": n, "theta": th, "strategy": s, "top_branch_share": top}
                if (th, s) in dead:
                    row["result"] = "timeout (smaller bulk exceeded the cap)"
                    rows.append(row)
                    continue
                ms, st = [], None
                for k in range(args.steps + 1):
                    db.reset()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    w0 = time.time()
                    e0.record(stream)
                    db.submit(type=t, param_off=o, param_words=w, on_device=True)
                    st = db.execute(s)
                    e1.record(stream)
                    e1.synchronize()
                    if k > 0:
                        ms.append(e0.elapsed_time(e1))
                    if time.time() - w0 > args.cap:
                        dead.add((th, s))
                        break
                if (th, s) in dead and len(ms) < args.steps:
                    row["result"] = f"timeout (> {args.cap:.0f} s per bulk)"
                else:
                    med = statistics.median(ms)
                    row.update(result="ok", ms=med, txn_per_s=n / (med / 1e3), depth=st["depth"],
                               max_chain=st["max_chain"], rank_passes=st["rank_passes"], ms_exec=st["ms_exec"],
                               chose=st["strategy"])
                rows.append(row)
                print(json.dumps(row), flush=True)
            del t, o, w
            print(f"# n={n} theta={th} generated in {gen_s:.1f} s", file=sys.stderr, flush=True)
    json.dump({"config": "TPC-B 1,000 branches, Zipf(theta) over branches, 15% remote accounts, 1 GPU",
               "steps": args.steps, "rows": rows}, open(args.out, "w"), indent=1)
    db.close()


if __name__ == "__main__":
    main()

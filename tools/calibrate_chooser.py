"""Calibrate Algorithm 1's thresholds (w0_bar, d_bar, c_bar; "the
threshold ... calibration") on this GPU: measure K-SET / PART / TPL on a set of workloads,
record each bulk's structural parameters (w0, d, c from a GPUTX_AUTO run), and grid-search
the thresholds that maximise the mean of (chosen strategy's throughput / best strategy's).

    python tools/calibrate_chooser.py [--out gpurun_out/calibration.json]
"""
import argparse
import itertools
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_1103_3105_b200 import Database  # noqa: E402

INF = 1 << 62


def cases():
    for name, wl in bench.WORKLOADS.items():
        if name in ("tpcb_tiny", "tpcb_hot"):        # (hot without ADD: ~1 s per K-SET bulk)
            continue
        yield name, wl["schema"], wl["dims"], wl["n"], wl["kw"], wl.get("add_rule", False)
    d = W.TpcbDims(1000, 10, 100_000)
    for lg in (12, 16, 20):
        for th in (0.0, 0.9):
            yield f"tpcb_n2^{lg}_zipf{th}", W.TPCB, d, 1 << lg, dict(remote_pct=15.0, zipf_theta=th), False
    # the micro benchmark: lock skew alpha, cheap procedures (x = 1)
    m = W.MicroDims(1 << 20, 8, 1)
    for a in (0.0, 0.01, 0.1):
        yield f"micro_alpha{a}", W.MICRO, m, 1 << 16, dict(alpha=a), False


def choose(w0, d, c, w0b, db, cb):
    if w0 >= w0b:
        return "kset"
    return "part" if (c <= cb or d >= db) else "tpl"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/calibration.json")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    rows = []
    for name, schema, dims, n, kw, add in cases():
        image = W.make_db(schema, dims, seed=1)
        bulk = W.make_bulk(schema, dims, n, 2, **kw)
        db = Database(schema, dims.dims, n, image, stream=stream.cuda_stream, insert_capacity=4 * args.steps + 8,
                      add_rule=add)
        t = torch.from_numpy(bulk.type).to(dev)
        o = torch.from_numpy(bulk.param_off.view(np.int32)).to(dev)
        w = torch.from_numpy(bulk.param_words.view(np.int32)).to(dev)
        row = {"case": name, "n": n}
        for s in ("auto", "kset", "part", "tpl"):
            ms = []
            for k in range(args.steps + 1):
                db.reset()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                db.submit(type=t, param_off=o, param_words=w, on_device=True)
                st = db.execute(s)
                e1.record(stream)
                e1.synchronize()
                if k:
                    ms.append(e0.elapsed_time(e1))
            if s == "auto":
                row.update(w0=st["zero_set"], d=st["depth"], c=st["cross"])
            else:
                row[s] = n / (statistics.median(ms) / 1e3)
        db.close()
        row["best"] = max(("kset", "part", "tpl"), key=lambda s: row[s])
        print(json.dumps(row), flush=True)
        rows.append(row)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    grid_w0 = sorted({0, 1_000, 64 * nsm, 10_000, 128 * nsm, 100_000, 500_000, 1_000_000, 4_000_000, INF})
    grid_d = [0, 64, 256, 1_024, 2_048, 8_192, 65_536, 1 << 20, INF]
    grid_c = [0, 100, 10_000, 100_000, 1_000_000, INF]

    def score(b, rs=None):
        rs = rows if rs is None else rs
        return statistics.mean(r[choose(r["w0"], r["d"], r["c"], *b)] / r[r["best"]] for r in rs)

    grid = list(itertools.product(grid_w0, grid_d, grid_c))
    best = max(grid, key=score)
    # held-out efficiency: leave each bulk out, fit on the others, score it alone
    loo = []
    for k, r in enumerate(rows):
        rest = rows[:k] + rows[k + 1:]
        fit = max(grid, key=lambda b: score(b, rest))
        loo.append(score(fit, [r]))
    default = (64 * nsm, 0, 0)                    # the library's defaults (engine.cu choose_strategy)
    paper = (128 * nsm, 2_048, 0)                 # an uncalibrated reading
    res = {"rows": rows, "library_default": {"w0_bar": default[0], "d_bar": default[1], "c_bar": default[2],
                                             "mean_efficiency": score(default)},
           "uncalibrated": {"w0_bar": paper[0], "d_bar": paper[1], "c_bar": paper[2], "mean_efficiency": score(paper)},
           "calibrated": {"w0_bar": best[0], "d_bar": best[1], "c_bar": best[2], "mean_efficiency": score(best)},
           "leave_one_out_mean_efficiency": statistics.mean(loo),
           "oracle_best_mean_efficiency": 1.0}
    print(json.dumps({k: v for k, v in res.items() if k != "rows"}), flush=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

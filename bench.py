#!/usr/bin/env python3
"""GPUTx B200 benchmark: bulk transactions/s (BASELINE.json metric).

Default workload (N=1): BASELINE config 2 — TM-1 (TATP), 1M subscribers, bulks of
1M transactions (TATP standard mix, NURand s_id), K-SET strategy (headline), with
PART and TPL measured on the same bulks.  One "step" = one bulk through the whole
hot path: submit (ingest: validation + split lookups) and execute (emit, sort, rank,
group, k-set rounds) — every §8(a) row.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload tm1|tpcb|tpcb_tiny|tpcc]
  python bench.py --impl reference ...   # the oracle (serial CPU executor) as reference arm

For N > 1 (torchrun, one rank per GPU) the database is N times the configuration's
root keys (subscribers / branches / warehouses), sharded by root key, and every rank
submits a bulk of the configuration's size whose home roots are its own (weak scaling:
per-GPU work fixed).  Cross-shard transactions (TPC-B remote accounts, TPC-C remote
supply warehouses / customers) are packed by the engine and exchanged with NCCL
all-to-all before ranking; remote fragment outputs come back the same way
(paper_1103_3105_b200/shard.py).  All of it is inside the timed step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "bulk transactions/sec (TM-1, TPC-B, TPC-C) at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "txn/s"

WORKLOADS = {
    "tm1": dict(schema=W.TM1, dims=W.Tm1Dims(1_000_000), n=1_000_000, kw=dict(dist="nurand"),
                desc="TM-1 (TATP) 1M subscribers, bulk 1M, standard mix, NURand s_id"),
    "tm1_uniform": dict(schema=W.TM1, dims=W.Tm1Dims(1_000_000), n=1_000_000, kw=dict(dist="uniform"),
                        desc="TM-1 (TATP) 1M subscribers, bulk 1M, standard mix, uniform s_id"),
    "tpcb": dict(schema=W.TPCB, dims=W.TpcbDims(1000, 10, 100_000), n=4_000_000, kw=dict(remote_pct=15.0),
                 desc="TPC-B 1,000 branches, bulk 4M, uniform, 15% remote accounts"),
    "tpcb_tiny": dict(schema=W.TPCB, dims=W.TpcbDims(1, 10, 100_000), n=4096, kw={},
                      desc="TPC-B tiny: 1 branch, 10 tellers, 100k accounts, bulk 4,096"),
    "tpcb_hot": dict(schema=W.TPCB, dims=W.TpcbDims(1000, 10, 100_000), n=4_000_000,
                     kw=dict(remote_pct=15.0, alpha=0.1),
                     desc="TPC-B 1,000 branches, bulk 4M, hot-branch alpha=0.1, 15% remote accounts"),
    "tpcc": dict(schema=W.TPCC, dims=W.TpccDims(64, 10, 3000, 100_000), n=1_000_000, kw={},
                 desc="TPC-C NewOrder+Payment, 64 warehouses, bulk 1M"),
}
# NEXT-1: the same bulks under the ADD conflict rule (GPUTX_FLAG_ADD_RULE:
# commutative balance increments do not conflict with each other; PAPER.md:475(c)).
for _k in ("tpcb", "tpcb_hot", "tpcc"):
    WORKLOADS[_k + "_add"] = dict(WORKLOADS[_k], add_rule=True,
                                  desc=WORKLOADS[_k]["desc"] + ", ADD conflict rule (commutative increments)")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# --------------------------------------------------------------------------------------
# algorithmic bytes (DESIGN.md §"Roofline"): what the method itself must move
# --------------------------------------------------------------------------------------
def exec_bytes(schema: int, bulk, status: np.ndarray) -> int:
    """Bytes the k-set executor must read/write for this bulk: perm index (4), type (1),
    param offset (4), params (4/word), the columns each procedure touches on its
    committed or aborted path (App. B profiles), status byte of aborts, output bytes."""
    t = bulk.type
    nw = np.diff(bulk.param_off.astype(np.int64))
    base = 9 + 4 * nw
    ok = status == 0
    if schema == W.TPCB:
        per = base + 3 * 16 + 20 + 8                 # A/T/B read+write, history row, output
        return int(per.sum())
    if schema == W.TM1:
        extra = np.zeros(t.shape[0], np.int64)
        extra[t == W.TM1_GSD] = 36 + 36
        g = t == W.TM1_GND
        extra[g] = 2 + np.where(ok[g], 6 + 2 * (8 + 8) + 4, 1)       # ~2 qualifying rows read+written
        a = t == W.TM1_GAD
        extra[a] = 1 + np.where(ok[a], 14 + 16, 1)
        u = t == W.TM1_USD
        extra[u] = 1 + np.where(ok[u], 5, 1)
        extra[t == W.TM1_UL] = 4
        i = t == W.TM1_ICF
        extra[i] = 2 + np.where(ok[i], 10, 1)
        d = t == W.TM1_DCF
        extra[d] = 1 + np.where(ok[d], 1, 1)
        return int((base + extra).sum())
    # TPC-C: NO: district r/w 8, per line stock 4x(r+w)=48 -> ~ (4+8+4+4)*2 + price 4 + orig 2 + OL row 32 + out 12;
    #        order/new_order rows 40, discount/tax 12, out 16.   Payment: W/D ytd 32, customer 40, hist 28, out 16.
    no = t == W.TPCC_NEWORDER
    cnt = np.zeros(t.shape[0], np.int64)
    offs = bulk.param_off[:-1].astype(np.int64)
    cnt[no] = bulk.param_words[offs[no] + 3]
    per = base.copy()
    per[no] += np.where(ok[no], 8 + 40 + 12 + 16 + cnt[no] * (40 + 6 + 32 + 12), 1)
    per[~no] += np.where(ok[~no], 32 + 40 + 28 + 16, 1)
    return int(per.sum())


def rank_bytes(schema: int, records: int, passes: int, n: int, kernel: str = "") -> int:
    """Iterated scan (TPC-B; TPC-C per window): per pass, read each sorted record (8 B) and gather
    its transaction's depth (4 B); plus the initial zeroing of D (4 B/txn).
    TM-1 streaming rank (one pass): read each record once (8 B), write D once per
    transaction (4 B) after zeroing it (4 B).
    Spine walk (TPC-B / TPC-C default, one pass over all records): each record read once (8 B)
    by the last-write scan and the link passes, one depth access per record (4 B), plus the
    zeroing of D (4 B/txn) -- the iterated-scan formula with one pass over the whole bulk."""
    if kernel == "sp_walk_kernel":
        return records * 12 + 4 * n
    if schema == W.TM1:
        return records * 8 + 8 * n
    if schema == W.TPCC:
        # windowed rank: a pass sweeps one window's records only; windows of
        # 2^17 transactions (the library default), records assumed even across windows
        nwin = max(1, -(-n // (1 << 17)))
        return passes * (records // nwin) * 12 + 4 * n
    return passes * records * 12 + 4 * n


def rank_kernel_name(schema: int, add_rule: bool = False) -> str:
    """The rank kernel the library runs by default (engine.cu gputx_open_db)."""
    if schema in (W.TPCB, W.TPCC) and not add_rule:
        return "sp_walk_kernel"                # spine-streaming rank (one pass)
    if schema == W.TPCB:
        return "rank_kernel"
    return {W.TM1: "rank_stream_tm1_kernel", W.TPCC: "rank_window_kernel"}[schema]


def ncu_traffic(workload: str, kernel: str):
    """DRAM bytes per launch of `kernel` on `workload` from the committed ncu --set full
    captures (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        e = json.load(open(p))[workload][kernel]
        return e["dram_bytes_per_launch"], e
    except Exception:
        return None, None


# --------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# --------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.time(), ln.strip()))

    def wait_first(self, timeout: float = 5.0):
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.05)

    def mark(self):
        return time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0: float = 0.0, t1: float = float("inf")):
        """Median SM clock and active throttle reasons of the samples taken in [t0, t1]
        (all samples if the window caught none: nvidia-smi samples every 100 ms)."""
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inwin = [ln for t, ln in self.lines if t0 <= t <= t1]
        window = "timed region"
        if not inwin:
            # nearest samples around the window
            inwin = [ln for t, ln in self.lines if t0 - 0.5 <= t <= t1 + 0.5] or [ln for _, ln in self.lines]
            window = "around the timed region"
        for ln in inwin:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


# --------------------------------------------------------------------------------------
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if (torch.cuda.is_available() and args.impl != "reference") else "gloo"
        # GPUTX_DIST_BACKEND=gloo: several ranks on one GPU (host-staged all-to-all; tests only)
        backend = os.environ.get("GPUTX_DIST_BACKEND", backend)
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        pg = dist
    return ws, rank, local, pg


def reduce_max(dist, x: float, dev=None) -> float:
    """Max of x over ranks (device time of the slowest rank); identity at N = 1."""
    if dist is None:
        return x
    import torch
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_inputs(wl, rank: int, ws: int, steps: int, seed: int):
    """(dims, image, bulks): the configuration itself at N = 1; at N > 1 the weak-scaled
    global database (same image on every rank) and this rank's home bulks (global ts)."""
    nb = min(steps, 3)
    if ws == 1:
        dims = wl["dims"]
        image = W.make_db(wl["schema"], dims, seed=seed)
        bulks = [W.make_bulk(wl["schema"], dims, wl["n"], seed + k, **wl["kw"]) for k in range(nb)]
        return dims, image, bulks
    dims = W.scaled_dims(wl["schema"], wl["dims"], ws)
    image = W.make_db(wl["schema"], dims, seed=seed)
    bulks = [W.shard_bulk(wl["schema"], dims, wl["n"], seed + k, rank, ws, **wl["kw"]) for k in range(nb)]
    return dims, image, bulks


def oracle_rate(wl, image, bulks, min_seconds: float, max_runs: int, first=None):
    """The oracle (serial ts-order executor, one host core) on a bounded sample:
    successive bulks on the evolving state until min_seconds of loop time; committed
    transactions per second of loop time.  `first`: the oracle's result of bulk 0 on
    `image` already computed (the parity gate's), counted as the first sample."""
    import oracle
    cur = image
    secs, txns, runs, committed = 0.0, 0, 0, 0
    while runs < max_runs and (secs < min_seconds or runs == 0):
        b = bulks[runs % len(bulks)]
        r = first if (runs == 0 and first is not None) else \
            oracle.run(wl["schema"], wl["dims"].dims, cur, b, first_ts=txns)
        cur = r.db
        secs += r.seconds
        txns += b.n
        committed += int((r.status == 0).sum())
        runs += 1
    return committed / secs, txns, runs, secs


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, wl, ws, rank):
    """The reference arm: the oracle (serial ts-order executor, one host core), as it
    stands, on the headline workload; rank 0 only (other ranks exit without work)."""
    if rank != 0:
        return 0
    _, image, bulks = make_inputs(wl, 0, 1, max(args.steps, 1), args.seed)
    import oracle
    cur = image
    for k in range(args.warmup):
        cur = oracle.run(wl["schema"], wl["dims"].dims, cur, bulks[k % len(bulks)]).db
    secs = []
    txns = committed = 0
    for k in range(args.steps):
        b = bulks[k % len(bulks)]
        r = oracle.run(wl["schema"], wl["dims"].dims, cur, b, first_ts=txns)
        cur = r.db
        secs.append(r.seconds)
        txns += b.n
        committed += int((r.status == 0).sum())
    value = committed / sum(secs)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sum(secs) / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": config_of(args, wl, wl["dims"], 1),
        "all_txn_per_s": txns / sum(secs),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} bulks of {wl['n']} txns ({wl['desc']}), serial loop only",
                         "cpu": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(args, wl, dims, ws):
    c = {"workload": wl["desc"], "strategy": args.strategy, "bulk": wl["n"], "dims": list(dims.dims),
         "conflict_rule": "R/W + ADD" if wl.get("add_rule") else "R/W (paper)",
         "l2": "flushed (256 MiB write) before every timed step", "inputs": "resident in HBM (value); "
         "pinned host (e2e)", "value_counts": "committed transactions (SPEC.md:500); all_txn_per_s counts aborts too"}
    if ws > 1:
        if args.scaling == "strong":
            c["sharding"] = (f"{ws} shards by root key of the configuration's {dims.dims[0]} roots, one bulk of "
                             f"{wl['n']} transactions in total (strong scaling); cross-shard fragments exchanged "
                             "inside the step")
        else:
            c["sharding"] = (f"{ws} shards by root key, bulk {wl['n']} per shard (weak scaling); cross-shard "
                             "fragments exchanged inside the step")
        c["exchange"] = ("torch.distributed all-to-all of library-packed records" if os.environ.get("GPUTX_NO_P2P")
                         else "fused in the library: P2P stores into the owner shard's HBM arena (CUDA IPC)")
    return c


def _diff(ref, st, out, got):
    """First difference between the oracle's result and the GPU's (None if identical)."""
    if not np.array_equal(st, ref.status):
        return f"status differs at {int(np.flatnonzero(st != ref.status)[0])}"
    if not np.array_equal(out, ref.out):
        return f"output differs at txn {int(np.flatnonzero((out != ref.out).any(axis=1))[0])}"
    for k, a in ref.db.items():
        if not np.array_equal(a, got[k]):
            return f"column {k} differs"
    return None


def parity_gate(wl, db, dims, image, bulk0, strategy):
    """SPEC.md:499 / SURVEY.md §2.5: before any number is reported, the GPU's result of
    bulk 0 on the pristine image must equal the oracle's (Definition 1) element by element:
    statuses, output records and every column.  Runs outside the timed region; the oracle
    result it compares against is the first sample of the cpu_baseline leg."""
    import oracle
    ref = oracle.run(wl["schema"], dims.dims, image, bulk0, first_ts=0)
    db.reset()
    db.submit(bulk0)
    db.execute(strategy)
    st, out = db.read_results()
    got = db.read_image(image)
    err = _diff(ref, st, out, got)
    db.reset()
    return ref, err


def spawn_ranks(args):
    """--gpus N without a launcher: re-run this script under torch.distributed.run with N
    processes (one per GPU), 127.0.0.1 rendezvous."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def make_inputs_strong(wl, rank: int, ws: int, steps: int, seed: int):
    """Strong scaling: the configuration's own database and ONE bulk of the configuration's
    size in total; rank r submits the transactions whose home root it owns (global ts)."""
    nb = min(steps, 3)
    dims = wl["dims"]
    image = W.make_db(wl["schema"], dims, seed=seed)
    bulks = [W.split_home(W.make_bulk(wl["schema"], dims, wl["n"], seed + k, **wl["kw"]), dims, ws)[rank]
             for k in range(nb)]
    return dims, image, bulks


def measure(args, name, ws, rank, dist, dev, stream, clk, headline: bool):
    """One workload: timed K-SET (or --strategy) steps on device-resident bulks, the e2e
    loop through the C ABI with pinned host buffers, the other strategies, the roofline of
    the dominant kernel, the cpu_baseline and the parity gate.  Returns the JSON object."""
    import torch
    from paper_1103_3105_b200 import Database

    wl = WORKLOADS[name]
    strong = ws > 1 and args.scaling == "strong"
    if strong:
        dims, image, bulks = make_inputs_strong(wl, rank, ws, max(args.steps, 1), args.seed)
    else:
        dims, image, bulks = make_inputs(wl, rank, ws, max(args.steps, 1), args.seed)
    n_total = wl["n"] if strong else ws * wl["n"]              # transactions of one global step
    cap = 3 * (args.warmup + args.steps) + 12          # bulks the merged insert tables must hold
    nmax = max(b.n for b in bulks)
    max_bulk = nmax if ws == 1 else min(1 << 24, nmax + nmax // 2 + 1024)
    # single GPU: packed output records (GPUTX_FLAG_PACKED_OUT) -- the result transfer moves
    # only what the procedures return; sharded handles keep the stride
    db = Database(wl["schema"], dims.dims, max_bulk, image, device=dev.index, stream=stream.cuda_stream,
                  insert_capacity=cap, shard=rank if ws > 1 else 0, nshards=ws,
                  add_rule=wl.get("add_rule", False), packed_out=ws == 1,
                  deferred_check=ws == 1)      # TM-1: the validation verdict comes with execute

    # ---- parity gate (N = 1): bulk 0 vs the oracle, before anything is timed ----------
    parity, parity_err, ref0 = None, None, None
    if ws == 1 and not args.no_parity:
        ref0, parity_err = parity_gate(wl, db, dims, image, bulks[0], args.strategy)
        parity = parity_err is None
    if ws > 1:
        del image
        image = None

    class DevBulk:
        def __init__(self, b):
            self.type = torch.from_numpy(b.type).to(dev)
            self.param_off = torch.from_numpy(b.param_off.view(np.int32)).to(dev)
            self.param_words = torch.from_numpy(b.param_words.view(np.int32)).to(dev)
            self.ts = torch.from_numpy(b.ts.view(np.int32)).to(dev) if b.ts is not None else None

    dbulks = [DevBulk(b) for b in bulks]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if ws > 1:
        from paper_1103_3105_b200 import shard as SH
        if not os.environ.get("GPUTX_NO_P2P"):
            SH.connect_p2p(db)         # the library's fused exchange over peer memory (CUDA IPC)

    def step_dev(k, strategy):
        """Launch one step; returns the function that completes it (-> stats).  Single
        GPU: gputx_execute_async, so the end event is recorded behind the bulk's last
        kernel, not behind the host's stats bookkeeping (gputx_wait)."""
        b = dbulks[k % len(dbulks)]
        if ws > 1:
            st = SH.step(db, b, strategy, on_device=True)
            return lambda: st
        db.submit(b, on_device=True)
        db.execute_async(strategy)
        return db.wait

    def barrier():
        if dist is not None:
            dist.barrier()

    window = [0.0, 0.0]

    def timed(strategy, steps, warmup):
        for k in range(warmup):
            step_dev(k, strategy)()
        torch.cuda.synchronize()
        barrier()
        clk.wait_first()
        window[0] = time.time()
        ms, stats = [], []
        for k in range(steps):
            flush.fill_(k & 0xFF)                        # L2 flush, outside the timed window
            stream.synchronize()                         # (done before the window opens)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            finish = step_dev(warmup + k, strategy)
            e1.record(stream)
            stats.append(finish())
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        window[1] = time.time()
        barrier()
        return ms, stats

    def max_over_ranks(x: float) -> float:
        return reduce_max(dist, x, dev)

    def sum_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t)
        return float(t.item())

    # ---- headline strategy, device-resident inputs -----------------------------------
    db.reset()
    ms, stats = timed(args.strategy, args.steps, args.warmup)
    clocks = clk.summary(*window)
    total_ms = max_over_ranks(sum(ms))
    committed = sum_over_ranks(float(sum(s["committed"] for s in stats)))
    allt = sum_over_ranks(float(sum(s["n"] for s in stats)))
    value = committed / (total_ms / 1e3)
    launches = int(sum(s["launches"] for s in stats))
    st_host, _ = db.read_results()                    # results of the last step (byte model)

    # ---- e2e through the C ABI with host (pinned) buffers ----------------------------
    class HostBulk:
        def __init__(self, b):
            self.type = torch.from_numpy(b.type).pin_memory().numpy()
            self.param_off = torch.from_numpy(b.param_off.view(np.int32)).pin_memory().numpy().view(np.uint32)
            self.param_words = torch.from_numpy(b.param_words.view(np.int32)).pin_memory().numpy().view(np.uint32)
            self.ts = (torch.from_numpy(b.ts.view(np.int32)).pin_memory().numpy().view(np.uint32)
                       if b.ts is not None else None)

        def nbytes(self):
            return sum(a.nbytes for a in (self.type, self.param_off, self.param_words, self.ts) if a is not None)

    hb = [HostBulk(b) for b in bulks]
    st_pin = torch.empty(nmax, dtype=torch.uint8).pin_memory().numpy()
    out_pin = torch.empty(nmax * db.stride, dtype=torch.uint8).pin_memory().numpy().reshape(nmax, db.stride)
    e2e_ms = []
    e2e_committed = 0
    e2e_out_bytes = 0.0
    if ws == 1:
        # gputx_run_bulks: the K bulks' H2D / D2H overlap the executions (two copy streams);
        # results alternate between two pinned host buffers (each read back at the end)
        st2 = [st_pin, torch.empty(nmax, dtype=torch.uint8).pin_memory().numpy()]
        out2 = [out_pin, torch.empty(nmax * db.stride, dtype=torch.uint8).pin_memory().numpy().reshape(nmax, db.stride)]
        seq = [hb[k % len(hb)] for k in range(args.warmup + args.steps)]
        db.run_bulks(seq[:args.warmup], args.strategy, [st2[k % 2] for k in range(args.warmup)],
                     [out2[k % 2] for k in range(args.warmup)])
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sts = db.run_bulks(seq[args.warmup:], args.strategy, [st2[k % 2] for k in range(args.steps)],
                           [out2[k % 2] for k in range(args.steps)], stats=True)
        e1.record(stream)
        e1.synchronize()
        e2e_ms = [e0.elapsed_time(e1)]
        e2e_committed = sum(x["committed"] for x in sts)
        e2e_out_bytes = float(np.mean([x["out_bytes"] for x in sts]))
    for k in range(args.warmup + args.steps) if ws > 1 else []:
        b = hb[k % len(hb)]
        nb_ = b.type.shape[0]
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if ws > 1:
            SH.step(db, b, args.strategy, on_device=False)
        else:
            db.submit(b, on_device=False)
            db.execute_nostats(args.strategy)
        db.read_results(st_pin[:nb_], out_pin[:nb_])
        e1.record(stream)
        e1.synchronize()
        if k >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
            e2e_committed += int((st_pin[:nb_] == 0).sum())
    e2e_total = max_over_ranks(sum(e2e_ms))
    e2e_committed = sum_over_ranks(float(e2e_committed))
    h2d = int(np.mean([b.nbytes() for b in hb]))
    # status u8[n] + the output records the result read moved (packed at N = 1)
    d2h = int(np.mean([b.type.shape[0] for b in hb]) + (e2e_out_bytes if ws == 1 else
                                                           np.mean([b.type.shape[0] for b in hb]) * db.stride))
    # the link the e2e number is bound by: pinned copies of one step's bytes, each direction
    # alone (outside every timed region); the overlapped e2e step can't beat max(H2D, D2H)
    pcie = {}
    for pkey, nbytes, hd in (("h2d_gbs", h2d, True), ("d2h_gbs", d2h, False)):
        hbuf = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        dbuf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        best = 1e9
        for _ in range(10):                        # (the first copies of a fresh pinned buffer are slow)
            torch.cuda.synchronize()
            c0 = torch.cuda.Event(enable_timing=True)
            c1 = torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            (dbuf.copy_(hbuf, non_blocking=True) if hd else hbuf.copy_(dbuf, non_blocking=True))
            c1.record(stream)
            c1.synchronize()
            best = min(best, c0.elapsed_time(c1))
        pcie[pkey] = nbytes / (best / 1e3) / 1e9
        del hbuf, dbuf
    pcie["transfer_floor_ms"] = max(h2d / pcie["h2d_gbs"], d2h / pcie["d2h_gbs"]) / 1e6
    # both directions at once on two streams, as the overlapped e2e step moves them (a
    # direction alone is faster than the two together on this link)
    hi, di = torch.empty(h2d, dtype=torch.uint8).pin_memory(), torch.empty(h2d, dtype=torch.uint8, device=dev)
    ho, do = torch.empty(d2h, dtype=torch.uint8).pin_memory(), torch.empty(d2h, dtype=torch.uint8, device=dev)
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = 1e9
    for _ in range(10):
        torch.cuda.synchronize()
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        sa.wait_event(c0)
        sb.wait_event(c0)
        with torch.cuda.stream(sa):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(sb):
            ho.copy_(do, non_blocking=True)
        stream.wait_stream(sa)
        stream.wait_stream(sb)
        c1.record(stream)
        c1.synchronize()
        best = min(best, c0.elapsed_time(c1))
    pcie["bidir_floor_ms"] = best
    del hi, di, ho, do

    # ---- other strategies on the same bulks ------------------------------------------
    others = {}
    for s in [x for x in args.others.split(",") if x and x != args.strategy]:
        m2, s2 = timed(s, max(2, args.steps // 2), 1)
        tot = max_over_ranks(sum(m2))
        c2 = sum_over_ranks(float(sum(x["committed"] for x in s2)))
        others[s] = {"value": c2 / (tot / 1e3), "ms_per_step": tot / len(m2),
                     "ms_exec": statistics.mean(x["ms_exec"] for x in s2),
                     "max_chain": s2[-1]["max_chain"], "parts": s2[-1]["parts"]}
        if s == "auto":
            others[s]["chose"] = s2[-1]["strategy"]
            others[s]["w0_d_c"] = [s2[-1]["zero_set"], s2[-1]["depth"], s2[-1]["cross"]]

    # ---- roofline of the dominant kernel ---------------------------------------------
    peak, peak_kind = _peaks()
    phase = {k: statistics.mean(s[k] for s in stats) for k in
             ("ms_ingest", "ms_exchange", "ms_emit", "ms_sort", "ms_rank", "ms_group", "ms_exec", "ms_total")}
    last = stats[-1]
    b_last = bulks[(args.warmup + args.steps - 1) % len(bulks)]
    cand = {}
    eff = last["strategy"]                                  # auto: the strategy Algorithm 1 chose
    nloc = b_last.n
    if last["rank_passes"]:
        rk = rank_kernel_name(wl["schema"], wl.get("add_rule", False))
        cand[rk] = (rank_bytes(wl["schema"], last["records"], last["rank_passes"], nloc, rk), phase["ms_rank"])
    if ws == 1:
        # K-SET's dataflow executor (TPC-C default, stats flag 2) runs the counter-lock kernels
        # owner-local rounds (TM-1 / TPC-B / micro default, stats flag 4) run kset_own_exec_kernel
        fl = last.get("flags", 0)
        ek = (("tpl_exec_warp_kernel" if wl["schema"] == W.TPCC else "tpl_exec_persistent_kernel")
              if eff == "kset" and (fl & 2) else "kset_chain_exec_kernel" if eff == "kset" and (fl & 16)
              else "kset_own_pipe_kernel" if eff == "kset" and (fl & 4) else f"{eff}_exec_kernel")
        cand[ek] = (exec_bytes(wl["schema"], b_last, st_host), phase["ms_exec"])
    if last["records"] and phase["ms_sort"] > 0:
        # the (item, ts) radix sort (the sort phase: histogram + digit passes): a sort's
        # algorithmic floor is one read and one write of every 8-B record
        cand["rs_pass_kernel"] = (16 * last["records"], phase["ms_sort"])
    kname = max(cand, key=lambda k: cand[k][1]) if cand else None
    roofline = None
    if kname:
        kbytes, kms = cand[kname]
        achieved = kbytes / (kms / 1e3) / 1e9
        traffic, tr = ncu_traffic(name, kname)
        roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_source": tr and tr["source"],
                    # the ncu DRAM fraction of the same capture (cold cache)
                    "ncu_dram_frac": tr and traffic / (tr["ncu_us_per_launch"] * 1e-6) / 1e9 / peak,
                    "ncu_l2_hit_pct": tr and tr["l2_hit_pct"],
                    "peak_source": peak_kind,
                    "algorithmic_bytes": kbytes, "kernel_ms": kms,
                    # K-SET exec is bounded by its d+1 dependent rounds: the
                    # per-round latency is the number that moves it on deep graphs
                    "critical_path": ({"rounds": last["depth"] + 1,
                                       "us_per_round": 1e3 * phase["ms_exec"] / (last["depth"] + 1)}
                                      if eff == "kset" else {"max_chain": last["max_chain"]} if eff == "part"
                                      else None),
                    "share_of_step": kms / phase["ms_total"] if phase["ms_total"] else None}

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N = 1) -----------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, txns, runs, secs = oracle_rate(wl, image, bulks, args.cpu_seconds, 1000, first=ref0)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{runs} bulk(s) x {wl['n']} txns of the same workload, serial loop {secs:.2f} s "
                         "(committed txn/s)",
               "cpu": cpu_model(), "nproc": os.cpu_count()}
    db.close()
    del flush
    torch.cuda.empty_cache()
    res = {
        "workload": name, "value": value if parity is not False else 0.0, "unit": UNIT,
        "ms_per_step": total_ms / args.steps, "all_txn_per_s": allt / (total_ms / 1e3),
        "parity": parity if parity is not None else "not checked (N>1: tests/test_gpu_shard.py)",
        "e2e": {"value": e2e_committed / (e2e_total / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / args.steps, "pcie": pcie,
                "method": ("gputx_run_bulks: H2D of bulk i+1 and D2H of bulk i-1 overlap bulk i (two copy "
                           "streams); back-to-back bulks, no L2 flush in between; packed output records "
                           "(GPUTX_FLAG_PACKED_OUT); TM-1 / micro K-SET pipelined (no host round trip "
                           "between bulks)") if ws == 1 else
                          "per step: H2D, sharded step, D2H (serial)"},
        "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
        "phases_ms": phase,
        "graph": {"depth": last["depth"], "zero_set": last["zero_set"], "records": last["records"],
                  "rank_passes": last["rank_passes"], "committed": last["committed"], "aborted": last["aborted"]},
        "strategies": {args.strategy: {"value": value, "ms_per_step": total_ms / args.steps}, **others},
        "config": config_of(args, wl, dims, ws), "n_total_per_step": n_total,
    }
    if parity_err:
        res["parity_error"] = parity_err
    if last.get("flags"):
        res["exec_flags"] = last["flags"]
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="tm1", choices=sorted(WORKLOADS))
    ap.add_argument("--also", default="default", help="further workloads measured after the headline, comma "
                    "separated; 'default' = tpcb,tpcc when the headline is tm1 (BASELINE's three metric "
                    "workloads), 'none' = headline only")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = bulk per GPU fixed, database N times the roots; strong = the "
                    "configuration's database and one bulk in total, sharded (BASELINE config 4)")
    ap.add_argument("--strategy", default="kset", choices=["kset", "part", "tpl", "auto"])
    ap.add_argument("--others", default="part,tpl,auto", help="extra strategies measured on the same bulks "
                    "(auto: Algorithm 1, PAPER.md:422-437, with the library's default thresholds)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU work of the cpu_baseline sample (the contract asks for ~10-30 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    wl = WORKLOADS[args.workload]
    ws, rank, local, dist = dist_setup(args)
    if ws != args.gpus and args.impl != "reference":
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.impl == "reference":
        return run_reference(args, wl, ws, rank)

    import torch

    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # one non-default stream for the engine (cfg.stream) and every torch op of the step:
    # copies, the L2 flush and the timing events are ordered with the engine's kernels
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    also = args.also
    if also == "default":
        also = "tpcb,tpcc" if args.workload == "tm1" else "none"
    extra = [x for x in also.split(",") if x and x != "none" and x != args.workload]
    clk = Clocks(local).__enter__()                      # sampling starts now
    head = measure(args, args.workload, ws, rank, dist, dev, stream, clk, True)
    subs = {x: measure(args, x, ws, rank, dist, dev, stream, clk, False) for x in extra}
    clk.__exit__()
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded generators, workloads/)",
        "config": head["config"], "parity": head["parity"], "all_txn_per_s": head["all_txn_per_s"],
        "e2e": head["e2e"], "gpu_launches": head["gpu_launches"], "roofline": head["roofline"],
        "cpu_baseline": head["cpu_baseline"], "clocks": head["clocks"], "phases_ms": head["phases_ms"],
        "graph": head["graph"], "strategies": head["strategies"],
    }
    for k in ("parity_error", "exec_flags"):
        if k in head:
            line[k] = head[k]
    if subs:
        line["workloads"] = subs
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0 if all(x["parity"] is not False for x in [head, *subs.values()]) else 3


if __name__ == "__main__":
    sys.exit(main())
